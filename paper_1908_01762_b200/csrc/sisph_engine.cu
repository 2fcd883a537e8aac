// sisph_engine.cu — host runtime behind the C ABI of include/sisph.h.
//
// One Engine<T, D> per handle (T = float | double, D = 2 | 3).  It owns the
// device state in cell-sorted structure-of-arrays order (fluid slots [0, Nf),
// static wall slots [Nf, Ntot)), runs every step of the hot path as the
// kernels of sisph_kernels.cuh on one stream, and keeps the PPE stop decision
// on the device (the host only polls a pinned copy of the control block
// between speculative batches of sweeps).
//
// Slab ranks (sisph_create_dist): the domain is cut into
// nranks slabs along one axis; a rank owns the particles of its slab and
// holds read-only halo copies ("ghosts") of the neighbour slabs' particles
// within Gw = 1.3 x 3h of its faces.  Slots: owned fluid [0, Nfo), ghost
// fluid [Nfo, Nf), owned walls [Nf, Nf + Nwo), ghost walls [Nf + Nwo, Ntot);
// ghosts carry the cell key + ncells, so one stable sort keeps each set
// cell-sorted and contiguous.  Every kernel computes owned rows only; each
// ghost value a kernel reads is refreshed from its owner first (halo
// exchange of the transport, sisph_comm.cuh), the sweep's residual sums and
// Lambda are allreduced, and every rank takes the same decisions from the
// same bits.  Migration of fluid particles to the neighbour slab happens at
// the start of each step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <utility>
#include <set>
#include <vector>

#include "../../include/sisph.h"
#include "sisph_comm.cuh"
#include "sisph_kernels.cuh"

namespace sb {

static thread_local std::string g_thread_err;

#define SCK(call)                                                                          \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            err = std::string(#call) + ": " + cudaGetErrorString(e_);                      \
            return SISPH_ECUDA;                                                            \
        }                                                                                  \
    } while (0)
#define SRET(x)                 \
    do {                        \
        int r_ = (x);           \
        if (r_) return r_;      \
    } while (0)

static inline int nblk(long n, int bs) { return (int)((n + bs - 1) / bs); }

enum Phase { IDLE = 0, PREDICTED = 1, SOLVED = 2 };

// distribution of a handle over slab ranks (resolved from sisph_dist)
struct DistInfo {
    int nranks = 1, rank = 0, axis = 0;
    Transport* tp = nullptr;   // owned by the engine (nranks > 1, or the slab path forced)
};

struct EngineBase {
    std::string err;
    int64_t n = 0, nf = 0, nw = 0;
    int dim = 2;
    virtual ~EngineBase() {}
    virtual int build() = 0;
    virtual int predict(double dt) = 0;
    virtual int solve(double tol, int max_iter, int* iters, double* res) = 0;
    virtual int correct(double dt) = 0;
    virtual int step(double dt, sisph_step_report* rep) = 0;
    virtual int get_field(int f, double* out, int64_t count) = 0;
    virtual int set_field(int f, const double* in, int64_t count) = 0;
    virtual int get_field_f32(int f, float* out, int64_t count) = 0;
    virtual int set_field_f32(int f, const float* in, int64_t count) = 0;
    virtual int stage_field(int f, const void* in, int64_t count, bool f32) = 0;
    virtual int commit_staged() = 0;
    virtual int fetch_field(int f, void* out, int64_t count, bool f32) = 0;
    virtual int fetch_wait() = 0;
    virtual int get_order(int64_t* ids) = 0;
    virtual int get_neighbors(int64_t* off, int64_t* ids, int64_t cap, int64_t* total) = 0;
    virtual int get_neighbors_of(const int64_t* which, int64_t m, int64_t* off, int64_t* ids, int64_t cap,
                                 int64_t* total) = 0;
    virtual int owned_counts(int64_t* nfo, int64_t* nwo) = 0;
    virtual int next_dt(double* dtn, double* dtc, double* dtf) = 0;
    virtual int sweep_timing(double* ms, int* n) = 0;
    virtual int sync() = 0;
    int timing = 0;
    int64_t nlaunch = 0;  // kernel launches issued (all entry points)
};

template <class T> static T* dalloc(size_t n, std::string& err, int& rc)
{
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
        err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        rc = SISPH_ENOMEM;
        return nullptr;
    }
    return (T*)p;
}

template <class T, int D> struct Engine : EngineBase {
    using V = V4<T>;
    Params<T> P;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int Nf = 0, Nw = 0, Ntot = 0, ncells = 0;
    int Nfo = 0, Nwo = 0;          // owned fluid / walls (= Nf / Nw on one GPU)
    int capT = 0, capF = 0;        // slot capacities (total, fluid)
    int phase = IDLE;
    int min_iter = 2, max_iter = 1000, K = 10;
    double tol = 1e-2;
    double last_dt = 0;

    // device state
    V *pos = nullptr, *pos_alt = nullptr, *vel = nullptr, *vel_alt = nullptr, *us = nullptr, *us_alt = nullptr;
    V *vt = nullptr, *vt_alt = nullptr, *rn = nullptr, *rstar = nullptr, *nrm = nullptr, *nstmp = nullptr;
    V* uwl = nullptr;         // prescribed wall velocity per relative wall slot (eq:vg-adami)
    bool uwl_set = false;     // uwl holds the walls' values (after the first wall sort)
    int pref_auto = 0;        // R33: p_ref from the first solve
    // R34 open boundaries: particle types of the fluid block, the dormant id pool
    int open_x = 0;
    std::set<int> pool;
    uint8_t *ptype = nullptr, *ptype_alt = nullptr;
    T* uout = nullptr;
    int* oflag = nullptr;
    int* olist = nullptr;
    int* onew = nullptr;
    int open_spawned = 0, open_deleted = 0;
    bool pref_done = false;
    // GTVF sub-step records (A14): per particle {r*, m / rho^2, r^k - r^0, 0} (two V4), ping-pong
    V *gtA = nullptr, *gtB = nullptr, *vk = nullptr;
    V *fx0 = nullptr, *dk = nullptr;   // fp32 GTVF: fixed-point r* (int4) and delta^k per slot
    V *recF = nullptr, *recS = nullptr;   // joint {r, m, u, rho} records of A8 / A11 (k_pack_rec)
    V* fnp = nullptr;       // non-pressure acceleration of A8 (adaptive dt)
    int* dcnt_w = nullptr;  // device flag of set_field's wall check
    bool stepped = false;   // a correct has completed: next_dt is defined
    bool pre_swept = false; // A11 ran the first Jacobi sweep (p^1 in p_alt, sums deferred)
    T *p = nullptr, *p_alt = nullptr, *rho = nullptr, *rho_alt = nullptr, *rhs = nullptr, *diag = nullptr;
    uint8_t *fs = nullptr, *fs_alt = nullptr;
    int *pid = nullptr, *pid_alt = nullptr;
    int *keys = nullptr, *rank = nullptr, *perm0 = nullptr, *perm = nullptr;
    int *ccount = nullptr, *fstart = nullptr, *wstart = nullptr, *bsum = nullptr;
    int *nbr = nullptr, *cnt = nullptr;
    int *nbr_in = nullptr, *cnt_in = nullptr;  // GTVF inner list (h~ < h)
    bool use_inner = false, inner_valid = false;
    int64_t gtvf_fallbacks = 0;
    // single per-step build (R3): loose list at r^n on the skin geometry PS,
    // walls binned for PS through wperm_s / wstart_s (recomputed when PS's grid changes)
    int *nbs = nullptr, *cnt_s = nullptr;
    int cap_s = 0;
    int *wperm_s = nullptr, *wstart_s = nullptr;
    int wnc_s[3] = {-1, -1, -1};
    Params<T> PS;
    int rebuild_mode = 0;   // 0: single build + filter when the skin fits, 1: always two exact builds
    int matrix_free = 0;    // 1: the sweep recomputes fac_ij from positions; 0: A11 stores it per pair
    T* coef = nullptr;      // stored per-pair part of fac_ij, blocked-ELL layout of nbr (fluid rows)
    uint4* code = nullptr;  // code mode: the sweep's 16-bit copy of the fluid rows' list (CodeWriter)
    int* nslot = nullptr;   // with coef in slot order
    int cc8 = 0;
    int build_mask = 1;     // 3D loose build: 1 = test-then-append (k_build_loose_m), 0 = k_build_loose (SISPH_BUILD_MASK)
    int use_codes = 0;      // SISPH_SWEEP_CODES=1: code mode (measured: sweep +12 %, A11 -20 %)
    bool skin_used = false;
    double skin_radius = 0;
    double extent = 0;      // max |coordinate| of the domain (rounding margin of the skin)
    Ctl* ctl = nullptr;
    Ctl* hctl = nullptr;  // pinned host mirror
    double* partials = nullptr;
    double* dtmp = nullptr;  // staging for get/set (n * 3 doubles)
    // sisph_stage_field / sisph_commit_staged: per-field device staging filled on an upload
    // stream (ust) while the handle's stream computes; commit scatters them on st
    struct Staged {
        void* buf = nullptr;
        size_t cap = 0;
        int64_t count = 0;
        bool f32 = false, pending = false;
        cudaEvent_t ev = nullptr;
    };
    static constexpr int NFIELD = 16;
    Staged stg[NFIELD];
    int stg_order[NFIELD] = {};
    int nstg = 0;
    cudaStream_t ust = nullptr;
    cudaEvent_t ev_consumed = nullptr;   // the last commit's scatters are done with the buffers
    bool consumed_rec = false;
    // sisph_fetch_field / sisph_fetch_wait: one field gathered into fbuf on st, copied to the
    // host on a download stream (dlst) while st goes on
    void* fbuf = nullptr;
    size_t fcap = 0;
    cudaStream_t dlst = nullptr;
    cudaEvent_t ev_fready = nullptr, ev_fdone = nullptr;
    bool fpending = false, fdone_rec = false;
    std::vector<int> tags_host;  // creation-order tags
    // timing mode: 0-3 step / predict / solve / correct boundaries; 4 after the build at r^n
    // (A1-A5); 5 / 6 around the r* filter (A9) or build; 7 / 8 around A11 (+ fused sweep)
    static constexpr int NEV = 9;
    cudaEvent_t ev[NEV] = {};
    unsigned evmask = 0;
    int mark(int k)
    {
        if (!timing) return SISPH_OK;
        SCK(cudaEventRecord(ev[k], st));
        evmask |= 1u << k;
        return SISPH_OK;
    }

    // ---------------------------------------------------------------- slab ranks
    Transport* tp = nullptr;
    int axis = 0;
    double slab_lo = 0, slab_hi = 0, glo = 0, ghi = 0;  // own slab and the global box along the axis
    int gper = 0;                                       // the axis is periodic globally
    double Gw = 0;                                      // halo width (>= every loose radius)
    int *dflag = nullptr, *dflag2 = nullptr, *dpre = nullptr, *dlist[3] = {nullptr, nullptr, nullptr};
    int *dcnt = nullptr, *hcnt = nullptr;               // small count exchanges (device / pinned host)
    int *fsend[2] = {nullptr, nullptr}, *fsend_pre[2] = {nullptr, nullptr};
    int nfs[2] = {0, 0}, nfr[2] = {0, 0};
    int* grecv = nullptr;                               // fluid halo record q -> ghost slot
    int *wsend[2] = {nullptr, nullptr};                 // owned-wall halo lists (relative slots)
    int nws[2] = {0, 0}, nwr[2] = {0, 0};
    int* wrecv = nullptr;                               // wall halo record q -> ghost wall (relative)
    int* inv = nullptr;
    char *sbuf[2] = {nullptr, nullptr}, *rbuf[2] = {nullptr, nullptr};
    size_t bufcap[2] = {0, 0};
    V* wtmp = nullptr;                                  // wall-block relocation staging
    char* wstage = nullptr;                             // relocate_walls: every array's wall block
    int64_t halo_bytes = 0;                             // bytes sent by halo / migration exchanges
    // fp32 GTVF sub-steps on slab ranks: the rows other ranks hold as ghosts (brow) are stepped
    // first, their delta halo runs on hst while the other rows (irow) are stepped (gcnt: the two
    // row counts on the device)
    int *bflag = nullptr, *brow = nullptr, *irow = nullptr, *gcnt = nullptr;
    cudaStream_t hst = nullptr;
    cudaEvent_t gev[2] = {nullptr, nullptr};
    // SISPH_GTVF_OVERLAP=1 (opt-in): measured on one B200 with the slab path talking to itself over
    // NCCL (bench.py --slab-self, C5), the 10 sub-steps take 1.19 ms overlapped against 1.13 ms
    // unsplit (an NCCL send to itself gains nothing from the overlap; the split costs a launch and
    // a tail per sub-step); across GPUs the halo's NVLink time is what it would hide
    int gtvf_overlap = 0;

    bool dist() const { return tp != nullptr; }

    ~Engine() override
    {
        void* ptrs[] = {pos, pos_alt, vel, vel_alt, us, us_alt, vt, vt_alt, rn, rstar, nrm, nstmp, uwl, gtA, gtB, vk, fx0, dk, recF, recS,
                        p, p_alt, rho, rho_alt, rhs, diag, fs, fs_alt, pid, pid_alt, keys, rank, perm0, perm,
                        ccount, fstart, wstart, bsum, nbr, cnt, ctl, partials, dtmp, nbr_in, cnt_in,
                        nbs, cnt_s, wperm_s, wstart_s, coef, dflag, dflag2, dpre, dlist[0], dlist[1], dlist[2],
                        dcnt, fsend[0], fsend[1], fsend_pre[0], fsend_pre[1], grecv, wsend[0], wsend[1], wrecv,
                        inv, sbuf[0], sbuf[1], rbuf[0], rbuf[1], wtmp, fnp, dcnt_w, ptype, ptype_alt, uout,
                        oflag, olist, onew, code, nslot, wstage, bflag, brow, irow, gcnt};
        if (st) cudaStreamSynchronize(st);
        for (void* q : ptrs)
            if (q) cudaFree(q);
        if (hctl) cudaFreeHost(hctl);
        if (hcnt) cudaFreeHost(hcnt);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : sev)
            if (e) cudaEventDestroy(e);
        delete tp;
        drop_graph();
        if (cst) cudaStreamDestroy(cst);
        if (ust) {
            cudaStreamSynchronize(ust);
            cudaStreamDestroy(ust);
        }
        for (auto& g : stg) {
            if (g.buf) cudaFree(g.buf);
            if (g.ev) cudaEventDestroy(g.ev);
        }
        if (ev_consumed) cudaEventDestroy(ev_consumed);
        if (dlst) {
            cudaStreamSynchronize(dlst);
            cudaStreamDestroy(dlst);
        }
        if (fbuf) cudaFree(fbuf);
        if (ev_fready) cudaEventDestroy(ev_fready);
        if (ev_fdone) cudaEventDestroy(ev_fdone);
        if (hst) {
            cudaStreamSynchronize(hst);
            cudaStreamDestroy(hst);
        }
        for (auto& e : gev)
            if (e) cudaEventDestroy(e);
        if (hdesc) cudaFreeHost(hdesc);
        if (ddesc) cudaFree(ddesc);
        if (own_stream && st) cudaStreamDestroy(st);
    }

    // ------------------------------------------------------------------ setup
    // Local particle arrays: fluid (tag 0) first, then walls; the first nwo
    // walls are owned (all of them on one GPU).  gid: creation id of each
    // local particle (NULL: its index).  n_glob: particle count of the whole
    // problem (size of the creation-id-order arrays of get/set_field).
    int init(const double* x, const double* u, const double* m, const double* r0, const int32_t* tags,
             const int64_t* gid, int64_t nloc, int64_t n_glob, const int32_t* tags_glob, double h,
             const sisph_domain* dom, const sisph_params* prm, const DistInfo* di, const double* slab)
    {
        n = n_glob;
        dim = D;
        tags_host.assign(tags_glob, tags_glob + n);
        std::vector<int> fid, wid;
        open_x = prm->open_x;
        for (int64_t k = 0; k < nloc; k++) {
            const int tg = tags[k];
            if (tg == SISPH_TAG_DORMANT) pool.insert(gid ? (int)gid[k] : (int)k);   // R34 id pool
            else if (tg == SISPH_TAG_WALL) wid.push_back((int)k);
            else fid.push_back((int)k);                                             // fluid, inlet, outlet
        }
        Nf = Nfo = (int)fid.size();
        Nw = (int)wid.size();
        Nwo = Nw;
        if (prm->device >= 0) SCK(cudaSetDevice(prm->device));
        if (prm->stream) {
            st = (cudaStream_t)prm->stream;
        } else {
            SCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own_stream = true;
        }
        for (auto& e : ev) SCK(cudaEventCreate(&e));
        const double R = 3.0 * h;
        if (di && di->tp) {
            tp = di->tp;
            axis = di->axis;
            glo = dom->lo[axis];
            ghi = dom->hi[axis];
            gper = dom->periodic[axis] ? 1 : 0;
            slab_lo = slab[0];
            slab_hi = slab[1];
            Gw = 1.3 * R * (1.0 + 1e-6);
        }
        // ------------------------------------------------ parameters
        memset(&P, 0, sizeof(P));
        P.dim = D;
        for (int a = 0; a < 3; a++) {
            P.nc[a] = 1;
            P.cell[a] = 1.0;
            P.lo[a] = dom->lo[a];
            P.hi[a] = dom->hi[a];
            P.per[a] = 0;
        }
        for (int a = 0; a < D; a++) {
            double lo = dom->lo[a], hi = dom->hi[a];
            int per = dom->periodic[a] ? 1 : 0;
            if (dist() && a == axis) {
                // the local box of a slab rank: its slab plus the halo layers, bounded
                lo = slab_lo - Gw;
                hi = slab_hi + Gw;
                per = 0;
            }
            double L = hi - lo;
            int nc = (int)floor(L / R);
            if (nc < 1) nc = 1;
            if (per && nc < 3) {
                err = "periodic axis " + std::to_string(a) + " has fewer than 3 cells of size >= 3h";
                return SISPH_EINVAL;
            }
            P.lo[a] = lo;
            P.hi[a] = hi;
            P.nc[a] = nc;
            P.cell[a] = L / nc;
            P.per[a] = per;
            P.Ld[a] = L;
            P.halfLd[a] = 0.5 * L;
            P.Lf[a] = (float)L;
            P.halfLf[a] = (float)(0.5 * L);
            P.L[a] = (T)L;
            P.halfL[a] = (T)(0.5 * L);
        }
        for (int a = 0; a < 3; a++) {
            P.fxs[a] = a < D ? P.Ld[a] / 4294967296.0 : 1.0;
            P.fxf[a] = (float)P.fxs[a];
        }
        long long nc_tot = (long long)P.nc[0] * P.nc[1] * P.nc[2];
        if (nc_tot > (1ll << 29)) {
            err = "cell grid too large";
            return SISPH_EINVAL;
        }
        ncells = (int)nc_tot;
        P.R2d = R * R;
        // fp32 prefilter band of the exact neighbour decision (R2): |fl32(r^2) - r^2| <= band R^2
        // for every pair near R with fp32 coordinates: each component difference carries <= u |d|
        // (u = 2^-24), a periodic image shift <= u 2 L_a (the shifted coordinate) + |L_f - L_d|
        // (the fp32 box length), the squares and sums <= 4 u r^2; doubled for safety.  Pairs
        // outside the band are decided by the fp32 comparison (it cannot disagree with the fp64
        // one there), pairs inside it in fp64 (exact_band): a narrow band keeps the lattices'
        // near-ties (C5: ~30 per particle at 3h) out of the fp64 path once they have moved
        {
            const double u = 1.0 / 16777216.0;
            double b = 10.0 * u;
            for (int a = 0; a < D; a++)
                if (P.per[a]) b += 2.0 * (2.0 * u * P.Ld[a] + fabs((double)P.Lf[a] - P.Ld[a])) / R;
            b *= 2.0;
            P.R2lo = nextafterf((float)(R * R * (1.0 - b)), 0.0f);
            P.R2hi = nextafterf((float)(R * R * (1.0 + b)), 1e30f);
        }
        P.R2cut = (T)(R * R * (1.0 + 1.0 / 1024.0));
        const double sigd = D == 2 ? 7.0 / (478.0 * M_PI) : 1.0 / (120.0 * M_PI);
        auto hd = [&](double hh, T& sig, T& dwk, T& inv_) {
            sig = (T)(sigd / pow(hh, D));
            dwk = (T)(-5.0 * sigd / pow(hh, D + 1));
            inv_ = (T)(1.0 / hh);
        };
        P.h = (T)h;
        hd(h, P.sig, P.dwk, P.inv_h);
        T dummy;
        P.h2 = (T)(0.5 * h);
        hd(0.5 * h, P.sig2, P.dwk2, P.inv_h2);
        P.ht = (T)(prm->h_tilde_factor * h);
        hd(prm->h_tilde_factor * h, dummy, P.dwkt, P.inv_ht);
        P.w0 = (T)(66.0 * sigd / pow(h, D));
        P.eta_h2 = (T)(prm->eta * h * h);
        P.rho0 = (T)prm->rho0;
        P.nu = (T)prm->nu;
        P.alpha = (T)prm->alpha;
        P.c_ref = (T)prm->c_ref;
        P.omega = (T)prm->omega;
        P.fs_ratio = (T)prm->fs_ratio;
        P.p_ref = (T)prm->p_ref;
        for (int a = 0; a < 3; a++) P.g[a] = (T)prm->g[a];
        P.pgrad = prm->pgrad;
        P.pref_external = prm->pref_external;
        P.ustar_noslip = prm->ustar_noslip;
        P.clamp_wall_p = prm->clamp_wall_p;
        P.wall_rho_summation = prm->wall_rho_summation;
        P.ghosts = dist() ? 1 : 0;
        rebuild_mode = prm->rebuild_mode;
        matrix_free = prm->matrix_free;
        if (const char* e = getenv("SISPH_SWEEP_CODES")) use_codes = atoi(e) != 0;
        if (const char* e = getenv("SISPH_PDL")) pdl = atoi(e) != 0;
        if (const char* e = getenv("SISPH_BUILD_MASK")) build_mask = atoi(e) != 0;
        if (const char* e = getenv("SISPH_GTVF_OVERLAP")) gtvf_overlap = atoi(e) != 0;
        ppe_loop = prm->ppe_loop;
        P.mean_free = prm->ppe_mean_free ? 1 : 0;
        pref_auto = prm->pref_auto;
        conv_mean = prm->conv_mean;
        nf_glob = 0;   // PPE unknowns: fluid (+ inlet, R34)
        for (int64_t k = 0; k < n; k++)
            nf_glob += (tags_glob[k] == SISPH_TAG_FLUID || tags_glob[k] == SISPH_TAG_INLET) ? 1 : 0;
        P.x_inlet = (T)prm->x_inlet;
        P.x_outlet = (T)prm->x_outlet;
        P.x_end = (T)prm->x_end;
        P.inlet_length = (T)prm->inlet_length;
        for (int a = 0; a < D; a++) extent = std::max(extent, std::max(fabs(dom->lo[a]), fabs(dom->hi[a])));
        min_iter = prm->min_iter;
        max_iter = prm->max_iter;
        tol = prm->tol;
        K = prm->K;
        // GTVF inner list: worth it when the GTVF kernel support 3 h~ is well inside 3 h
        {
#ifndef SISPH_GTVF_SKIN
#define SISPH_GTVF_SKIN 0.1   // B200, C5: 0.25 h -> 0.1 h: 107 -> 81 us per sub-step (fewer dead pairs)
#endif
            // the inner list's skin covers the K sub-steps' displacement (checked per step:
            // a particle moving more than skin / 2 sends the step back to the full list)
            const double ht = prm->h_tilde_factor * h, skin = SISPH_GTVF_SKIN * h;
            const double rin = 3.0 * ht + skin;
            use_inner = rin < 0.85 * R && prm->p_ref != 0.0 && prm->K > 0;
            P.Rin2f = (float)(rin * rin * (1.0 + 1.0 / 1024.0));
            P.skin_half2 = (T)(0.25 * skin * skin);
        }
        // slab ranks: the owned walls' halo lists are chosen on the host (same
        // arithmetic as k_halo_flags on the working-precision positions) so that
        // the ghost-wall count is known before the allocation
        std::vector<int> hws[2];
        if (dist() || open_x) {
            SCK(cudaHostAlloc((void**)&hcnt, 16 * sizeof(int), cudaHostAllocDefault));
            int rc = 0;
            dcnt = dalloc<int>(16, err, rc);
            if (rc) return rc;
        }
        if (dist()) {
            for (int w = 0; w < Nw; w++) {
                const double y = (double)(T)x[(size_t)wid[w] * D + axis];
                if (tp->nb[0] >= 0 && y < slab_lo + Gw) hws[0].push_back(w);
                if (tp->nb[1] >= 0 && y >= slab_hi - Gw) hws[1].push_back(w);
            }
            for (int f = 0; f < 2; f++) nws[f] = (int)hws[f].size();
            SRET(exchange_counts(nws, nwr));
            Nw = Nwo + nwr[0] + nwr[1];
        }
        Ntot = Nf + Nw;
        nf = Nfo;
        nw = Nwo;
        capF = dist() ? (int)(1.6 * Nfo) + 4096 : Nf;
        if (open_x) capF = Nf + (int)pool.size() + 64;   // R34: every dormant particle may enter
        capT = capF + Nw;
        SRET(sync_counts());
        // ------------------------------------------------ allocation
        int rc = 0;
        size_t NT = (size_t)std::max(capT, 1), NF = (size_t)std::max(capF, 1), NW = (size_t)std::max(Nw, 1);
        size_t NCT = 2 * (size_t)ncells + 2;   // cell tables: owned keys + ghost keys (+ end)
#define AL(ptr, Ty, cntx)                    \
    ptr = dalloc<Ty>((cntx), err, rc);       \
    if (rc) return rc;
        AL(pos, V, NT) AL(pos_alt, V, NT) AL(vel, V, NT) AL(vel_alt, V, NT) AL(us, V, NT) AL(us_alt, V, NT)
        AL(vt, V, NF) AL(vt_alt, V, NF) AL(rn, V, NT) AL(rstar, V, NT) AL(nrm, V, NW) AL(nstmp, V, NW) AL(uwl, V, NW)
        AL(gtA, V, 2 * NT) AL(gtB, V, 2 * NT) AL(fx0, V, NT) AL(dk, V, NT) AL(recF, V, 2 * NT) AL(recS, V, 2 * NT) AL(vk, V, NF) AL(fnp, V, NF) AL(dcnt_w, int, 4)
        AL(p, T, NT) AL(p_alt, T, NT) AL(rho, T, NT) AL(rho_alt, T, NT) AL(rhs, T, NF) AL(diag, T, NF)
        AL(fs, uint8_t, NF) AL(fs_alt, uint8_t, NF) AL(pid, int, NT) AL(pid_alt, int, NT)
        AL(keys, int, NT) AL(rank, int, NT) AL(perm0, int, NT) AL(perm, int, NT)
        AL(ccount, int, NCT) AL(fstart, int, NCT) AL(wstart, int, NCT)
        // scan block sums: cell tables (NCT) and the particle compactions (NT items)
        AL(bsum, int, (size_t)nblk(std::max(NCT, NT), SCAN_B) + 1) AL(cnt, int, NT) AL(ctl, Ctl, 1) AL(cnt_in, int, NF)
        AL(cnt_s, int, NT) AL(wperm_s, int, NW) AL(wstart_s, int, NCT)
        AL(partials, double, 2 * std::max((size_t)nblk(NF, RHS_T), (size_t)8192) + 2) AL(dtmp, double, 3 * (size_t)n)
        if (open_x) {
            AL(ptype, uint8_t, NF) AL(ptype_alt, uint8_t, NF) AL(uout, T, NF) AL(oflag, int, NF) AL(olist, int, NF)
            AL(onew, int, NF)
            if (!dist()) {
                AL(wtmp, V, NW)   // wall-block relocation staging (the slab path allocates it too)
                AL(wstage, char, (8 * sizeof(V) + 4 * sizeof(T) + 8) * NW)
            }
        }
        if (dist()) {
            AL(dflag, int, NT) AL(dflag2, int, NT) AL(dpre, int, NT + 1) AL(dlist[0], int, NF) AL(dlist[1], int, NF)
            AL(dlist[2], int, NF) AL(fsend[0], int, NF) AL(fsend[1], int, NF) AL(fsend_pre[0], int, NF)
            AL(fsend_pre[1], int, NF) AL(grecv, int, NF) AL(wsend[0], int, NW) AL(wsend[1], int, NW)
            AL(wrecv, int, NW) AL(inv, int, NT) AL(wtmp, V, NW)
            AL(wstage, char, (8 * sizeof(V) + 4 * sizeof(T) + 8) * NW)
            AL(bflag, int, NF) AL(brow, int, NF) AL(irow, int, NF) AL(gcnt, int, 2)
        }
#undef AL
        SCK(cudaHostAlloc((void**)&hctl, sizeof(Ctl), cudaHostAllocDefault));
        SCK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
        SCK(cudaMemsetAsync(fs, 0, NF, st));
        SCK(cudaMemsetAsync(vt, 0, NF * sizeof(V), st));
        SCK(cudaMemsetAsync(p, 0, NT * sizeof(T), st));
        SCK(cudaMemsetAsync(p_alt, 0, NT * sizeof(T), st));
        SCK(cudaMemsetAsync(us, 0, NT * sizeof(V), st));
        SCK(cudaMemsetAsync(us_alt, 0, NT * sizeof(V), st));
        SCK(cudaMemsetAsync(nrm, 0, NW * sizeof(V), st));
        SCK(cudaMemsetAsync(uwl, 0, NW * sizeof(V), st));
        SCK(cudaMemsetAsync(rhs, 0, NF * sizeof(T), st));
        SCK(cudaMemsetAsync(diag, 0, NF * sizeof(T), st));
        // ------------------------------------------------ upload (fluid, then owned walls, given order)
        std::vector<V> hpos(NT), hvel(NT);
        std::vector<T> hrho(NT);
        std::vector<int> hid(NT);
        const int nup = Nf + Nwo;
        for (int s = 0; s < nup; s++) {
            int k = s < Nf ? fid[s] : wid[s - Nf];
            hid[s] = gid ? (int)gid[k] : k;
            const double* xk = x + (size_t)k * D;
            const double* uk = u + (size_t)k * D;
            hpos[s] = mkh(xk[0], xk[1], D == 3 ? xk[2] : 0.0, m[k]);
            hvel[s] = mkh(uk[0], uk[1], D == 3 ? uk[2] : 0.0, 0.0);
            hrho[s] = (T)r0[k];
        }
        SCK(cudaMemcpyAsync(pos, hpos.data(), nup * sizeof(V), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(vel, hvel.data(), nup * sizeof(V), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(vt, hvel.data(), (size_t)Nf * sizeof(V), cudaMemcpyHostToDevice, st));  // R23
        SCK(cudaMemcpyAsync(rho, hrho.data(), nup * sizeof(T), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(pid, hid.data(), nup * sizeof(int), cudaMemcpyHostToDevice, st));
        std::vector<uint8_t> hty;
        if (open_x) {
            // R34: particle types of the fluid block (0 fluid, 2 inlet, 3 outlet)
            hty.resize(std::max(Nf, 1));
            for (int s = 0; s < Nf; s++) hty[s] = (uint8_t)tags[fid[s]];
            SCK(cudaMemcpyAsync(ptype, hty.data(), Nf, cudaMemcpyHostToDevice, st));
            P.ptype = ptype;
        }
        if (dist())
            for (int f = 0; f < 2; f++)
                if (nws[f]) SCK(cudaMemcpyAsync(wsend[f], hws[f].data(), nws[f] * sizeof(int), cudaMemcpyHostToDevice, st));
        SCK(cudaStreamSynchronize(st));  // host vectors go out of scope
        // ------------------------------------------------ walls, first build, normals, capacity
        int cap = prm->nbr_cap;
        if (cap <= 0) cap = D == 2 ? 48 : 160;
        cap = (cap + 3) / 4 * 4;   // blocked ELL stores 16-byte chunks of 4 entries
        SRET(alloc_list(cap));
        SRET(sort_walls(true));
        SRET(first_build());
        if (prm->nbr_cap <= 0) {
            // automatic capacity: 1.5 x the largest count of the first build (slab ranks: of all ranks)
            SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
            int mc = hctl->max_count;
            if (dist()) SRET(allreduce_host(&mc, 1));
            int want = std::max((int)ceil(1.5 * mc) + 8, D == 2 ? 48 : 128);
            want = (want + 7) / 8 * 8;
            if (want != P.cap) {
                SRET(alloc_list(want));
                SRET(first_build());
            }
        }
        return check_overflow();
    }

    static V mkh(double a, double b, double c, double d)
    {
        V v;
        v.x = (T)a;
        v.y = (T)b;
        v.z = (T)c;
        v.w = (T)d;
        return v;
    }

    static size_t rows32(int n_) { return ((size_t)std::max(n_, 1) + 31) / 32 * 32; }

    int sync_counts()
    {
        P.Nf = Nf;
        P.Nw = Nw;
        P.Ntot = Ntot;
        P.Nfo = Nfo;
        P.Nwo = Nwo;
        PS.Nf = Nf;
        PS.Nw = Nw;
        PS.Ntot = Ntot;
        PS.Nfo = Nfo;
        PS.Nwo = Nwo;
        return SISPH_OK;
    }

    int alloc_list(int cap)
    {
        if (nbr) cudaFree(nbr);
        if (nbr_in) cudaFree(nbr_in);
        if (coef) cudaFree(coef);
        if (code) cudaFree(code);
        if (nslot) cudaFree(nslot);
        nbr = nbr_in = nullptr;
        coef = nullptr;
        code = nullptr;
        nslot = nullptr;
        int rc = 0;
        nbr = dalloc<int>((size_t)cap * rows32(capT), err, rc);
        if (rc) return rc;
        if (!matrix_free) {
            // code mode: a long step takes two slots, so a row needs at most 2 cap slots
            cc8 = use_codes ? (2 * cap + 7) / 8 : 0;
            coef = dalloc<T>((size_t)(use_codes ? 8 * cc8 : cap) * rows32(capF), err, rc);
            if (rc) return rc;
            if (use_codes) {
                code = dalloc<uint4>((size_t)cc8 * rows32(capF), err, rc);
                if (rc) return rc;
                nslot = dalloc<int>(rows32(capF), err, rc);
                if (rc) return rc;
            }
        }
        P.cap = cap;
        if (use_inner) {
            // the inner list holds a subset of each fluid row: the full capacity is an upper bound
            P.cap_in = cap;
            nbr_in = dalloc<int>((size_t)cap * rows32(capF), err, rc);
            if (rc) return rc;
        }
        return SISPH_OK;
    }

    int check_overflow()
    {
        SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        if (hctl->overflow) {
            err = "neighbour list capacity exceeded: a particle has " + std::to_string(hctl->max_count) +
                  " neighbours, capacity " + std::to_string(P.cap);
            return SISPH_EOVERFLOW;
        }
        return SISPH_OK;
    }

    // exclusive scan of ccount[0..nc] into out[0..nc]
    int scan(const int* in, int* out, int nitems)
    {
        int nb = nblk(nitems, SCAN_B);
        ++nlaunch, k_scan_local<<<nb, SCAN_T, 0, st>>>(in, out, nitems, bsum);
        ++nlaunch, k_scan_sums<<<1, 1024, 0, st>>>(bsum, nb);
        ++nlaunch, k_scan_add<<<nb, SCAN_T, 0, st>>>(out, nitems, bsum);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    static int ncells_of(const Params<T>& G) { return G.nc[0] * G.nc[1] * G.nc[2]; }

    // A1 + A2 + A4: stable counting sort of n particles at xs by cell key
    // (elements at i >= nown are ghosts: key + ncells); writes
    // start[0 .. 2 ncells] (ghosts present) and perm_out[0..n) (relative slots)
    int sort_set(const Params<T>& G, const V* xs, int nn, int nown, int* start, int* perm_out)
    {
        const int nk = ncells_of(G) * (G.ghosts ? 2 : 1);
        SCK(cudaMemsetAsync(ccount, 0, ((size_t)nk + 1) * sizeof(int), st));
        if (nn > 0) {
            ++nlaunch, k_hash_count<T, D><<<nblk(nn, 256), 256, 0, st>>>(G, xs, nn, nown, keys, rank, ccount);
            SCK(cudaGetLastError());
        }
        SRET(scan(ccount, start, nk + 1));
        if (nn > 0) {
            ++nlaunch, k_scatter<<<nblk(nn, 256), 256, 0, st>>>(keys, rank, start, perm0, nn);
            ++nlaunch, k_stabilize<<<nblk(nn, 256), 256, 0, st>>>(perm0, keys, start, perm_out, nn);
            SCK(cudaGetLastError());
        }
        return SISPH_OK;
    }

    int gather(GatherList& G, const int* pm, int nn)
    {
        if (nn <= 0 || G.nf == 0) return SISPH_OK;
        ++nlaunch, k_gather<<<nblk(nn, 256), 256, 0, st>>>(G, pm, nn);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }
    static void gl_add(GatherList& G, const void* s, void* d, int size, int cnt_)
    {
        G.src[G.nf] = s;
        G.dst[G.nf] = d;
        G.size[G.nf] = size;
        G.n[G.nf] = cnt_;
        G.nf++;
    }

    int build_list(bool inner = false)
    {
        SCK(cudaMemsetAsync(&ctl->max_count, 0, 2 * sizeof(int) + 2 * sizeof(unsigned long long), st));
        int* ni = inner && nbr_in ? nbr_in : nullptr;
        ++nlaunch, k_build_cells<T, D><<<nblk(ncells, BL_WARPS), 32 * BL_WARPS, 0, st>>>(
            P, ncells, pos, fstart, wstart, nullptr, nbr, cnt, ni, cnt_in, ctl);
        SCK(cudaGetLastError());
        inner_valid = ni != nullptr;
        return SISPH_OK;
    }

    // loose list at the current positions on the skin geometry PS (R3)
    int build_loose()
    {
        SCK(cudaMemsetAsync(&ctl->max_count_s, 0, 2 * sizeof(int), st));
        const int nc = ncells_of(PS);
        bool done = false;
        if constexpr (D == 3) {
            if (build_mask) {
                ++nlaunch, k_build_loose_m<T, D><<<nblk(nc, BM_WARPS), 32 * BM_WARPS, 0, st>>>(
                    PS, nc, pos, fstart, wstart_s, Nw ? wperm_s : nullptr, nbs, cnt_s, ctl);
                done = true;
            }
        }
        if (!done)
            ++nlaunch, k_build_loose<T, D><<<nblk(nc, BL_WARPS), 32 * BL_WARPS, 0, st>>>(
                PS, nc, pos, fstart, wstart_s, Nw ? wperm_s : nullptr, nbs, cnt_s, ctl);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    // r* of the fluid slots (eq:int:rnp1); slab ranks: the ghosts' from their owners
    int compute_rstar(double dt)
    {
        if (Nfo) ++nlaunch, k_rstar<T, D><<<nblk(Nfo, 256), 256, 0, st>>>(P, (T)dt, Nfo, pos, vt, rstar);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList L{};
            pl_add(L, rstar, sizeof(V), 1);
            SRET(halo_fluid(L));
        }
        return SISPH_OK;
    }

    // exact sets at r* out of the loose list (+ GTVF inner list)
    int filter_list()
    {
        // the loose build keeps its own count / overflow (max_count_s, overflow_s)
        SCK(cudaMemsetAsync(&ctl->max_count, 0, 2 * sizeof(int), st));
        SCK(cudaMemsetAsync(&ctl->pairs_fluid, 0, 2 * sizeof(unsigned long long), st));
        int* ni = nbr_in;
        const int rows = Nfo + Nwo;
        if (rows)
            ++nlaunch, (ni ? k_filter<T, D, true> : k_filter<T, D, false>)<<<nblk(rows, 128), 128, 0, st>>>(
                           P, rows, rstar, nbs, cnt_s, cap_s, nbr, cnt, ni, cnt_in, ctl);
        SCK(cudaGetLastError());
        inner_valid = ni != nullptr;
        return SISPH_OK;
    }

    // Decide whether this step can use the single build: skin s = 2 dt max|u~|
    // (+ a rounding margin); the skin geometry has cells >= 3h + s, at least 3
    // per periodic axis, and 3h + s <= 1.3 * 3h (list capacity; slab ranks:
    // the halo width).  Slab ranks take the max over all ranks' owned fluid
    // (ghosts are not present yet).  Sets PS.
    int plan_skin(double dt, bool& ok)
    {
        ok = false;
        skin_used = false;
        skin_radius = 0;
        if (rebuild_mode != 0 || (Nf == 0 && !dist())) return SISPH_OK;
        SCK(cudaMemsetAsync(&ctl->umax2_bits, 0, sizeof(unsigned long long), st));
        const int nmax = dist() ? Nfo : Nf;
        if (nmax) ++nlaunch, k_max_speed<T, D><<<std::min(nblk(nmax, 256), 148 * 8), 256, 0, st>>>(vt, nmax, ctl);
        SCK(cudaGetLastError());
        if (dist()) SRET(xallreduce(reinterpret_cast<double*>(&ctl->umax2_bits), 1, 1));
        SCK(cudaMemcpyAsync(&hctl->umax2_bits, &ctl->umax2_bits, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            st));
        SCK(cudaStreamSynchronize(st));
        double um2;
        unsigned long long b = hctl->umax2_bits;
        memcpy(&um2, &b, sizeof(double));
        if (!std::isfinite(um2)) return SISPH_OK;
        const double R = 3.0 * (double)P.h;
        const double eps = std::is_same<T, float>::value ? 1e-6 : 1e-14;
        const double Rs = R + 2.0 * dt * sqrt(um2) * (1.0 + 1e-6) + eps * (extent + R) + 1e-9 * R;
        if (Rs > 1.3 * R) return SISPH_OK;
        Params<T> G = P;
        for (int a = 0; a < D; a++) {
            int nc = (int)floor(P.Ld[a] / (Rs * (1.0 + 1.0 / (1 << 20))));
            if (nc < 1) nc = 1;
            if (P.per[a] && nc < 3) return SISPH_OK;
            if (nc > P.nc[a]) nc = P.nc[a];
            G.nc[a] = nc;
            G.cell[a] = P.Ld[a] / nc;
        }
        G.Rs2 = (T)(Rs * Rs * (1.0 + 1.0 / 1024.0));
        // loose-list capacity: the exact capacity scaled by the volume ratio
        int want = (int)ceil(P.cap * pow(Rs / R, D)) + 8;
        want = (want + 7) / 8 * 8;
        if (want > cap_s) {
            if (nbs) cudaFree(nbs);
            nbs = nullptr;
            int rc = 0;
            nbs = dalloc<int>((size_t)want * rows32(capT), err, rc);
            if (rc) return rc;
            cap_s = want;
        }
        G.cap = cap_s;
        PS = G;
        ok = true;
        skin_used = true;
        skin_radius = Rs;
        return SISPH_OK;
    }

    // walls binned on the skin grid (static: only when the grid changes)
    int bin_walls_skin()
    {
        const Params<T>& G = PS;
        if (Nw && (G.nc[0] != wnc_s[0] || G.nc[1] != wnc_s[1] || G.nc[2] != wnc_s[2])) {
            SRET(sort_set(G, pos + Nf, Nw, Nwo, wstart_s, wperm_s));
            for (int a = 0; a < 3; a++) wnc_s[a] = G.nc[a];
        } else if (!Nw) {
            SCK(cudaMemsetAsync(wstart_s, 0, (2 * (size_t)ncells_of(G) + 2) * sizeof(int), st));
        }
        return SISPH_OK;
    }

    // ------------------------------------------------------------------ slab-rank plumbing
    int tperr()
    {
        err = "transport: " + tp->err;
        return SISPH_ENCCL;
    }
    int xallreduce(double* dbuf, int count, int op)
    {
        if (tp->allreduce(dbuf, count, op, st)) return tperr();
        return SISPH_OK;
    }
    // host ints -> max over ranks (through the device)
    int allreduce_host(int* v, int count)
    {
        std::vector<double> h(count);
        for (int q = 0; q < count; q++) h[q] = v[q];
        double* d = partials;   // scratch (>= 2 doubles)
        SCK(cudaMemcpyAsync(d, h.data(), count * sizeof(double), cudaMemcpyHostToDevice, st));
        SRET(xallreduce(d, count, 1));
        SCK(cudaMemcpyAsync(h.data(), d, count * sizeof(double), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        for (int q = 0; q < count; q++) v[q] = (int)h[q];
        return SISPH_OK;
    }
    // send s[f] to the face-f neighbour, receive r[f] from it (host ints)
    int exchange_counts(const int s[2], int r[2])
    {
        hcnt[0] = s[0];
        hcnt[1] = s[1];
        hcnt[2] = hcnt[3] = 0;
        SCK(cudaMemcpyAsync(dcnt, hcnt, 4 * sizeof(int), cudaMemcpyHostToDevice, st));
        const void* sb[2] = {dcnt, dcnt + 1};
        void* rb[2] = {dcnt + 2, dcnt + 3};
        const size_t sz[2] = {sizeof(int), sizeof(int)};
        if (tp->sendrecv(sb, sz, rb, sz, st)) return tperr();
        SCK(cudaMemcpyAsync(hcnt, dcnt, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        r[0] = tp->nb[0] >= 0 ? hcnt[2] : 0;
        r[1] = tp->nb[1] >= 0 ? hcnt[3] : 0;
        return SISPH_OK;
    }
    int ensure_buf(int f, size_t bytes)
    {
        if (bytes <= bufcap[f]) return SISPH_OK;
        size_t want = bytes + bytes / 4 + 4096;
        if (sbuf[f]) cudaFree(sbuf[f]);
        if (rbuf[f]) cudaFree(rbuf[f]);
        sbuf[f] = rbuf[f] = nullptr;
        int rc = 0;
        sbuf[f] = dalloc<char>(want, err, rc);
        if (rc) return rc;
        rbuf[f] = dalloc<char>(want, err, rc);
        if (rc) return rc;
        bufcap[f] = want;
        return SISPH_OK;
    }
    static void pl_add(PackList& L, void* ptr, int size, int shift = 0)
    {
        L.ptr[L.nf] = ptr;
        L.size[L.nf] = size;
        L.sh[L.nf] = shift;
        L.nf++;
        L.rec += size;
    }
    // periodic image shift of records crossing face f of this rank
    double face_shift(int f) const
    {
        if (!gper) return 0.0;
        if (f == 0 && tp->rank == 0) return ghi - glo;                  // to the last slab, above its top
        if (f == 1 && tp->rank == tp->nranks - 1) return -(ghi - glo);  // to the first slab, below its bottom
        return 0.0;
    }
    // One face exchange: pack list[f] (count ns[f]; NULL list = slots base +
    // q) of the fields of L, send, unpack the received records (counts nr[f])
    // to map (NULL: base_r + q), face-0 records first.  L.ptr are the arrays
    // (for pack and unpack alike: a halo refresh writes the same arrays).
    int exchange(PackList L, int* const list[2], const int ns[2], const int nr[2], const int* map, int base_r)
    {
        L.rec = (L.rec + 15) / 16 * 16;
        L.axis = axis;
        for (int f = 0; f < 2; f++) {
            SRET(ensure_buf(f, (size_t)std::max(ns[f], nr[f]) * L.rec));
        }
        if (list[0] && list[1] && ns[0] + ns[1] > 0) {
            ++nlaunch, k_pack2<T><<<nblk(ns[0] + ns[1], 256), 256, 0, st>>>(
                           L, face_shift(0), face_shift(1), list[0], list[1], ns[0], ns[1], sbuf[0], sbuf[1]);
            halo_bytes += (int64_t)(ns[0] + ns[1]) * L.rec;
        } else {
            for (int f = 0; f < 2; f++) {
                if (!ns[f]) continue;
                PackList Lf = L;
                Lf.shift = face_shift(f);
                ++nlaunch, k_pack<T><<<nblk(ns[f], 256), 256, 0, st>>>(Lf, list[f], 0, ns[f], sbuf[f]);
                halo_bytes += (int64_t)ns[f] * L.rec;
            }
        }
        SCK(cudaGetLastError());
        const void* sb[2] = {sbuf[0], sbuf[1]};
        void* rb[2] = {rbuf[0], rbuf[1]};
        const size_t sz[2] = {(size_t)ns[0] * L.rec, (size_t)ns[1] * L.rec};
        const size_t rz[2] = {(size_t)nr[0] * L.rec, (size_t)nr[1] * L.rec};
        if (tp->sendrecv(sb, sz, rb, rz, st)) return tperr();
        if (nr[0] + nr[1] > 0)
            ++nlaunch, k_unpack2<T><<<nblk(nr[0] + nr[1], 256), 256, 0, st>>>(L, map, base_r, nr[0], nr[1], rbuf[0],
                                                                               rbuf[1]);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }
    // halo refresh of fluid fields (owned rows -> the neighbours' ghost rows)
    int halo_fluid(PackList L) { return exchange(L, fsend, nfs, nfr, grecv, 0); }
    // halo refresh of wall fields; L.ptr point at the wall blocks (relative slots)
    int halo_walls(PackList L) { return exchange(L, wsend, nws, nwr, wrecv, 0); }
    // the p^k buffer of a solve is chosen on the device (iteration parity):
    // refresh both, the copy of the unused one is harmless
    int halo_p(bool walls)
    {
        PackList L{};
        pl_add(L, walls ? (void*)(p + Nf) : (void*)p, sizeof(T));
        pl_add(L, walls ? (void*)(p_alt + Nf) : (void*)p_alt, sizeof(T));
        return walls ? halo_walls(L) : halo_fluid(L);
    }

    // stable compaction of flag == v (or flag != 0 with v < 0) over n items
    // into out; the count reaches the host
    int compact(const int* flag, int nn, int v, int* out, int& count)
    {
        count = 0;
        if (nn <= 0) return SISPH_OK;
        const int* f01 = flag;
        if (v >= 0) {
            ++nlaunch, k_flag_eq<<<nblk(nn, 256), 256, 0, st>>>(flag, nn, v, dflag2);
            f01 = dflag2;
        }
        SRET(scan(f01, dpre, nn));
        ++nlaunch, k_compact<<<nblk(nn, 256), 256, 0, st>>>(f01, dpre, nn, out, dcnt + 4);
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(hcnt + 4, dcnt + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        count = hcnt[4];
        return SISPH_OK;
    }

    // stable compaction without a host wait: the count goes to dcnt[slot]
    // (slots 8..15; read by counts_sync)
    int compact_async(const int* flag, int nn, int v, int* out, int slot)
    {
        if (nn <= 0) {
            SCK(cudaMemsetAsync(dcnt + slot, 0, sizeof(int), st));
            return SISPH_OK;
        }
        const int* f01 = flag;
        if (v >= 0) {
            ++nlaunch, k_flag_eq<<<nblk(nn, 256), 256, 0, st>>>(flag, nn, v, dflag2);
            f01 = dflag2;
        }
        SRET(scan(f01, dpre, nn));
        ++nlaunch, k_compact<<<nblk(nn, 256), 256, 0, st>>>(f01, dpre, nn, out, dcnt + slot);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }
    // send the counts in dcnt[s0] / dcnt[s1] to the face-0 / face-1 neighbours, receive
    // theirs into dcnt[r0] / dcnt[r1] (0 without a neighbour), then ONE host wait for all
    // of dcnt[8..15]
    int counts_sync(int s0, int s1, int r0, int r1)
    {
        SCK(cudaMemsetAsync(dcnt + r0, 0, sizeof(int), st));
        SCK(cudaMemsetAsync(dcnt + r1, 0, sizeof(int), st));
        const void* sb[2] = {dcnt + s0, dcnt + s1};
        void* rb[2] = {dcnt + r0, dcnt + r1};
        const size_t sz[2] = {sizeof(int), sizeof(int)};
        if (tp->sendrecv(sb, sz, rb, sz, st)) return tperr();
        SCK(cudaMemcpyAsync(hcnt + 8, dcnt + 8, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        if (tp->nb[0] < 0) hcnt[r0] = 0;
        if (tp->nb[1] < 0) hcnt[r1] = 0;
        return SISPH_OK;
    }

    // move the wall block of every wall-carrying array from [Nf, ...) to [newNf, ...)
    int relocate_walls(int newNf)
    {
        if (newNf + Nw > capT) {
            err = "slab rank: fluid slot capacity exceeded (" + std::to_string(newNf) + " fluid + halo slots)";
            return SISPH_ENOMEM;
        }
        if (newNf == Nf) return SISPH_OK;
        if (Nw == 0) {
            Nf = newNf;
            Ntot = Nf;
            return sync_counts();
        }
        // every wall-carrying array in two launches (staged: the old and new blocks may overlap)
        MoveList M{};
        size_t off = 0;
        auto add = [&](void* base, int esz) {
            M.ptr[M.n] = (char*)base;
            M.esz[M.n] = esz;
            M.toff[M.n] = off;
            off += (size_t)Nw * esz;
            M.n++;
        };
        void* vecs[] = {pos, pos_alt, rn, rstar, vel, vel_alt, us, us_alt};
        for (void* q : vecs) add(q, sizeof(V));
        void* scs[] = {p, p_alt, rho, rho_alt};
        for (void* q : scs) add(q, sizeof(T));
        add(pid, sizeof(int));
        add(pid_alt, sizeof(int));
        const dim3 g((unsigned)std::min(nblk((long)Nw * sizeof(V) / 4, 256), 148 * 8), (unsigned)M.n);
        ++nlaunch, k_move_block<<<g, 256, 0, st>>>(M, Nf, Nw, wstage, 1);
        ++nlaunch, k_move_block<<<g, 256, 0, st>>>(M, newNf, Nw, wstage, 0);
        SCK(cudaGetLastError());
        Nf = newNf;
        Ntot = Nf + Nw;
        return sync_counts();
    }

    // Slab ranks, step start: owned fluid particles that left the slab move
    // to the neighbour rank (whole carried state: r, m, u, u~, p, id).
    int migrate()
    {
        const int has[2] = {tp->nb[0] >= 0, tp->nb[1] >= 0};
        // the classification counts the leavers per face; the counts are exchanged and read
        // with one host wait; the stable compactions run only when someone moves
        SCK(cudaMemsetAsync(dcnt + 9, 0, 2 * sizeof(int), st));
        if (Nfo) ++nlaunch, k_classify<T><<<nblk(Nfo, 256), 256, 0, st>>>(pos, Nfo, axis, slab_lo, slab_hi, glo, ghi, gper,
                                                                          has[0], has[1], dflag, dcnt + 9);
        SCK(cudaGetLastError());
        SRET(counts_sync(9, 10, 11, 12));
        const int nout[2] = {hcnt[9], hcnt[10]}, nin[2] = {hcnt[11], hcnt[12]};
        const int nstay = Nfo - nout[0] - nout[1];
        // nobody leaves or arrives: the stayers are the owned block in its order, and the
        // ghosts of the previous step are dropped by the caller's relocation
        if (nout[0] + nout[1] + nin[0] + nin[1] == 0) return sync_counts();
        SRET(compact_async(dflag, Nfo, 0, dlist[0], 13));
        SRET(compact_async(dflag, Nfo, 1, dlist[1], 14));
        SRET(compact_async(dflag, Nfo, 2, dlist[2], 15));
        const int nnew = nstay + nin[0] + nin[1];
        // ghosts of the previous step are dropped: the fluid block is owned only
        if (nnew + Nw > capT) {
            err = "slab rank: fluid slot capacity exceeded by migration";
            return SISPH_ENOMEM;
        }
        // stayers -> alternates [0, nstay)
        GatherList G{};
        gl_add(G, pos, pos_alt, sizeof(V), nstay);
        gl_add(G, vel, vel_alt, sizeof(V), nstay);
        gl_add(G, vt, vt_alt, sizeof(V), nstay);
        gl_add(G, p, p_alt, sizeof(T), nstay);
        gl_add(G, pid, pid_alt, sizeof(int), nstay);
        SRET(gather(G, dlist[0], nstay));
        // migrants: pack from the current arrays, unpack behind the stayers
        PackList L{};
        pl_add(L, pos, sizeof(V));
        pl_add(L, vel, sizeof(V));
        pl_add(L, vt, sizeof(V));
        pl_add(L, p, sizeof(T));
        pl_add(L, pid, sizeof(int));
        L.rec = (L.rec + 15) / 16 * 16;
        L.axis = axis;
        for (int f = 0; f < 2; f++) SRET(ensure_buf(f, (size_t)std::max(nout[f], nin[f]) * L.rec));
        int* lists[2] = {dlist[1], dlist[2]};
        for (int f = 0; f < 2; f++)
            if (nout[f]) {
                ++nlaunch, k_pack<T><<<nblk(nout[f], 256), 256, 0, st>>>(L, lists[f], 0, nout[f], sbuf[f]);
                halo_bytes += (int64_t)nout[f] * L.rec;
            }
        SCK(cudaGetLastError());
        {
            const void* sb[2] = {sbuf[0], sbuf[1]};
            void* rb[2] = {rbuf[0], rbuf[1]};
            const size_t sz[2] = {(size_t)nout[0] * L.rec, (size_t)nout[1] * L.rec};
            const size_t rz[2] = {(size_t)nin[0] * L.rec, (size_t)nin[1] * L.rec};
            if (tp->sendrecv(sb, sz, rb, rz, st)) return tperr();
        }
        PackList U{};
        pl_add(U, pos_alt, sizeof(V));
        pl_add(U, vel_alt, sizeof(V));
        pl_add(U, vt_alt, sizeof(V));
        pl_add(U, p_alt, sizeof(T));
        pl_add(U, pid_alt, sizeof(int));
        U.rec = L.rec;
        int off = nstay;
        for (int f = 0; f < 2; f++) {
            if (nin[f]) ++nlaunch, k_unpack<T><<<nblk(nin[f], 256), 256, 0, st>>>(U, nullptr, off, nin[f], rbuf[f]);
            off += nin[f];
        }
        SCK(cudaGetLastError());
        SRET(copy_walls_to_alt());
        std::swap(pos, pos_alt);
        std::swap(vel, vel_alt);
        std::swap(vt, vt_alt);
        std::swap(p, p_alt);
        std::swap(pid, pid_alt);
        // the alternates' wall blocks are at Nf: the position buffers keep theirs
        SRET(copy_pos_walls(pos_alt, pos));
        Nfo = nnew;
        // the fluid block is now [0, Nfo): walls move down to Nfo
        SRET(relocate_walls(Nfo));
        return sync_counts();
    }
    // R34 conversions after the position update.  The device
    // classifies each fluid-block row on its pre-step type; the host does the
    // id bookkeeping in the oracle's order (deletions return ids to the pool,
    // spawning rows draw the lowest dormant ids in ascending id order of the
    // rows that left the inlet); the device compacts the kept rows and appends
    // the new inlet rows behind them; the walls move to the new block end.
    int open_boundaries()
    {
        open_spawned = open_deleted = 0;
        if (Nfo == 0) return SISPH_OK;
        ++nlaunch, k_open_classify<T><<<nblk(Nfo, 256), 256, 0, st>>>(P, pos, ptype, oflag);
        SCK(cudaGetLastError());
        std::vector<int> hf(Nfo), hp(Nfo);
        std::vector<uint8_t> ht(Nfo);
        SCK(cudaMemcpyAsync(hf.data(), oflag, Nfo * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(hp.data(), pid, Nfo * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(ht.data(), ptype, Nfo, cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        std::vector<int> keep, src;
        keep.reserve(Nfo);
        for (int s = 0; s < Nfo; s++) {
            if (hf[s] == 1) {
                pool.insert(hp[s]);          // outlet -> dormant: the id returns to the pool
                open_deleted++;
            } else {
                keep.push_back(s);
                if (hf[s] == 2) src.push_back(s);
            }
        }
        std::sort(src.begin(), src.end(), [&](int a, int b) { return hp[a] < hp[b]; });
        std::vector<int> nid(src.size());
        for (size_t q = 0; q < src.size(); q++) {
            if (pool.empty()) {
                err = "open boundaries: the dormant pool is exhausted (add particles with tag SISPH_TAG_DORMANT)";
                return SISPH_ENOMEM;
            }
            nid[q] = *pool.begin();
            pool.erase(pool.begin());
        }
        open_spawned = (int)src.size();
        const int nkeep = (int)keep.size(), nsp = (int)src.size(), nnew = nkeep + nsp;
        if (nnew + Nw > capT) {
            err = "open boundaries: fluid slot capacity exceeded";
            return SISPH_ENOMEM;
        }
        // a growing block first moves the walls up, so that the new rows never overlap them
        const int nf_old = Nf;
        if (nnew > nf_old) SRET(relocate_walls(nnew));
        if (nkeep) SCK(cudaMemcpyAsync(perm, keep.data(), nkeep * sizeof(int), cudaMemcpyHostToDevice, st));
        if (nsp) {
            SCK(cudaMemcpyAsync(olist, src.data(), nsp * sizeof(int), cudaMemcpyHostToDevice, st));
            SCK(cudaMemcpyAsync(onew, nid.data(), nsp * sizeof(int), cudaMemcpyHostToDevice, st));
        }
        GatherList G{};
        gl_add(G, pos, pos_alt, sizeof(V), nkeep);
        gl_add(G, vel, vel_alt, sizeof(V), nkeep);
        gl_add(G, vt, vt_alt, sizeof(V), nkeep);
        gl_add(G, p, p_alt, sizeof(T), nkeep);
        gl_add(G, pid, pid_alt, sizeof(int), nkeep);
        gl_add(G, rho, rho_alt, sizeof(T), nkeep);
        gl_add(G, ptype, ptype_alt, 1, nkeep);
        SRET(gather(G, perm, nkeep));
        if (nsp)
            ++nlaunch, k_open_spawn<T><<<nblk(nsp, 256), 256, 0, st>>>(P, nkeep, nsp, olist, onew, pos, vel, p, rho,
                                                                         pos_alt, vel_alt, vt_alt, p_alt, rho_alt,
                                                                         pid_alt, ptype_alt);
        SCK(cudaGetLastError());
        SRET(copy_walls_to_alt());
        std::swap(pos, pos_alt);
        std::swap(vel, vel_alt);
        std::swap(vt, vt_alt);
        std::swap(p, p_alt);
        std::swap(pid, pid_alt);
        std::swap(rho, rho_alt);
        std::swap(ptype, ptype_alt);
        P.ptype = PS.ptype = ptype;
        SRET(copy_pos_walls(pos_alt, pos));
        // host view of the types (TAG field) and the PPE unknown count (R12b means)
        for (int64_t k = 0; k < n; k++)
            if (tags_host[k] != SISPH_TAG_WALL) tags_host[k] = SISPH_TAG_DORMANT;
        int64_t unk = 0;
        for (int q = 0; q < nkeep; q++) {
            const int t = ht[keep[q]];
            tags_host[hp[keep[q]]] = t;
            unk += (t == 0 || t == 2);
        }
        for (int q = 0; q < nsp; q++) tags_host[nid[q]] = SISPH_TAG_INLET;
        nf_glob = unk + nsp;
        Nfo = nnew;
        if (nnew < nf_old) SRET(relocate_walls(nnew));   // a shrinking block: walls move down after
        return sync_counts();
    }

    int copy_pos_walls(V* dst, const V* src)
    {
        if (Nw) SCK(cudaMemcpyAsync(dst + Nf, src + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
        return SISPH_OK;
    }

    // Slab ranks: halo selection on the owned fluid, exchange of the ghost
    // records (r with the periodic image shift, m, u, u~, p, rho, id) into
    // [Nfo, Nf).  The lists refer to pre-sort slots (remapped after the sort).
    int fetch_ghosts()
    {
        const int has[2] = {tp->nb[0] >= 0, tp->nb[1] >= 0};
        if (Nfo) ++nlaunch, k_halo_flags<T><<<nblk(Nfo, 256), 256, 0, st>>>(pos, Nfo, axis, slab_lo, slab_hi, Gw, has[0],
                                                                            has[1], dflag, dflag2);
        SCK(cudaGetLastError());
        SRET(compact_async(dflag, Nfo, -1, fsend_pre[0], 8));
        SRET(compact_async(dflag2, Nfo, -1, fsend_pre[1], 9));
        SRET(counts_sync(8, 9, 10, 11));
        nfs[0] = hcnt[8];
        nfs[1] = hcnt[9];
        nfr[0] = hcnt[10];
        nfr[1] = hcnt[11];
        const int ng = nfr[0] + nfr[1];
        SRET(relocate_walls(Nfo + ng));
        PackList L{};
        pl_add(L, pos, sizeof(V), 1);
        pl_add(L, vel, sizeof(V));
        pl_add(L, vt, sizeof(V));
        pl_add(L, p, sizeof(T));
        pl_add(L, rho, sizeof(T));
        pl_add(L, pid, sizeof(int));
        return exchange(L, fsend_pre, nfs, nfr, nullptr, Nfo);
    }

    // walls (create): sort owned + ghost walls by cell; slab ranks first fetch
    // the ghost walls (static) from the neighbours and keep the halo maps
    int sort_walls(bool fetch)
    {
        if (dist() && fetch) {
            // ghost walls appended behind the owned ones (relative slots Nwo + q)
            PackList L{};
            pl_add(L, pos + Nf, sizeof(V), 1);
            pl_add(L, vel + Nf, sizeof(V));
            pl_add(L, rho + Nf, sizeof(T));
            pl_add(L, pid + Nf, sizeof(int));
            SRET(exchange(L, wsend, nws, nwr, nullptr, Nwo));
        }
        if (Nw > 0) {
            // relative wall slots go to rank[] (free after the sort): gather through it
            int* wp = rank + Nf;
            SRET(sort_set(P, pos + Nf, Nw, Nwo, wstart, wp));
            GatherList G{};
            gl_add(G, pos + Nf, pos_alt + Nf, sizeof(V), Nw);
            gl_add(G, vel + Nf, vel_alt + Nf, sizeof(V), Nw);
            gl_add(G, rho + Nf, rho_alt + Nf, sizeof(T), Nw);
            gl_add(G, pid + Nf, pid_alt + Nf, sizeof(int), Nw);
            gl_add(G, p + Nf, p_alt + Nf, sizeof(T), Nw);
            if (uwl_set) gl_add(G, uwl, nstmp, sizeof(V), Nw);   // re-sort: carry the prescribed velocities
            SRET(gather(G, wp, Nw));
            // first sort: the walls' creation velocities are their prescribed velocities
            SCK(cudaMemcpyAsync(uwl, uwl_set ? nstmp : vel_alt + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            uwl_set = true;
            SCK(cudaMemcpyAsync(pos + Nf, pos_alt + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(vel + Nf, vel_alt + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rho + Nf, rho_alt + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(pid + Nf, pid_alt + Nf, Nw * sizeof(int), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(p + Nf, p_alt + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
            V* bufs[] = {pos_alt, rn, rstar};
            for (V* q : bufs) SCK(cudaMemcpyAsync(q + Nf, pos + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            if (dist()) {
                // new relative slot of every pre-sort wall slot
                ++nlaunch, k_invperm<<<nblk(Nw, 256), 256, 0, st>>>(wp, Nw, inv);
                for (int f = 0; f < 2; f++)
                    if (nws[f]) ++nlaunch, k_remap<<<nblk(nws[f], 256), 256, 0, st>>>(wsend[f], 0, nws[f], inv, wsend[f]);
                const int ngw = nwr[0] + nwr[1];
                if (ngw) ++nlaunch, k_remap<<<nblk(ngw, 256), 256, 0, st>>>(nullptr, Nwo, ngw, inv, wrecv);
                SCK(cudaGetLastError());
            }
        } else {
            SCK(cudaMemsetAsync(wstart, 0, (2 * (size_t)ncells + 2) * sizeof(int), st));
        }
        wnc_s[0] = wnc_s[1] = wnc_s[2] = -1;
        return SISPH_OK;
    }

    // first build at create (exact) and the wall normals (A0)
    int first_build()
    {
        SRET(build_fluid());
        if (Nw > 0) {
            if (Nwo) ++nlaunch, k_normals_raw<T, D><<<nblk(Nwo, 128), 128, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, nstmp);
            SCK(cudaGetLastError());
            if (dist()) {
                PackList L{};
                pl_add(L, nstmp, sizeof(V));
                SRET(halo_walls(L));
            }
            if (Nwo) ++nlaunch, k_normals_smooth<T, D><<<nblk(Nwo, 128), 128, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, nstmp, nrm);
            SCK(cudaGetLastError());
        }
        return SISPH_OK;
    }

    // sort the fluid block [0, Nf) on geometry G (owned first, ghosts after),
    // reorder the carried state; slab ranks remap their halo lists
    int sort_fluid(const Params<T>& G)
    {
        SRET(sort_set(G, pos, Nf, Nfo, fstart, perm));
        GatherList L{};
        gl_add(L, pos, pos_alt, sizeof(V), Nf);
        gl_add(L, vel, vel_alt, sizeof(V), Nf);
        gl_add(L, vt, vt_alt, sizeof(V), Nf);
        gl_add(L, p, p_alt, sizeof(T), Nf);
        gl_add(L, pid, pid_alt, sizeof(int), Nf);
        gl_add(L, rho, rho_alt, sizeof(T), Nf);
        gl_add(L, fs, fs_alt, 1, Nf);
        if (ptype) gl_add(L, ptype, ptype_alt, 1, Nf);
        SRET(gather(L, perm, Nf));
        // wall parts of the alternates
        SRET(copy_walls_to_alt());
        std::swap(pos, pos_alt);
        std::swap(vel, vel_alt);
        std::swap(vt, vt_alt);
        std::swap(p, p_alt);
        std::swap(pid, pid_alt);
        std::swap(rho, rho_alt);
        std::swap(fs, fs_alt);
        if (ptype) {
            std::swap(ptype, ptype_alt);
            P.ptype = PS.ptype = ptype;
        }
        if (dist() && Nf) {
            ++nlaunch, k_invperm<<<nblk(Nf, 256), 256, 0, st>>>(perm, Nf, inv);
            for (int f = 0; f < 2; f++)
                if (nfs[f]) ++nlaunch, k_remap<<<nblk(nfs[f], 256), 256, 0, st>>>(fsend_pre[f], 0, nfs[f], inv, fsend[f]);
            const int ng = nfr[0] + nfr[1];
            if (ng) ++nlaunch, k_remap<<<nblk(ng, 256), 256, 0, st>>>(nullptr, Nfo, ng, inv, grecv);
            SCK(cudaGetLastError());
        }
        return SISPH_OK;
    }

    // build at the current fluid positions: (slab ranks: migrate, halos,)
    // sort, reorder the carried state, neighbour lists
    int build_fluid(bool loose = false)
    {
        if (dist()) {
            SRET(migrate());
            SRET(fetch_ghosts());
        }
        if (loose) SRET(bin_walls_skin());
        SRET(sort_fluid(loose ? PS : P));
        if (loose && defer_loose_check) return build_loose();
        return loose ? build_loose_grow() : build_list_grow();
    }

    // ---- list capacities grow instead of failing: after a build or filter
    // the host reads the overflow flag (one small D2H); on overflow the list
    // is reallocated at 1.25 x the largest row and the same pass is redone
    // (the positions it reads have not changed).
    int read_overflow(int& mc)
    {
        SCK(cudaMemcpyAsync(&hctl->max_count, &ctl->max_count, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        mc = hctl->max_count;
        return SISPH_OK;
    }
    static int grown(int mc) { return ((int)ceil(1.25 * mc) + 8 + 7) / 8 * 8; }
    int build_list_grow(bool inner = false)
    {
        SRET(build_list(inner));
        int mc;
        SRET(read_overflow(mc));
        if (hctl->overflow) {
            SRET(alloc_list(grown(mc)));
            SRET(build_list(inner));
        }
        return SISPH_OK;
    }
    int regrow_loose(int mc)
    {
        const int want = grown(mc);
        if (nbs) cudaFree(nbs);
        nbs = nullptr;
        int rc = 0;
        nbs = dalloc<int>((size_t)want * rows32(capT), err, rc);
        if (rc) return rc;
        cap_s = PS.cap = want;
        return SISPH_OK;
    }
    int build_loose_grow()
    {
        SRET(build_loose());
        SCK(cudaMemcpyAsync(&hctl->max_count_s, &ctl->max_count_s, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        if (hctl->overflow_s) {
            SRET(regrow_loose(hctl->max_count_s));
            SRET(build_loose());
        }
        return SISPH_OK;
    }
    // single GPU, single build: the loose build's and the filter's capacities are checked with ONE
    // host wait after the filter (a loose overflow leaves a truncated loose list, the filter of it
    // is redone after the regrow; the positions neither pass reads have changed)
    bool defer_loose_check = false;
    int filter_checked()
    {
        for (int round = 0; round < 8; round++) {
            SRET(filter_list());
            SCK(cudaMemcpyAsync(&hctl->max_count, &ctl->max_count, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
            SCK(cudaMemcpyAsync(&hctl->max_count_s, &ctl->max_count_s, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                                st));
            SCK(cudaStreamSynchronize(st));
            if (hctl->overflow_s) {
                SRET(regrow_loose(hctl->max_count_s));
                SRET(build_loose());
                continue;
            }
            if (hctl->overflow) {
                SRET(alloc_list(grown(hctl->max_count)));
                continue;
            }
            return SISPH_OK;
        }
        err = "neighbour list capacity: no fit after repeated growth";
        return SISPH_EOVERFLOW;
    }
    int filter_list_grow()
    {
        SRET(filter_list());
        int mc;
        SRET(read_overflow(mc));
        if (hctl->overflow) {
            SCK(cudaMemsetAsync(&ctl->overflow, 0, sizeof(int), st));
            SRET(alloc_list(grown(mc)));
            SRET(filter_list());
        }
        return SISPH_OK;
    }

    int copy_walls_to_alt()
    {
        if (!Nw) return SISPH_OK;
        SCK(cudaMemcpyAsync(vel_alt + Nf, vel + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
        SCK(cudaMemcpyAsync(p_alt + Nf, p + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
        SCK(cudaMemcpyAsync(pid_alt + Nf, pid + Nf, Nw * sizeof(int), cudaMemcpyDeviceToDevice, st));
        SCK(cudaMemcpyAsync(rho_alt + Nf, rho + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
        SCK(cudaMemcpyAsync(us_alt + Nf, us + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
        return SISPH_OK;
    }

    // ------------------------------------------------------------------ API
    int build() override
    {
        SRET(build_fluid());
        phase = IDLE;
        return check_overflow();
    }

    int predict(double dt) override
    {
        if (!(dt > 0)) {
            err = "dt must be > 0";
            return SISPH_EINVAL;
        }
        last_dt = dt;
        bool single = false;
        if (dist()) {
            // migrate first: the skin is the max over the owned fluid of all ranks
#ifdef SISPH_DIST_PROF
            static cudaEvent_t pe[6];
            static bool pe_init = false;
            if (!pe_init) {
                for (auto& e : pe) cudaEventCreate(&e);
                pe_init = true;
            }
#define DPROF(k) cudaEventRecord(pe[k], st)
#else
#define DPROF(k)
#endif
            DPROF(0);
            SRET(migrate());
            DPROF(1);
            SRET(plan_skin(dt, single));
            if (!single) {
                err = "slab ranks need the single per-step build: 2 dt max|u~| exceeds 0.3 x 3h (reduce dt)";
                return SISPH_EINVAL;
            }
            DPROF(2);
            SRET(fetch_ghosts());
            DPROF(3);
            SRET(bin_walls_skin());
            SRET(sort_fluid(PS));
            DPROF(4);
            SRET(build_loose_grow());
            DPROF(5);
#ifdef SISPH_DIST_PROF
            cudaEventSynchronize(pe[5]);
            float t[5];
            for (int k = 0; k < 5; k++) cudaEventElapsedTime(&t[k], pe[k], pe[k + 1]);
            fprintf(stderr, "dist build ms: migrate %.3f plan_skin %.3f fetch_ghosts %.3f bin+sort %.3f loose %.3f\n",
                    t[0], t[1], t[2], t[3], t[4]);
#endif
#undef DPROF
        } else {
            SRET(plan_skin(dt, single));
            // A1-A5 at r^n (single build: the loose list on the skin grid, its capacity checked
            // together with the filter's)
            defer_loose_check = single;
            SRET(build_fluid(single));
            defer_loose_check = false;
        }
        SRET(mark(4));
        if (single) {
            // A9 (R3): r* = r^n + dt u~^n is known now: the exact sets at r* out of the loose list
            SRET(mark(5));
            SRET(compute_rstar(dt));
            SRET(dist() ? filter_list_grow() : filter_checked());
            SRET(mark(6));
        }
        const int* nb1 = single ? nbs : nbr;
        const int* cn1 = single ? cnt_s : cnt;
        const int cap1 = single ? cap_s : P.cap;
        // A6 (loose pairs beyond 3h contribute exactly 0: W, dW/dr vanish for q >= 3)
        if (Ntot) ++nlaunch, k_density<T, D><<<nblk(Ntot, 256), 256, 0, st>>>(P, pos, nb1, cn1, cap1, rho, fs, vel);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList L{};
            pl_add(L, vel, sizeof(V));   // rho rides in the 4th lane
            pl_add(L, rho, sizeof(T));
            SRET(halo_fluid(L));
            if (P.wall_rho_summation) {
                PackList W{};
                pl_add(W, rho + Nf, sizeof(T));
                SRET(halo_walls(W));
            }
        }
        // A7
        if (Nwo) ++nlaunch, k_wall_velocity<T, D><<<nblk(Nwo, 256), 256, 0, st>>>(P, pos, nb1, cn1, cap1, nrm, rho, uwl, vel, 0);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList W{};
            pl_add(W, vel + Nf, sizeof(V));
            SRET(halo_walls(W));
        }
        // A8 (neighbours' {r, m, u, rho} packed into one 256-bit record)
        if (Ntot) ++nlaunch, k_pack_rec<T><<<nblk(Ntot, 256), 256, 0, st>>>(pos, vel, Ntot, reinterpret_cast<T*>(recF));
        if (Nfo) ++nlaunch, k_forces_predict<T, D><<<nblk(Nfo, 128), 128, 0, st>>>(P, (T)dt, pos, vel, vt, rho, nb1, cn1, cap1, us,
                                                                                   single ? nullptr : rstar, fnp,
                                                                                   reinterpret_cast<const T*>(recF));
        SCK(cudaGetLastError());
        if (dist()) {
            PackList L{};
            if (!single) pl_add(L, rstar, sizeof(V), 1);   // single build: compute_rstar did
            pl_add(L, us, sizeof(V));
            SRET(halo_fluid(L));
        }
        if (single) {
            // r* becomes the current position set (walls are in every buffer), r^n is kept as rn
            std::swap(pos, rstar);
            std::swap(rn, rstar);
        } else {
            SRET(mark(5));
            // A9: build at r*; carry r^n along as rn
            SRET(sort_set(P, rstar, Nf, Nf, fstart, perm));
            GatherList G{};
            gl_add(G, rstar, pos_alt, sizeof(V), Nf);
            gl_add(G, pos, rn, sizeof(V), Nf);
            gl_add(G, vel, vel_alt, sizeof(V), Nf);
            gl_add(G, vt, vt_alt, sizeof(V), Nf);
            gl_add(G, us, us_alt, sizeof(V), Nf);
            gl_add(G, rho, rho_alt, sizeof(T), Nf);
            gl_add(G, fs, fs_alt, 1, Nf);
            gl_add(G, p, p_alt, sizeof(T), Nf);
            gl_add(G, pid, pid_alt, sizeof(int), Nf);
            if (ptype) gl_add(G, ptype, ptype_alt, 1, Nf);
            SRET(gather(G, perm, Nf));
            if (ptype) {
                std::swap(ptype, ptype_alt);
                P.ptype = PS.ptype = ptype;
            }
            SRET(copy_walls_to_alt());
            std::swap(pos, pos_alt);
            std::swap(vel, vel_alt);
            std::swap(vt, vt_alt);
            std::swap(us, us_alt);
            std::swap(rho, rho_alt);
            std::swap(fs, fs_alt);
            std::swap(p, p_alt);
            std::swap(pid, pid_alt);
            SRET(build_list_grow(true));   // + GTVF inner list
            SRET(mark(6));
        }
        // A10
        if (Nwo) ++nlaunch, k_wall_velocity<T, D><<<nblk(Nwo, 256), 256, 0, st>>>(P, pos, nbr, cnt, P.cap, nrm, rho, uwl, us, P.ustar_noslip ? 0 : 1);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList W{};
            pl_add(W, us + Nf, sizeof(V));
            SRET(halo_walls(W));
        }
        // A11 with the first PPE sweep fused (walls first get p^0, R14); neighbours' {r*, m, u*, rho}
        // packed into one 256-bit record
        if (Ntot) ++nlaunch, k_pack_rec<T><<<nblk(Ntot, 256), 256, 0, st>>>(pos, us, Ntot, reinterpret_cast<T*>(recS));
        SCK(cudaMemsetAsync(&ctl->lambda_bits, 0, sizeof(unsigned long long), st));
        SCK(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), st));  // ticket, iter, done, nonfinite
        SRET(mark(7));   // t_PPE starts at A11 (wall p^0, RHS, D_ii, sweep 1)
        if (Nwo) ++nlaunch, k_wall_pressure<T, D><<<nblk((long)Nwo * WL, 256), 256, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, p);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList W{};
            pl_add(W, p + Nf, sizeof(T));
            SRET(halo_walls(W));
        }
        ++nlaunch, (code ? k_rhs_diag<T, D, true> : k_rhs_diag<T, D, false>)<<<std::max(nblk(Nfo, RHS_T), 1), RHS_T, 0,
                                                                                  st>>>(
                       P, (T)(1.0 / dt), pos, us, rho, fs, nbr, cnt, P.cap, rhs, diag, coef, ctl, p, p_alt, partials,
                       reinterpret_cast<const T*>(recS), code, nslot, cc8);
        SCK(cudaGetLastError());
        SRET(mark(8));
        pre_swept = true;
        // Lambda is global (eq:convergence): the bits of a non-negative double order as the value
        if (dist()) SRET(xallreduce(reinterpret_cast<double*>(&ctl->lambda_bits), 1, 1));
        phase = PREDICTED;
        return SISPH_OK;
    }

    static constexpr int MAXREC = 64;
    cudaEvent_t sev[2 * MAXREC] = {};
    int nrec = 0;
    double last_ms_sweeps = 0;
    int last_sweeps_timed = 0;

    // ---- the PPE iteration: per-solve state in a device descriptor, so the
    // same kernels run host-polled (speculative batches; timing, slab ranks)
    // or as the WHILE body of a captured CUDA graph (one launch per solve,
    // the loop condition set on the device by the sweep's last block)
    PpeDesc<T>* ddesc = nullptr;
    PpeDesc<T>* hdesc = nullptr;   // pinned
    int ppe_loop = 0;              // 0 auto, 1 host-polled batches, 2 graph WHILE node, 3 persistent
    int pgrid_max = 0;             // co-resident blocks of the persistent PPE kernel
    int pgrid_cache = -1;          // ... with the row cache's dynamic shared memory (-1: not asked yet)
    int pcache_csm = -1;           // the cached chunks per row pgrid_cache was computed for
    cudaStream_t cst = nullptr;    // capture stream (the handle's stream may be the legacy default)
    cudaGraph_t pgraph = nullptr;
    cudaGraphExec_t pexec = nullptr;
    cudaGraphConditionalHandle pcond = 0;
    long long gkey[5] = {-1, -1, -1, -1, -1};

    // R12b: eq:convergence on means (1 / global fluid count) or on the printed sums (1)
    int conv_mean = 0;
    int64_t nf_glob = 0;
    double cscale() const { return conv_mean && nf_glob > 0 ? 1.0 / (double)nf_glob : 1.0; }

    int write_desc(double tl, int mi, int mx)
    {
        if (!ddesc) {
            int rc = 0;
            ddesc = dalloc<PpeDesc<T>>(1, err, rc);
            if (rc) return rc;
            SCK(cudaHostAlloc((void**)&hdesc, sizeof(PpeDesc<T>), cudaHostAllocDefault));
        }
        hdesc->pos = pos;
        hdesc->rho = rho;
        hdesc->fs = fs;
        hdesc->nbr = nbr;
        hdesc->coef = coef;
        hdesc->code = code;
        hdesc->nslot = nslot;
        hdesc->cc8 = cc8;
        hdesc->pA = p;
        hdesc->pB = p_alt;
        hdesc->tol = tl;
        hdesc->cscale = cscale();
        hdesc->min_it = mi;
        hdesc->max_it = mx;
        SCK(cudaMemcpyAsync(ddesc, hdesc, sizeof(PpeDesc<T>), cudaMemcpyHostToDevice, st));
        return SISPH_OK;
    }

    void drop_graph()
    {
        if (pexec) cudaGraphExecDestroy(pexec);
        if (pgraph) cudaGraphDestroy(pgraph);
        pexec = nullptr;
        pgraph = nullptr;
    }

    // (re)capture the loop when what the kernels take by value changes
    int ensure_graph()
    {
        const long long key[5] = {P.cap, Nfo, Nwo, coef ? 1 : 0, Nf};
        if (pexec && !memcmp(key, gkey, sizeof(key))) return SISPH_OK;
        drop_graph();
        if (!cst) SCK(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
        SCK(cudaGraphCreate(&pgraph, 0));
        SCK(cudaGraphConditionalHandleCreate(&pcond, pgraph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = pcond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        SCK(cudaGraphAddNode(&node, pgraph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        SCK(cudaStreamBeginCaptureToGraph(cst, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        if (Nwo) SCK(klaunch(k_ppe_wall<T, D>, nblk((long)Nwo * WL, 256), 256, cst, P, (const PpeDesc<T>*)ddesc,
                             (const int*)cnt, P.cap, (const Ctl*)ctl));
        const int nb = std::max(nblk(Nfo, SWEEP_T), 1);
        const int uh = P.mean_free ? 0 : 1;   // mean-free: k_mean_fix decides and sets the condition
        SCK(klaunch(coef ? (code ? k_sweep<T, D, true, true> : k_sweep<T, D, true, false>) : k_sweep<T, D, false>, nb, SWEEP_T, cst, P, (const PpeDesc<T>*)ddesc,
                    (const T*)rhs, (const T*)diag, (const int*)cnt, P.cap, ctl, partials, 0, pcond, uh));
        if (P.mean_free)
            SCK(klaunch(k_mean_fix<T>, nb, SWEEP_T, cst, P, (const PpeDesc<T>*)ddesc, (const T*)diag, ctl, partials, 0,
                        pcond, 1));
        cudaError_t le = cudaGetLastError();
        SCK(cudaStreamEndCapture(cst, &body));
        SCK(le);
        SCK(cudaGraphInstantiate(&pexec, pgraph, 0));
        memcpy(gkey, key, sizeof(key));
        return SISPH_OK;
    }

    // the whole PPE loop in one thread-block cluster (k_ppe_cluster): up to 16 blocks of 1024
    // threads (non-portable cluster size; 8 if the device refuses 16)
    int cluster_max = 16;
    int launch_cluster()
    {
        void* fn = coef ? (void*)k_ppe_cluster<T, D, true> : (void*)k_ppe_cluster<T, D, false>;
        const long need = std::max((long)Nfo, (long)Nwo * WL);
        for (;;) {
            int nbk = (int)std::min<long>(cluster_max, std::max<long>(1, (need + CLUSTER_T - 1) / CLUSTER_T));
            if (nbk > 8) SCK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nbk);
            cfg.blockDim = dim3(CLUSTER_T);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = nbk;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int cap = P.cap;
            cudaError_t le;
            if (coef)
                le = cudaLaunchKernelEx(&cfg, k_ppe_cluster<T, D, true>, P, (const PpeDesc<T>*)ddesc, (const T*)rhs,
                                        (const T*)diag, (const int*)cnt, cap, ctl);
            else
                le = cudaLaunchKernelEx(&cfg, k_ppe_cluster<T, D, false>, P, (const PpeDesc<T>*)ddesc, (const T*)rhs,
                                        (const T*)diag, (const int*)cnt, cap, ctl);
            if (le == cudaSuccess) break;
            (void)cudaGetLastError();
            if (cluster_max <= 1) {
                err = std::string("cluster PPE launch: ") + cudaGetErrorString(le);
                return SISPH_ECUDA;
            }
            cluster_max /= 2;   // e.g. no 16-SM cluster available: retry smaller
        }
        ++nlaunch;
        return SISPH_OK;
    }

    int launch_persistent()
    {
        void* fn = coef ? (void*)k_ppe_persistent<T, D, true> : (void*)k_ppe_persistent<T, D, false>;
        if (!pgrid_max) {
            int per = 0, dev = 0, sms = 0;
            SCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, SWEEP_T, 0));
            SCK(cudaGetDevice(&dev));
            SCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            pgrid_max = std::max(1, std::min(per * sms, 4096));   // partials: 2 parities x 2 per block
        }
        const int want = nblk(std::max((long)Nfo, (long)Nwo * WL), SWEEP_T);
        // the row cache (k_ppe_persistent): csm chunks per thread of dynamic shared memory, when
        // the blocks that give every thread at most one row are still co-resident with it
        int csm_try = coef ? (sizeof(T) == 4 ? 8 : 3) : 0;
        if (const char* e = getenv("SISPH_PERS_CACHE")) csm_try = coef ? std::max(0, std::min(atoi(e), 8)) : 0;   // A/B
        const size_t dyn_try = (size_t)csm_try * SWEEP_T * (4 * sizeof(T) + 4 * sizeof(unsigned short)) +
                               (size_t)WCE * SWEEP_T * (sizeof(int) + sizeof(T));   // + the wall cache
        if (pgrid_cache < 0 || pcache_csm != csm_try) {   // (the A/B switch may change between launches)
            pgrid_cache = 0;
            pcache_csm = csm_try;
            {
                int per = 0, dev = 0, sms = 0;
                if (csm_try && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_try) == cudaSuccess &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, SWEEP_T, dyn_try) == cudaSuccess) {
                    SCK(cudaGetDevice(&dev));
                    SCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
                    pgrid_cache = std::min(per * sms, 4096);
                } else {
                    cudaGetLastError();
                }
            }
        }
        const bool use_cache = csm_try && want <= pgrid_cache;
        int csm = use_cache ? csm_try : 0;
        const size_t dyn = use_cache ? dyn_try : 0;
        const int grid = std::max(1, std::min(use_cache ? pgrid_cache : pgrid_max, want));
        int cap = P.cap;
        void* args[] = {&P, &ddesc, &rhs, &diag, &cnt, &cap, &ctl, &partials, &csm};
        SCK(cudaMemsetAsync(&ctl->gbar, 0, sizeof(unsigned int), st));
        ++nlaunch;
        SCK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(SWEEP_T), args, dyn, st));
        return SISPH_OK;
    }

    // R32: remove the live-row mean of the iterate the sweep just wrote
    // (slab ranks: the live sum and count are allreduced first, the residual
    // sums after) and reduce eq:convergence on the corrected iterate
    int mean_fix()
    {
        if (dist()) SRET(xallreduce(ctl->red, 3, 0));
        const int nb = std::max(nblk(Nfo, SWEEP_T), 1);
        ++nlaunch;
        SCK(klaunch(k_mean_fix<T>, nb, SWEEP_T, st, P, (const PpeDesc<T>*)ddesc, (const T*)diag, ctl, partials,
                    dist() ? 1 : 0, pcond, 0));
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    // the PPE loop's kernels (k_ppe_wall, k_sweep, k_mean_fix) with programmatic dependent
    // launch on problems whose sweeps are launch-latency bound (each kernel waits on its
    // predecessor before reading anything: griddepcontrol.wait)
    int pdl = -1;   // -1: auto (Nfo <= 400000), SISPH_PDL=0/1 overrides
    template <class... KArgs, class... Args>
    cudaError_t klaunch(void (*k)(KArgs...), int grid, int block, cudaStream_t s, Args... args)
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = (pdl < 0 ? Nfo <= 400000 : pdl != 0) ? 1 : 0;
        return cudaLaunchKernelEx(&cfg, k, args...);
    }

    int launch_sweeps(int count, double tl, int mi, int mx)
    {
        for (int c = 0; c < count; c++) {
            if (Nwo) {
                ++nlaunch;
                SCK(klaunch(k_ppe_wall<T, D>, nblk((long)Nwo * WL, 256), 256, st, P, (const PpeDesc<T>*)ddesc,
                            (const int*)cnt, P.cap, (const Ctl*)ctl));
            }
            if (dist()) SRET(halo_p(true));
            bool rec = timing && nrec < MAXREC;
            if (rec) {
                if (!sev[2 * nrec]) {
                    SCK(cudaEventCreate(&sev[2 * nrec]));
                    SCK(cudaEventCreate(&sev[2 * nrec + 1]));
                }
                SCK(cudaEventRecord(sev[2 * nrec], st));
            }
            const int defer = dist() ? 1 : 0;
            const int nb = std::max(nblk(Nfo, SWEEP_T), 1);   // one block at least: the last block decides
            ++nlaunch;
            SCK(klaunch(coef ? (code ? k_sweep<T, D, true, true> : k_sweep<T, D, true, false>) : k_sweep<T, D, false>, nb, SWEEP_T, st, P,
                        (const PpeDesc<T>*)ddesc, (const T*)rhs, (const T*)diag, (const int*)cnt, P.cap, ctl, partials,
                        defer, pcond, 0));
            if (P.mean_free) SRET(mean_fix());
            if (rec) {
                SCK(cudaEventRecord(sev[2 * nrec + 1], st));
                nrec++;
            }
            if (dist()) {
                // eq:convergence over all ranks: allreduce the local sums, decide, refresh p^{k+1}
                SRET(xallreduce(ctl->red, 3, 0));
                ++nlaunch, k_decide<<<1, 1, 0, st>>>(ctl, tl, mi, mx, cscale());
                SRET(halo_p(false));
            }
        }
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    int solve(double tl, int mx, int* iters, double* res) override
    {
        if (phase == IDLE) {
            err = "sisph_ppe_solve needs a preceding sisph_predict";
            return SISPH_EINVAL;
        }
        if (tl < 0 || mx < 1) {
            err = "tol must be >= 0 and max_iter >= 1";
            return SISPH_EINVAL;
        }
        int mi = std::min(min_iter, mx);
        int launched = 0;
        nrec = 0;
        const bool pre = pre_swept;
        pre_swept = false;
        SRET(write_desc(tl, mi, mx));
        if (pre) {
            // sweep 1 ran inside A11 as a deferred sweep: decide it now with this
            // solve's tolerance and bounds (slab ranks: sums allreduced first;
            // mean-free: the mean is removed first, k_mean_fix decides one handle)
            if (P.mean_free) SRET(mean_fix());
            if (dist() || !P.mean_free) {
                if (dist()) SRET(xallreduce(ctl->red, 3, 0));
                ++nlaunch, k_decide<<<1, 1, 0, st>>>(ctl, tl, mi, mx, cscale());
            }
            SCK(cudaGetLastError());
            if (dist()) SRET(halo_p(false));
            launched = 1;
        } else {
            SCK(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), st));  // ticket, iter, done, nonfinite
        }
        // the loop form: one handle with timing off may run the whole loop on the device.
        // Auto (0): one thread-block cluster for <= 16k rows (C1: 2.37 -> 1.83 ms per step),
        // the persistent cooperative kernel up to 400k rows (C2: 1.67 vs 2.15 ms with the
        // graph's WHILE node, 10-step runs; the mean-free loop falls back to the graph), host
        // batches for large ones (a few HBM-bound sweeps per step)
        int mode = ppe_loop == 0 ? (Nfo <= 16384 ? 4 : (Nfo <= 400000 ? 3 : 1)) : ppe_loop;
        if (dist() || timing || Nf == 0 || launched >= mx) mode = 1;
        if (mode == 3 && P.mean_free) mode = 2;   // the persistent loop has no mean-free phase
        if (mode == 4) {
            // one thread-block cluster runs the loop (walls, sweep, mean, reduction, decision),
            // separated by hardware cluster barriers
            SRET(launch_cluster());
            SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
#ifdef SISPH_PERS_PROF
            {
                std::vector<unsigned long long> hp(4096 * 6);
                SCK(cudaMemcpyFromSymbol(hp.data(), g_pers_prof, hp.size() * sizeof(unsigned long long)));
                const int its = std::max(hctl->iter - launched, 1);
                fprintf(stderr, "cluster its=%d us/it (block 0): walls %.2f sweep %.2f blocksum %.2f barrier %.2f "
                        "clustersum %.2f r32+decide %.2f\n", its, hp[0] * 1e-3 / its, hp[1] * 1e-3 / its,
                        hp[2] * 1e-3 / its, hp[3] * 1e-3 / its, hp[4] * 1e-3 / its, hp[5] * 1e-3 / its);
            }
#endif
        } else if (mode == 3) {
            // one cooperative launch: walls, sweep, fixed-order reduction and decision per
            // iteration, separated by grid syncs (small problems: no per-sweep launches)
            SRET(launch_persistent());
            SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
#ifdef SISPH_PERS_PROF
            {
                std::vector<unsigned long long> hp(4096 * 6);
                SCK(cudaMemcpyFromSymbol(hp.data(), g_pers_prof, hp.size() * sizeof(unsigned long long)));
                const int nb = std::max(1, std::min(pgrid_max, nblk(std::max((long)Nfo, (long)Nwo * WL), SWEEP_T)));
                const int its = std::max(hctl->iter - launched, 1);
                double mean[5] = {0}, mx[5] = {0};
                int ntiled = 0;
                unsigned long long tmax = 0;
                for (int b = 0; b < nb; b++) {
                    ntiled += hp[b * 6 + 5] != 0;
                    tmax = std::max(tmax, hp[b * 6 + 5]);
                }
                fprintf(stderr, "pers tiled blocks %d of %d, largest span %llu\n", ntiled, nb, tmax);
                for (int b = 0; b < nb; b++)
                    for (int k = 0; k < 5; k++) {
                        const double v = hp[b * 6 + k] * 1e-3 / its;
                        mean[k] += v / nb;
                        mx[k] = std::max(mx[k], v);
                    }
                fprintf(stderr, "pers its=%d blocks=%d us/it mean|max: sweep %.2f|%.2f bar2 %.2f|%.2f walls+decide %.2f|%.2f "
                        "bar1 %.2f|%.2f - %.2f|%.2f\n", its, nb, mean[0], mx[0], mean[1], mx[1], mean[2], mx[2],
                        mean[3], mx[3], mean[4], mx[4]);
            }
#endif
        } else if (mode == 2) {
            // one launch: WHILE (not done) { wall pressure; sweep }  (sweeps after the
            // decision never run; the host waits once)
            SRET(ensure_graph());
            SCK(cudaGraphLaunch(pexec, st));
            SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
            // kernels the body ran: one (wall, sweep) pair per sweep + the one that saw done
            nlaunch += (Nwo ? 2 : 1) * (std::max(hctl->iter - launched, 0) + 1);
            if (P.mean_free) nlaunch += std::max(hctl->iter - launched, 0) + 1;
        } else if (Nf > 0 || dist()) {
            // speculative batches: sweeps after convergence are no-ops on the device
            // (slab ranks take the same decisions, so they run the same batches)
            int batch = std::min(mx - launched, std::max(mi, 2) + 1 - launched);
            for (;;) {
                if (batch > 0) {
                    SRET(launch_sweeps(batch, tl, mi, mx));
                    launched += batch;
                }
                SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
                SCK(cudaStreamSynchronize(st));
                if (hctl->done || launched >= mx) break;
                batch = std::min(mx - launched, std::min(2 * std::max(batch, 1), 32));
            }
        } else {
            hctl->iter = 0;
            hctl->residual = 0;
            hctl->nonfinite = 0;
        }
        int k = hctl->iter;
        if (k & 1) std::swap(p, p_alt);
        // p^k's buffer holds fluid p^k; the wall values of the last sweep (from
        // p^{k-1}, R14) are in the other buffer
        if (Nw && k > 0)
            SCK(cudaMemcpyAsync(p + Nf, p_alt + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
        last_ms_sweeps = 0;
        last_sweeps_timed = std::min(k - (pre ? 1 : 0), nrec);   // the fused first sweep is not timed apart
        for (int q = 0; q < last_sweeps_timed; q++) {
            float ms = 0;
            SCK(cudaEventElapsedTime(&ms, sev[2 * q], sev[2 * q + 1]));
            last_ms_sweeps += ms;
        }
        if (iters) *iters = k;
        if (res) *res = hctl->residual;
        phase = SOLVED;
        if (hctl->nonfinite) {
            err = "non-finite pressure in the PPE sweep";
            return SISPH_ENONFINITE;
        }
        return SISPH_OK;
    }

    // K modified-GTVF sub-steps (A14) from r* = pos; returns delta^K = r^K - r^0 in rK (stride
    // rstride working-precision values per slot, delta in the last four)
    // slab ranks, fp32 GTVF: the ghosts' delta^k from their owners (no image shift),
    // unpacked straight into their fixed-point records (pack, send / receive, fused unpack)
    int gtvf_halo_fx(cudaStream_t hs, int4* f0, float4* dl, const int4* src, int4* dst)
    {
        if constexpr (std::is_same<T, float>::value) {
            PackList L{};
            pl_add(L, dk, sizeof(V));
            L.rec = sizeof(V);
            L.axis = axis;
            for (int f = 0; f < 2; f++) SRET(ensure_buf(f, (size_t)std::max(nfs[f], nfr[f]) * L.rec));
            if (nfs[0] + nfs[1] > 0) {
                ++nlaunch, k_pack2<T><<<nblk(nfs[0] + nfs[1], 256), 256, 0, hs>>>(
                               L, 0.0, 0.0, fsend[0], fsend[1], nfs[0], nfs[1], sbuf[0], sbuf[1]);
                halo_bytes += (int64_t)(nfs[0] + nfs[1]) * L.rec;
            }
            const void* sb[2] = {sbuf[0], sbuf[1]};
            void* rb[2] = {rbuf[0], rbuf[1]};
            const size_t sz[2] = {(size_t)nfs[0] * L.rec, (size_t)nfs[1] * L.rec};
            const size_t rz[2] = {(size_t)nfr[0] * L.rec, (size_t)nfr[1] * L.rec};
            if (tp->sendrecv(sb, sz, rb, rz, hs)) return tperr();
            if (nfr[0] + nfr[1] > 0)
                ++nlaunch, k_unpack_gtvf_fx<<<nblk(nfr[0] + nfr[1], 256), 256, 0, hs>>>(
                               grecv, nfr[0], nfr[1], reinterpret_cast<const float4*>(rbuf[0]),
                               reinterpret_cast<const float4*>(rbuf[1]), f0, dl, src, dst, P.fxf[0], P.fxf[1],
                               P.fxf[2], D == 3);
            SCK(cudaGetLastError());

        }
        return SISPH_OK;
    }

    int gtvf_substeps(T dtau, bool inner, const T*& rK, int& rstride)
    {
        if (inner) SCK(cudaMemsetAsync(&ctl->gtvf_far, 0, sizeof(int), st));
        if constexpr (std::is_same<T, float>::value) {
            // fp32: 16-byte fixed-point records (k_gtvf_substep_fx)
            int4* a = reinterpret_cast<int4*>(gtA);
            int4* b = reinterpret_cast<int4*>(gtB);
            int4* f0 = reinterpret_cast<int4*>(fx0);
            float4* dl = reinterpret_cast<float4*>(dk);
            float4* vv = reinterpret_cast<float4*>(vk);
#ifdef SISPH_DIST_PROF
            static cudaEvent_t ge[2] = {nullptr, nullptr};
            if (!ge[0]) {
                cudaEventCreate(&ge[0]);
                cudaEventCreate(&ge[1]);
            }
            cudaEventRecord(ge[0], st);
#endif
            if (Ntot) ++nlaunch, k_gtvf_prep_fx<D><<<nblk(Ntot, 256), 256, 0, st>>>(P, pos, rho, Ntot, a, b, f0, dl);
            bool iso = true;   // one fixed-point unit on every axis (k_gtvf_substep_fx<D, true>)
            for (int q = 1; q < D; q++) iso = iso && P.fxf[q] == P.fxf[0];
            auto kf = iso ? k_gtvf_substep_fx<D, true> : k_gtvf_substep_fx<D, false>;
            const int* lst = inner ? nbr_in : nbr;
            const int lcap = inner ? P.cap_in : P.cap;
            const int* lcnt = inner ? cnt_in : cnt;
            const int chk = inner ? 1 : 0;
            // slab ranks: rows other ranks hold as ghosts first, their halo overlapped with the rest
            const int nbnd = dist() ? nfs[0] + nfs[1] : 0;
            const bool ovl = dist() && gtvf_overlap && Nfo > 0 && nbnd > 0;
            if (ovl) {
                if (!hst) {
                    // the halo stream's blocks go first whenever an SM frees up (the interior rows'
                    // blocks are short), so the exchange does not wait for the whole interior kernel
                    int lo = 0, hi = 0;
                    SCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                    SCK(cudaStreamCreateWithPriority(&hst, cudaStreamNonBlocking, hi));
                }
                for (auto& e : gev)
                    if (!e) SCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                SCK(cudaMemsetAsync(bflag, 0, (size_t)Nfo * sizeof(int), st));
                for (int f = 0; f < 2; f++)
                    if (nfs[f]) ++nlaunch, k_set_flag<<<nblk(nfs[f], 256), 256, 0, st>>>(fsend[f], nfs[f], bflag);
                SRET(scan(bflag, dpre, Nfo));
                ++nlaunch, k_split_rows<<<nblk(Nfo, 256), 256, 0, st>>>(bflag, dpre, Nfo, brow, irow, gcnt);
                SCK(cudaGetLastError());
            }
            const int4* src = b;
            for (int k = 0; k < K; k++) {
                int4* dst = (k & 1) ? b : a;
                if (ovl) {
                    ++nlaunch, kf<<<nblk(nbnd, 128), 128, 0, st>>>(P, dtau, src, dst, f0, dl, vv, p, lst, lcap, lcnt,
                                                                   k == 0, chk, ctl, brow, gcnt);
                    SCK(cudaEventRecord(gev[0], st));
                    ++nlaunch, kf<<<nblk(Nfo, 128), 128, 0, st>>>(P, dtau, src, dst, f0, dl, vv, p, lst, lcap, lcnt,
                                                                  k == 0, chk, ctl, irow, gcnt + 1);
                    SCK(cudaGetLastError());
                    SCK(cudaStreamWaitEvent(hst, gev[0], 0));
                    SRET(gtvf_halo_fx(hst, f0, dl, src, dst));
                    SCK(cudaEventRecord(gev[1], hst));
                    SCK(cudaStreamWaitEvent(st, gev[1], 0));
                } else {
                    if (Nfo)
                        ++nlaunch, kf<<<nblk(Nfo, 128), 128, 0, st>>>(P, dtau, src, dst, f0, dl, vv, p, lst, lcap,
                                                                      lcnt, k == 0, chk, ctl, nullptr, nullptr);
                    SCK(cudaGetLastError());
                    if (dist()) SRET(gtvf_halo_fx(st, f0, dl, src, dst));
                }
                src = dst;
            }
#ifdef SISPH_DIST_PROF
            cudaEventRecord(ge[1], st);
            cudaEventSynchronize(ge[1]);
            float gms = 0;
            cudaEventElapsedTime(&gms, ge[0], ge[1]);
            fprintf(stderr, "gtvf substeps ms %.3f\n", gms);
#endif
            rK = reinterpret_cast<const T*>(dk);
            rstride = 4;
        } else {
            T* a = reinterpret_cast<T*>(gtA);
            T* b = reinterpret_cast<T*>(gtB);
            if (Ntot) ++nlaunch, k_gtvf_prep<T><<<nblk(Ntot, 256), 256, 0, st>>>(pos, rho, Ntot, a, b);
            const T* src = b;
            for (int k = 0; k < K; k++) {
                T* dst = (k & 1) ? b : a;
                if (Nfo) {
                    if (inner)
                        ++nlaunch, k_gtvf_substep<T, D><<<nblk(Nfo, 128), 128, 0, st>>>(P, dtau, src, dst, vk, p, nbr_in,
                                                                                        P.cap_in, cnt_in, k == 0, 1, ctl);
                    else
                        ++nlaunch, k_gtvf_substep<T, D><<<nblk(Nfo, 128), 128, 0, st>>>(P, dtau, src, dst, vk, p, nbr,
                                                                                        P.cap, cnt, k == 0, 0, ctl);
                }
                SCK(cudaGetLastError());
                if (dist()) {
                    // the record's r* carries the periodic image shift of the ghost, delta does not
                    PackList L{};
                    pl_add(L, dst, 2 * sizeof(V), 1);
                    SRET(halo_fluid(L));
                }
                src = dst;
            }
            rK = src;   // delta^K in the second V4 of each record
            rstride = 8;
        }
        return SISPH_OK;
    }

    int correct(double dt) override
    {
        if (phase != SOLVED) {
            err = "sisph_correct needs a preceding sisph_ppe_solve";
            return SISPH_EINVAL;
        }
        if (!(dt > 0)) {
            err = "dt must be > 0";
            return SISPH_EINVAL;
        }
        // A13
        if (Nwo) ++nlaunch, k_wall_pressure<T, D><<<nblk((long)Nwo * WL, 256), 256, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, p);
        SCK(cudaGetLastError());
        if (dist()) {
            PackList W{};
            pl_add(W, p + Nf, sizeof(T));
            SRET(halo_walls(W));
        }
        SCK(cudaMemsetAsync(&ctl->fmax2_bits, 0, 2 * sizeof(unsigned long long), st));
        if (pref_auto && !pref_done) {
            // R33: p_ref = 2 max p over the fluid of this first solve (all ranks), then constant
            double* dm = reinterpret_cast<double*>(&ctl->red[3]);
            ++nlaunch, k_fluid_pmax<T><<<1, 1024, 0, st>>>(p, Nfo, ptype, dm);
            SCK(cudaGetLastError());
            if (dist()) SRET(xallreduce(dm, 1, 1));
            double mx = 0;
            SCK(cudaMemcpyAsync(&mx, dm, sizeof(double), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
            const double pr = std::isfinite(mx) ? 2.0 * mx : 0.0;
            P.p_ref = (T)pr;
            PS.p_ref = (T)pr;
            pref_done = true;
        }
        if (Nfo) ++nlaunch, k_pgrad_correct<T, D><<<nblk(Nfo, 128), 128, 0, st>>>(P, (T)dt, pos, rho, p, us, nbr, cnt, P.cap, vel, fnp, ctl);
        // A14: K sub-steps (p0 = 0 everywhere when p_ref == 0: the shift is exactly zero)
        const T* rK = nullptr;   // delta^K = r^K - r^0 of the GTVF sub-steps (none when p0 = 0)
        int rstride = 4;
        if (P.p_ref != T(0) && K > 0 && (Nf || dist())) {
            SRET(gtvf_substeps((T)(dt / K), inner_valid, rK, rstride));
            if (inner_valid) {
                // the inner list is exact only while no particle moved more than skin/2
                // (slab ranks: if any rank's did, all repeat)
                if (dist()) {
                    int far = 0;
                    SCK(cudaMemcpyAsync(&hctl->gtvf_far, &ctl->gtvf_far, sizeof(int), cudaMemcpyDeviceToHost, st));
                    SCK(cudaStreamSynchronize(st));
                    far = hctl->gtvf_far;
                    SRET(allreduce_host(&far, 1));
                    hctl->gtvf_far = far;
                } else {
                    SCK(cudaMemcpyAsync(&hctl->gtvf_far, &ctl->gtvf_far, sizeof(int), cudaMemcpyDeviceToHost, st));
                    SCK(cudaStreamSynchronize(st));
                }
                if (hctl->gtvf_far) {
                    gtvf_fallbacks++;
                    SRET(gtvf_substeps((T)(dt / K), false, rK, rstride));
                }
            }
        }
        // A15 (R34: the outlet's advection velocity first, from the fluid's u^{n+1} at r*)
        if (open_x && Nfo)
            ++nlaunch, k_outlet_velocity<T, D><<<nblk(Nfo, 256), 256, 0, st>>>(P, pos, vel, nbr, cnt, P.cap, uout);
        if (Nfo) ++nlaunch, k_advance<T, D><<<nblk(Nfo, 256), 256, 0, st>>>(P, (T)dt, rK, rstride, rn, vel, pos, vt, ctl, uout);
        SCK(cudaGetLastError());
        if (open_x) SRET(open_boundaries());
        phase = IDLE;
        stepped = true;
        return SISPH_OK;
    }

    int step(double dt, sisph_step_report* rep) override
    {
        int64_t l0 = nlaunch;
        int64_t hb0 = halo_bytes;
        evmask = 0;
        SRET(mark(0));
        SRET(predict(dt));
        SRET(mark(1));
        int it = 0;
        double res = 0;
        SRET(solve(tol, max_iter, &it, &res));
        SRET(mark(2));
        SRET(correct(dt));
        SRET(mark(3));
        if (rep) {
            memset(rep, 0, sizeof(*rep));
            rep->dt = dt;
            rep->iters = it;
            rep->residual = res;
            unsigned long long lb = hctl->lambda_bits;
            memcpy(&rep->lambda, &lb, sizeof(double));
            rep->max_neighbors = hctl->max_count;
            rep->pairs = (int64_t)hctl->pairs_fluid;
            rep->ms_sweeps = last_ms_sweeps;
            rep->sweeps_timed = last_sweeps_timed;
            rep->launches = nlaunch - l0;
            rep->single_build = skin_used ? 1 : 0;
            rep->skin_radius = skin_radius;
            rep->n_owned_fluid = Nfo;
            rep->n_ghost_fluid = Nf - Nfo;
            rep->halo_bytes = halo_bytes - hb0;
            if (timing) {
                SCK(cudaEventSynchronize(ev[3]));
                float a, b, c;
                cudaEventElapsedTime(&a, ev[0], ev[1]);
                cudaEventElapsedTime(&b, ev[1], ev[2]);
                cudaEventElapsedTime(&c, ev[2], ev[3]);
                rep->ms_predict = a;
                rep->ms_solve = b;
                rep->ms_correct = c;
                auto span = [&](int u, int v) -> double {
                    float x = 0;
                    if ((evmask >> u & 1) && (evmask >> v & 1)) cudaEventElapsedTime(&x, ev[u], ev[v]);
                    return x;
                };
                rep->ms_build = span(0, 4);
                rep->ms_filter = span(5, 6);
                rep->ms_rhs = span(7, 8);
                rep->ms_ppe = span(7, 2);
            }
        }
        if (hctl->overflow) return check_overflow();
        return SISPH_OK;
    }

    // ------------------------------------------------------------------ fields
    int ncomp(int f)
    {
        switch (f) {
            case SISPH_FIELD_POSITION:
            case SISPH_FIELD_VELOCITY:
            case SISPH_FIELD_TRANSPORT_VELOCITY:
            case SISPH_FIELD_USTAR:
            case SISPH_FIELD_RSTAR:
            case SISPH_FIELD_NORMAL:
            case SISPH_FIELD_WALL_VELOCITY: return D;
            case SISPH_FIELD_PRESSURE:
            case SISPH_FIELD_DENSITY:
            case SISPH_FIELD_MASS:
            case SISPH_FIELD_RHS:
            case SISPH_FIELD_DIAG:
            case SISPH_FIELD_FREE_SURFACE:
            case SISPH_FIELD_TAG: return 1;
        }
        return -1;
    }

    // owned particles only (slab ranks: the entries of other ranks' particles stay 0)
    int get_field(int f, double* out, int64_t count) override { return get_field_t(f, out, count); }
    int get_field_f32(int f, float* out, int64_t count) override { return get_field_t(f, out, count); }
    int set_field(int f, const double* in, int64_t count) override { return set_field_t(f, in, count); }
    int set_field_f32(int f, const float* in, int64_t count) override { return set_field_t(f, in, count); }

    // H: the host element type of the caller's buffer (double, or float for the _f32 calls)
    template <class H>
    int get_field_t(int f, H* out, int64_t count)
    {
        int nc = ncomp(f);
        if (nc < 0 || count != (int64_t)nc * n) {
            err = "get_field: unknown field or count != n * components";
            return SISPH_EINVAL;
        }
        if (f == SISPH_FIELD_TAG) {
            for (int64_t k = 0; k < n; k++) out[k] = tags_host[k];
            return SISPH_OK;
        }
        SRET(gather_field(f, reinterpret_cast<H*>(dtmp), count));   // device staging (3 n doubles >= count H)
        SCK(cudaMemcpyAsync(out, dtmp, (size_t)count * sizeof(H), cudaMemcpyDefault, st));
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    // sisph_fetch_field: field f gathered on st into fbuf, then copied to `out` on the download
    // stream; the host waits only in fetch_wait
    int fetch_field(int f, void* out, int64_t count, bool f32) override
    {
        int nc = ncomp(f);
        if (nc < 0 || count != (int64_t)nc * n || f == SISPH_FIELD_TAG) {
            err = "fetch_field: unknown field, TAG, or count != n * components";
            return SISPH_EINVAL;
        }
        if (fpending) {
            err = "fetch_field: a fetch is pending (sisph_fetch_wait first)";
            return SISPH_EINVAL;
        }
        const size_t bytes = (size_t)count * (f32 ? sizeof(float) : sizeof(double));
        if (!dlst) SCK(cudaStreamCreateWithFlags(&dlst, cudaStreamNonBlocking));
        if (!ev_fready) SCK(cudaEventCreateWithFlags(&ev_fready, cudaEventDisableTiming));
        if (!ev_fdone) SCK(cudaEventCreateWithFlags(&ev_fdone, cudaEventDisableTiming));
        if (fcap < bytes) {
            SCK(cudaStreamSynchronize(dlst));
            SCK(cudaStreamSynchronize(st));
            if (fbuf) SCK(cudaFree(fbuf));
            fbuf = nullptr;
            fcap = 0;
            SCK(cudaMalloc(&fbuf, bytes));
            fcap = bytes;
        }
        if (fdone_rec) SCK(cudaStreamWaitEvent(st, ev_fdone, 0));   // the last download has read fbuf
        if (f32) SRET(gather_field(f, reinterpret_cast<float*>(fbuf), count));
        else SRET(gather_field(f, reinterpret_cast<double*>(fbuf), count));
        SCK(cudaEventRecord(ev_fready, st));
        SCK(cudaStreamWaitEvent(dlst, ev_fready, 0));
        SCK(cudaMemcpyAsync(out, fbuf, bytes, cudaMemcpyDefault, dlst));
        SCK(cudaEventRecord(ev_fdone, dlst));
        fdone_rec = fpending = true;
        return SISPH_OK;
    }

    int fetch_wait() override
    {
        if (!fpending) return SISPH_OK;
        fpending = false;
        SCK(cudaEventSynchronize(ev_fdone));
        return SISPH_OK;
    }

    // stream-ordered gather of field f into a creation-id-order device buffer (get_field and
    // fetch_field)
    template <class H>
    int gather_field(int f, H* htmp, int64_t count)
    {
        bool mid = phase != IDLE;
        if (f == SISPH_FIELD_RSTAR && !mid) {
            err = "RSTAR is only defined between sisph_predict and sisph_correct";
            return SISPH_EINVAL;
        }
        SCK(cudaMemsetAsync(htmp, 0, (size_t)count * sizeof(H), st));
        const int B = 256;
        auto vec = [&](const V* src, int base, int cntx) {
            if (cntx > 0) ++nlaunch, k_to_ids_vec<T, H><<<nblk(cntx, B), B, 0, st>>>(src + base, pid + base, cntx, D, htmp);
        };
        auto sc = [&](const auto* src, int base, int cntx) {
            if (cntx > 0) ++nlaunch, k_to_ids_sc<<<nblk(cntx, B), B, 0, st>>>(src + base, pid + base, cntx, htmp);
        };
        switch (f) {
            case SISPH_FIELD_POSITION:
                vec(mid ? rn : pos, 0, Nfo);
                vec(pos, Nf, Nwo);
                break;
            case SISPH_FIELD_RSTAR:
                vec(pos, 0, Nfo);
                vec(pos, Nf, Nwo);
                break;
            case SISPH_FIELD_VELOCITY:
                vec(vel, 0, Nfo);
                vec(vel, Nf, Nwo);
                break;
            case SISPH_FIELD_TRANSPORT_VELOCITY: vec(vt, 0, Nfo); break;
            case SISPH_FIELD_USTAR:
                vec(us, 0, Nfo);
                vec(us, Nf, Nwo);
                break;
            case SISPH_FIELD_NORMAL:
                if (Nwo) ++nlaunch, k_to_ids_vec<T, H><<<nblk(Nwo, B), B, 0, st>>>(nrm, pid + Nf, Nwo, D, htmp);
                break;
            case SISPH_FIELD_WALL_VELOCITY:
                if (Nwo) ++nlaunch, k_to_ids_vec<T, H><<<nblk(Nwo, B), B, 0, st>>>(uwl, pid + Nf, Nwo, D, htmp);
                break;
            case SISPH_FIELD_PRESSURE:
                sc(p, 0, Nfo);
                sc(p, Nf, Nwo);
                break;
            case SISPH_FIELD_DENSITY:
                sc(rho, 0, Nfo);
                sc(rho, Nf, Nwo);
                break;
            case SISPH_FIELD_RHS: sc(rhs, 0, Nfo); break;
            case SISPH_FIELD_DIAG: sc(diag, 0, Nfo); break;
            case SISPH_FIELD_FREE_SURFACE: sc(fs, 0, Nfo); break;
            case SISPH_FIELD_MASS:
                if (Nfo) ++nlaunch, k_to_ids_w<T, H><<<nblk(Nfo, B), B, 0, st>>>(pos, pid, Nfo, htmp);
                if (Nwo) ++nlaunch, k_to_ids_w<T, H><<<nblk(Nwo, B), B, 0, st>>>(pos + Nf, pid + Nf, Nwo, htmp);
                break;
        }
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    bool settable(int f, int64_t count)
    {
        int nc = ncomp(f);
        if (nc < 0 || count != (int64_t)nc * n || f == SISPH_FIELD_TAG || f == SISPH_FIELD_RSTAR) {
            err = "set_field: unknown or read-only field, or count != n * components";
            return false;
        }
        return true;
    }

    template <class H>
    int set_field_t(int f, const H* in, int64_t count)
    {
        if (!settable(f, count)) return SISPH_EINVAL;
        SCK(cudaMemcpyAsync(dtmp, in, (size_t)count * sizeof(H), cudaMemcpyDefault, st));
        SRET(scatter_field(f, reinterpret_cast<const H*>(dtmp)));
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    // stream-ordered scatter of a creation-id-order device buffer into field f (set_field and
    // commit_staged)
    template <class H>
    int scatter_field(int f, const H* htmp)
    {
        pre_swept = false;   // the sweep fused into A11 used the old state: the solve redoes it
        const int B = 256;
        auto vec = [&](V* dst, int base, int cntx, int keep_w) {
            if (cntx > 0) ++nlaunch, k_from_ids_vec<T, H><<<nblk(cntx, B), B, 0, st>>>(htmp, pid + base, cntx, D, dst + base, keep_w);
        };
        auto sc = [&](auto* dst, int base, int cntx) {
            using S = std::remove_pointer_t<decltype(dst)>;
            if (cntx > 0) ++nlaunch, k_from_ids_sc<T, S, H><<<nblk(cntx, B), B, 0, st>>>(htmp, pid + base, cntx, dst + base);
        };
        switch (f) {
            case SISPH_FIELD_POSITION: {
                bool mid = phase != IDLE;
                vec(mid ? rn : pos, 0, Nfo, 1);
                if (Nwo) {
                    // wall geometry is static; re-sort walls + normals only if it changed
                    // (compared on the device against the input, in working precision)
                    SCK(cudaMemsetAsync(dcnt_w, 0, sizeof(int), st));
                    ++nlaunch, k_walls_changed<T, H><<<nblk(Nwo, B), B, 0, st>>>(htmp, pid + Nf, Nwo, D, pos + Nf, dcnt_w);
                    int changed = 0;
                    SCK(cudaMemcpyAsync(&changed, dcnt_w, sizeof(int), cudaMemcpyDeviceToHost, st));
                    SCK(cudaStreamSynchronize(st));
                    if (changed) {
                        if (dist()) {
                            err = "set_field: slab ranks keep the wall geometry of sisph_create_dist";
                            return SISPH_EINVAL;
                        }
                        vec(pos, Nf, Nw, 1);
                        SRET(sort_walls(false));
                        SRET(first_build());
                        phase = IDLE;
                    }
                }
            } break;
            case SISPH_FIELD_VELOCITY:
                vec(vel, 0, Nfo, 0);
                vec(vel, Nf, Nwo, 0);
                break;
            case SISPH_FIELD_TRANSPORT_VELOCITY: vec(vt, 0, Nfo, 0); break;
            case SISPH_FIELD_USTAR:
                vec(us, 0, Nfo, 0);
                vec(us, Nf, Nwo, 0);
                break;
            case SISPH_FIELD_NORMAL:
                if (Nwo) ++nlaunch, k_from_ids_vec<T, H><<<nblk(Nwo, B), B, 0, st>>>(htmp, pid + Nf, Nwo, D, nrm, 0);
                break;
            case SISPH_FIELD_WALL_VELOCITY:
                // owned walls (ghost walls take their ghost velocities from the owner's halo)
                if (Nwo) ++nlaunch, k_from_ids_vec<T, H><<<nblk(Nwo, B), B, 0, st>>>(htmp, pid + Nf, Nwo, D, uwl, 0);
                break;
            case SISPH_FIELD_PRESSURE:
                sc(p, 0, Nfo);
                sc(p, Nf, Nwo);
                break;
            case SISPH_FIELD_DENSITY:
                sc(rho, 0, Nfo);
                sc(rho, Nf, Nwo);
                break;
            case SISPH_FIELD_RHS: sc(rhs, 0, Nfo); break;
            case SISPH_FIELD_DIAG: sc(diag, 0, Nfo); break;
            case SISPH_FIELD_FREE_SURFACE: sc(fs, 0, Nfo); break;
            case SISPH_FIELD_MASS:
                if (Nfo) ++nlaunch, k_from_ids_w<T, H><<<nblk(Nfo, B), B, 0, st>>>(htmp, pid, Nfo, pos);
                if (Nwo) ++nlaunch, k_from_ids_w<T, H><<<nblk(Nwo, B), B, 0, st>>>(htmp, pid + Nf, Nwo, pos + Nf);
                break;
        }
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    // sisph_stage_field: the host->device copy of a field's next value runs on the upload stream
    // (after the previous commit's scatters released the buffer) and overlaps whatever the
    // handle's stream is computing; nothing changes until commit_staged
    int stage_field(int f, const void* in, int64_t count, bool f32) override
    {
        if (!settable(f, count)) return SISPH_EINVAL;
        if (f < 0 || f >= NFIELD) return SISPH_EINVAL;
        Staged& g = stg[f];
        if (g.pending) {
            err = "stage_field: the field is already staged (sisph_commit_staged first)";
            return SISPH_EINVAL;
        }
        const size_t bytes = (size_t)count * (f32 ? sizeof(float) : sizeof(double));
        if (!ust) SCK(cudaStreamCreateWithFlags(&ust, cudaStreamNonBlocking));
        if (!ev_consumed) SCK(cudaEventCreateWithFlags(&ev_consumed, cudaEventDisableTiming));
        if (!g.ev) SCK(cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming));
        if (g.cap < bytes) {
            SCK(cudaStreamSynchronize(ust));
            SCK(cudaStreamSynchronize(st));
            if (g.buf) SCK(cudaFree(g.buf));
            g.buf = nullptr;
            g.cap = 0;
            SCK(cudaMalloc(&g.buf, bytes));
            g.cap = bytes;
        }
        if (consumed_rec) SCK(cudaStreamWaitEvent(ust, ev_consumed, 0));
        SCK(cudaMemcpyAsync(g.buf, in, bytes, cudaMemcpyDefault, ust));
        SCK(cudaEventRecord(g.ev, ust));
        g.count = count;
        g.f32 = f32;
        g.pending = true;
        stg_order[nstg++] = f;
        return SISPH_OK;
    }

    // sisph_commit_staged: the handle's stream waits for each staged copy and scatters it, in
    // staging order; stream-ordered (no host wait except POSITION's wall-geometry check)
    int commit_staged() override
    {
        for (int q = 0; q < nstg; q++) {
            Staged& g = stg[stg_order[q]];
            SCK(cudaStreamWaitEvent(st, g.ev, 0));
            int rc = g.f32 ? scatter_field(stg_order[q], reinterpret_cast<const float*>(g.buf))
                           : scatter_field(stg_order[q], reinterpret_cast<const double*>(g.buf));
            g.pending = false;
            if (rc != SISPH_OK) {
                for (int r = q + 1; r < nstg; r++) stg[stg_order[r]].pending = false;
                nstg = 0;
                return rc;
            }
        }
        nstg = 0;
        if (ev_consumed) {
            SCK(cudaEventRecord(ev_consumed, st));
            consumed_rec = true;
        }
        return SISPH_OK;
    }

    int get_field_walls_pos(double* out)
    {
        SCK(cudaMemsetAsync(dtmp, 0, (size_t)n * D * sizeof(double), st));
        if (Nwo) ++nlaunch, k_to_ids_vec<T, double><<<nblk(Nwo, 256), 256, 0, st>>>(pos + Nf, pid + Nf, Nwo, D, dtmp);
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(out, dtmp, (size_t)n * D * sizeof(double), cudaMemcpyDefault, st));
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    // owned slots: fluid [0, Nfo), walls [Nf, Nf + Nwo)
    bool owned_slot(int s) const { return s < Nfo || (s >= Nf && s < Nf + Nwo); }

    int get_order(int64_t* ids) override
    {
        std::vector<int> h(Ntot);
        SCK(cudaMemcpyAsync(h.data(), pid, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        int64_t q = 0;
        for (int s = 0; s < Ntot; s++)
            if (owned_slot(s)) ids[q++] = h[s];
        for (; q < n; q++) ids[q] = -1;
        return SISPH_OK;
    }

    // id -> owned slot (-1: not owned here)
    int slot_map(std::vector<int>& hc, std::vector<int>& hp, std::vector<int>& slot_of)
    {
        hc.resize(Ntot);
        hp.resize(Ntot);
        SCK(cudaMemcpyAsync(hc.data(), cnt, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(hp.data(), pid, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        slot_of.assign(n, -1);
        for (int s = 0; s < Ntot; s++)
            if (owned_slot(s)) slot_of[hp[s]] = s;
        return SISPH_OK;
    }

    int get_neighbors(int64_t* off, int64_t* ids, int64_t cap, int64_t* total) override
    {
        std::vector<int> hc, hp, slot_of;
        SRET(slot_map(hc, hp, slot_of));
        std::vector<int> hn((size_t)P.cap * rows32(Ntot));
        SCK(cudaMemcpyAsync(hn.data(), nbr, hn.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        off[0] = 0;
        for (int64_t k = 0; k < n; k++) off[k + 1] = off[k] + (slot_of[k] >= 0 ? hc[slot_of[k]] : 0);
        *total = off[n];
        if (cap < off[n]) {
            err = "get_neighbors: cap < total";
            return SISPH_EINVAL;
        }
        for (int64_t k = 0; k < n; k++) {
            int s = slot_of[k];
            if (s < 0) continue;
            int64_t* row = ids + off[k];
            // blocked ELL (see sisph_kernels.cuh): (s / 32) 32 cap + (q / 4) 128 + (s % 32) 4 + q % 4
            const size_t b = (size_t)(s >> 5) * ((size_t)P.cap << 5) + ((s & 31) << 2);
            for (int q = 0; q < hc[s]; q++) row[q] = hp[hn[b + ((size_t)(q >> 2) << 7) + (q & 3)]];
            std::sort(row, row + hc[s]);
        }
        return SISPH_OK;
    }

    // rows of the listed particles only (large problems): each row's 16-byte
    // chunks sit 512 bytes apart in the blocked layout -> one 2D copy per row.
    // Particles not owned by this handle get an empty row.
    int get_neighbors_of(const int64_t* which, int64_t m, int64_t* off, int64_t* ids, int64_t cap,
                         int64_t* total) override
    {
        std::vector<int> hc, hp, slot_of;
        SRET(slot_map(hc, hp, slot_of));
        off[0] = 0;
        for (int64_t q = 0; q < m; q++) {
            if (which[q] < 0 || which[q] >= n) {
                err = "get_neighbors_of: id out of range";
                return SISPH_EINVAL;
            }
            const int s = slot_of[which[q]];
            off[q + 1] = off[q] + (s >= 0 ? hc[s] : 0);
        }
        *total = off[m];
        if (cap < off[m]) {
            err = "get_neighbors_of: cap < total";
            return SISPH_EINVAL;
        }
        const int nch = P.cap / 4;
        std::vector<int> rows((size_t)m * P.cap);
        for (int64_t q = 0; q < m; q++) {
            const int s = slot_of[which[q]];
            if (s < 0) continue;
            const size_t b = (size_t)(s >> 5) * ((size_t)P.cap << 5) + ((s & 31) << 2);
            SCK(cudaMemcpy2DAsync(rows.data() + (size_t)q * P.cap, 16, nbr + b, 512, 16, nch, cudaMemcpyDeviceToHost,
                                  st));
        }
        SCK(cudaStreamSynchronize(st));
        for (int64_t q = 0; q < m; q++) {
            const int s = slot_of[which[q]];
            if (s < 0) continue;
            int64_t* row = ids + off[q];
            for (int k = 0; k < hc[s]; k++) row[k] = hp[rows[(size_t)q * P.cap + k]];
            std::sort(row, row + hc[s]);
        }
        return SISPH_OK;
    }

    // adaptive time step of the next step from the maxima the last
    // correct reduced on the device (slab ranks: allreduced)
    int next_dt(double* dtn, double* dtc, double* dtf) override
    {
        if (!stepped) {
            err = "next_dt needs a completed step";
            return SISPH_EINVAL;
        }
        if (dist()) SRET(xallreduce(reinterpret_cast<double*>(&ctl->fmax2_bits), 2, 1));
        SCK(cudaMemcpyAsync(&hctl->fmax2_bits, &ctl->fmax2_bits, 2 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        double f2, v2;
        memcpy(&f2, &hctl->fmax2_bits, sizeof(double));
        memcpy(&v2, &hctl->vmax2_bits, sizeof(double));
        const double hh = (double)P.h;
        const double a = v2 > 0.0 ? 0.25 * hh / sqrt(v2) : INFINITY;
        const double b = f2 > 0.0 ? 0.25 * sqrt(hh / sqrt(f2)) : INFINITY;
        if (dtc) *dtc = a;
        if (dtf) *dtf = b;
        if (dtn) *dtn = a < b ? a : b;
        return SISPH_OK;
    }

    int sweep_timing(double* ms, int* nn) override
    {
        if (ms) *ms = last_ms_sweeps;
        if (nn) *nn = last_sweeps_timed;
        return SISPH_OK;
    }

    int owned_counts(int64_t* nfo, int64_t* nwo) override
    {
        if (nfo) *nfo = Nfo;
        if (nwo) *nwo = Nwo;
        return SISPH_OK;
    }

    int sync() override
    {
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }
};

}  // namespace sb

using namespace sb;

struct sisph {
    EngineBase* e;
};

struct sisph_local_group {
    LocalHub hub;
    explicit sisph_local_group(int n) : hub(n) {}
};

extern "C" void sisph_params_default(sisph_params* p)
{
    if (!p) return;
    memset(p, 0, sizeof(*p));
    p->precision = 64;
    p->rho0 = 1.0;
    p->omega = 0.5;
    p->eta = 0.01;
    p->fs_ratio = 0.8;
    p->h_tilde_factor = 1.0;
    p->K = 10;
    p->min_iter = 2;
    p->max_iter = 1000;
    p->tol = 1e-2;
    p->conv_mean = 1;   // reading R12b
    p->device = -1;
}

static int fail_thread(int code, const std::string& m)
{
    g_thread_err = m;
    return code;
}

static int validate(const double* positions, const double* velocities, const double* masses, const double* densities,
                    const int32_t* tags, int64_t n, double h, const sisph_domain* domain, sisph_params& prm,
                    const sisph_params* params)
{
    if (!positions || !velocities || !masses || !densities || !tags || !domain)
        return fail_thread(SISPH_EINVAL, "NULL input array");
    if (n <= 0 || n > (1ll << 30)) return fail_thread(SISPH_EINVAL, "n must be in [1, 2^30]");
    if (!(h > 0) || !std::isfinite(h)) return fail_thread(SISPH_EINVAL, "h must be finite and > 0");
    int dim = domain->dim;
    if (dim != 2 && dim != 3) return fail_thread(SISPH_EINVAL, "dim must be 2 or 3");
    if (params) prm = *params;
    else sisph_params_default(&prm);
    if (prm.precision != 32 && prm.precision != 64) return fail_thread(SISPH_EINVAL, "precision must be 32 or 64");
    if (!(prm.rho0 > 0)) return fail_thread(SISPH_EINVAL, "rho0 must be > 0");
    if (prm.K < 0 || prm.min_iter < 0 || prm.max_iter < 1) return fail_thread(SISPH_EINVAL, "bad K / iteration bounds");
    for (int a = 0; a < dim; a++) {
        if (!(domain->hi[a] > domain->lo[a]) || !std::isfinite(domain->lo[a]) || !std::isfinite(domain->hi[a]))
            return fail_thread(SISPH_EINVAL, "domain hi must exceed lo on every axis");
        if (domain->periodic[a] && floor((domain->hi[a] - domain->lo[a]) / (3.0 * h)) < 3)
            return fail_thread(SISPH_EINVAL, "a periodic axis needs at least 3 cells of size >= 3h (R26)");
    }
    int64_t nfl = 0;
    for (int64_t k = 0; k < n; k++) {
        if (tags[k] < 0 || tags[k] > (prm.open_x ? 4 : 1))
            return fail_thread(SISPH_EINVAL, "tag must be 0 (fluid) or 1 (wall) (2-4 with open_x)");
        nfl += tags[k] == 0;
        if (!(masses[k] > 0) || !(densities[k] > 0) || !std::isfinite(masses[k]) || !std::isfinite(densities[k]))
            return fail_thread(SISPH_EINVAL, "masses and densities must be finite and > 0");
        for (int a = 0; a < dim; a++) {
            double x = positions[k * dim + a];
            if (!std::isfinite(x) || !std::isfinite(velocities[k * dim + a]))
                return fail_thread(SISPH_EINVAL, "non-finite position or velocity");
            double L = domain->hi[a] - domain->lo[a];
            if (domain->periodic[a]) {
                if (x < domain->lo[a] || x >= domain->hi[a])
                    return fail_thread(SISPH_EINVAL, "position outside a periodic axis' [lo, hi)");
            } else if (x < domain->lo[a] - L || x > domain->hi[a] + L) {
                return fail_thread(SISPH_EINVAL, "position far outside a bounded axis' box");
            }
        }
    }
    if (nfl == 0) return fail_thread(SISPH_EINVAL, "no fluid particle");
    if (prm.open_x && (domain->periodic[0] || !(prm.inlet_length > 0) || !(prm.x_inlet <= prm.x_outlet) ||
                       !(prm.x_outlet <= prm.x_end)))
        return fail_thread(SISPH_EINVAL, "open_x needs a bounded x axis, inlet_length > 0 and x_inlet <= x_outlet <= x_end");
    return SISPH_OK;
}

static EngineBase* new_engine(int prec, int dim)
{
    if (prec == 32) {
        if (dim == 2) return new Engine<float, 2>();
        return new Engine<float, 3>();
    }
    if (dim == 2) return new Engine<double, 2>();
    return new Engine<double, 3>();
}

template <class E>
static int init_as(EngineBase* e, const double* x, const double* u, const double* m, const double* r0,
                   const int32_t* tags, const int64_t* gid, int64_t nloc, int64_t n, const int32_t* tags_glob, double h,
                   const sisph_domain* dom, const sisph_params* prm, const DistInfo* di, const double* slab)
{
    return static_cast<E*>(e)->init(x, u, m, r0, tags, gid, nloc, n, tags_glob, h, dom, prm, di, slab);
}

static int init_engine(EngineBase* e, int prec, int dim, const double* x, const double* u, const double* m,
                       const double* r0, const int32_t* tags, const int64_t* gid, int64_t nloc, int64_t n,
                       const int32_t* tags_glob, double h, const sisph_domain* dom, const sisph_params* prm,
                       const DistInfo* di, const double* slab)
{
    if (prec == 32) {
        if (dim == 2) return init_as<Engine<float, 2>>(e, x, u, m, r0, tags, gid, nloc, n, tags_glob, h, dom, prm, di, slab);
        return init_as<Engine<float, 3>>(e, x, u, m, r0, tags, gid, nloc, n, tags_glob, h, dom, prm, di, slab);
    }
    if (dim == 2) return init_as<Engine<double, 2>>(e, x, u, m, r0, tags, gid, nloc, n, tags_glob, h, dom, prm, di, slab);
    return init_as<Engine<double, 3>>(e, x, u, m, r0, tags, gid, nloc, n, tags_glob, h, dom, prm, di, slab);
}

extern "C" {

int sisph_create(const double* positions, const double* velocities, const double* masses, const double* densities,
                 const int32_t* tags, int64_t n, double h, const sisph_domain* domain, const sisph_params* params,
                 sisph_t** out)
{
    if (!out) return fail_thread(SISPH_EINVAL, "out is NULL");
    *out = nullptr;
    sisph_params prm;
    int rc = validate(positions, velocities, masses, densities, tags, n, h, domain, prm, params);
    if (rc) return rc;
    EngineBase* e = new_engine(prm.precision, domain->dim);
    rc = init_engine(e, prm.precision, domain->dim, positions, velocities, masses, densities, tags, nullptr, n, n, tags,
                     h, domain, &prm, nullptr, nullptr);
    if (rc) {
        g_thread_err = e->err;
        delete e;
        return rc;
    }
    sisph_t* s = new sisph;
    s->e = e;
    *out = s;
    return SISPH_OK;
}

int sisph_nccl_unique_id(const char* nccl_lib, uint8_t id[128])
{
    if (!id) return fail_thread(SISPH_EINVAL, "NULL id");
    std::string err;
    NcclApi& a = nccl_api();
    if (!a.load(nccl_lib, err)) return fail_thread(SISPH_ENCCL, err);
    ncclUniqueId u;
    ncclResult_t r = a.GetUniqueId(&u);
    if (r != ncclSuccess) return fail_thread(SISPH_ENCCL, std::string("ncclGetUniqueId: ") + a.GetErrorString(r));
    memcpy(id, u.internal, 128);
    return SISPH_OK;
}

int sisph_local_group_create(int nranks, sisph_local_group_t** out)
{
    if (!out || nranks < 1) return fail_thread(SISPH_EINVAL, "bad arguments");
    *out = new sisph_local_group(nranks);
    return SISPH_OK;
}

void sisph_local_group_destroy(sisph_local_group_t* g) { delete g; }

int sisph_slab_bounds(const sisph_domain* domain, int axis, int nranks, int rank, double* lo, double* hi)
{
    if (!domain || !lo || !hi || axis < 0 || axis >= domain->dim || nranks < 1 || rank < 0 || rank >= nranks)
        return fail_thread(SISPH_EINVAL, "bad arguments");
    const double a = domain->lo[axis], b = domain->hi[axis], L = b - a;
    *lo = rank == 0 ? a : a + L * rank / nranks;
    *hi = rank == nranks - 1 ? b : a + L * (rank + 1) / nranks;
    return SISPH_OK;
}

int sisph_slab_owner(const sisph_domain* domain, int axis, int nranks, double y)
{
    if (!domain || axis < 0 || axis >= domain->dim || nranks < 1) return -1;
    // the slab whose [lo, hi) holds y; below the box -> first, above -> last
    // (a periodic axis has its inputs inside [lo, hi) already)
    for (int r = 0; r < nranks; r++) {
        double lo, hi;
        sisph_slab_bounds(domain, axis, nranks, r, &lo, &hi);
        if ((r == 0 || y >= lo) && (r == nranks - 1 || y < hi)) return r;
    }
    return nranks - 1;
}

int sisph_create_dist(const double* positions, const double* velocities, const double* masses,
                      const double* densities, const int32_t* tags, int64_t n, double h, const sisph_domain* domain,
                      const sisph_params* params, const sisph_dist* dist, sisph_t** out)
{
    if (!out) return fail_thread(SISPH_EINVAL, "out is NULL");
    *out = nullptr;
    if (!dist) return fail_thread(SISPH_EINVAL, "NULL dist");
    sisph_params prm;
    int rc = validate(positions, velocities, masses, densities, tags, n, h, domain, prm, params);
    if (rc) return rc;
    const int P_ = dist->nranks, r = dist->rank, ax = dist->slab_axis, dim = domain->dim;
    if (P_ < 1 || r < 0 || r >= P_ || ax < 0 || ax >= dim) return fail_thread(SISPH_EINVAL, "bad nranks / rank / slab_axis");
    if (P_ == 1 && !dist->always_slab)
        return sisph_create(positions, velocities, masses, densities, tags, n, h, domain, params, out);
    if (prm.open_x) return fail_thread(SISPH_EINVAL, "open boundaries (open_x) run on a single handle");
    const double L = domain->hi[ax] - domain->lo[ax];
    if (L / P_ < 1.3 * 3.0 * h * 1.01)
        return fail_thread(SISPH_EINVAL, "slabs thinner than the halo width 1.3 x 3h");
    double slab[2];
    sisph_slab_bounds(domain, ax, P_, r, &slab[0], &slab[1]);
    // ownership of the global particles: slab-axis coordinate in [lo, hi) (the
    // first / last slab also own what lies below / above a bounded box)
    std::vector<int64_t> own;
    for (int pass = 0; pass < 2; pass++)   // fluid, then walls
        for (int64_t k = 0; k < n; k++) {
            if ((tags[k] == SISPH_TAG_WALL) != (pass == 1)) continue;
            if (sisph_slab_owner(domain, ax, P_, positions[k * dim + ax]) == r) own.push_back(k);
        }
    const int64_t nl = (int64_t)own.size();
    std::vector<double> x(nl * dim), u(nl * dim), m(nl), r0(nl);
    std::vector<int32_t> tg(nl);
    for (int64_t q = 0; q < nl; q++) {
        const int64_t k = own[q];
        for (int a = 0; a < dim; a++) {
            x[q * dim + a] = positions[k * dim + a];
            u[q * dim + a] = velocities[k * dim + a];
        }
        m[q] = masses[k];
        r0[q] = densities[k];
        tg[q] = tags[k];
    }
    // transport
    DistInfo di;
    di.nranks = P_;
    di.rank = r;
    di.axis = ax;
    Transport* t = nullptr;
    if (dist->local_group) {
        auto* lt = new LocalTransport();
        lt->hub = &dist->local_group->hub;
        if (lt->hub->nranks != P_) {
            delete lt;
            return fail_thread(SISPH_EINVAL, "local group size != nranks");
        }
        t = lt;
    } else {
        if (prm.device >= 0 && cudaSetDevice(prm.device) != cudaSuccess)
            return fail_thread(SISPH_ECUDA, "cudaSetDevice failed");
        auto* nt = new NcclTransport();
        if (nt->init(dist->nccl_lib, dist->nccl_id, P_, r)) {
            std::string m_ = nt->err;
            delete nt;
            return fail_thread(SISPH_ENCCL, m_);
        }
        t = nt;
    }
    t->rank = r;
    t->nranks = P_;
    const bool per = domain->periodic[ax] != 0;
    t->nb[0] = r > 0 ? r - 1 : (per ? P_ - 1 : -1);
    t->nb[1] = r < P_ - 1 ? r + 1 : (per ? 0 : -1);
    di.tp = t;
    EngineBase* e = new_engine(prm.precision, dim);
    rc = init_engine(e, prm.precision, dim, x.data(), u.data(), m.data(), r0.data(), tg.data(), own.data(), nl, n,
                     tags, h, domain, &prm, &di, slab);
    if (rc) {
        g_thread_err = e->err;
        delete e;   // owns the transport once init has taken it
        return rc;
    }
    sisph_t* s = new sisph;
    s->e = e;
    *out = s;
    return SISPH_OK;
}

void sisph_destroy(sisph_t* s)
{
    if (!s) return;
    delete s->e;
    delete s;
}

#define CHK_HANDLE(s)                                                        \
    if (!s) return fail_thread(SISPH_EINVAL, "NULL handle");

int sisph_build_neighbors(sisph_t* s)
{
    CHK_HANDLE(s);
    return s->e->build();
}
int sisph_predict(sisph_t* s, double dt)
{
    CHK_HANDLE(s);
    return s->e->predict(dt);
}
int sisph_ppe_solve(sisph_t* s, double tol, int max_iter, int* iters_out, double* residual_out)
{
    CHK_HANDLE(s);
    return s->e->solve(tol, max_iter, iters_out, residual_out);
}
int sisph_correct(sisph_t* s, double dt)
{
    CHK_HANDLE(s);
    return s->e->correct(dt);
}
int sisph_step(sisph_t* s, double dt, sisph_step_report* rep)
{
    CHK_HANDLE(s);
    return s->e->step(dt, rep);
}
int sisph_get_field(sisph_t* s, sisph_field f, double* out, int64_t count)
{
    CHK_HANDLE(s);
    if (!out) return fail_thread(SISPH_EINVAL, "NULL out");
    return s->e->get_field((int)f, out, count);
}
int sisph_set_field(sisph_t* s, sisph_field f, const double* in, int64_t count)
{
    CHK_HANDLE(s);
    if (!in) return fail_thread(SISPH_EINVAL, "NULL in");
    return s->e->set_field((int)f, in, count);
}
int sisph_get_field_f32(sisph_t* s, sisph_field f, float* out, int64_t count)
{
    CHK_HANDLE(s);
    if (!out) return fail_thread(SISPH_EINVAL, "NULL out");
    return s->e->get_field_f32((int)f, out, count);
}
int sisph_set_field_f32(sisph_t* s, sisph_field f, const float* in, int64_t count)
{
    CHK_HANDLE(s);
    if (!in) return fail_thread(SISPH_EINVAL, "NULL in");
    return s->e->set_field_f32((int)f, in, count);
}
int sisph_stage_field(sisph_t* s, sisph_field f, const double* in, int64_t count)
{
    CHK_HANDLE(s);
    if (!in) return fail_thread(SISPH_EINVAL, "NULL in");
    return s->e->stage_field((int)f, in, count, false);
}
int sisph_stage_field_f32(sisph_t* s, sisph_field f, const float* in, int64_t count)
{
    CHK_HANDLE(s);
    if (!in) return fail_thread(SISPH_EINVAL, "NULL in");
    return s->e->stage_field((int)f, in, count, true);
}
int sisph_commit_staged(sisph_t* s)
{
    CHK_HANDLE(s);
    return s->e->commit_staged();
}
int sisph_fetch_field(sisph_t* s, sisph_field f, double* out, int64_t count)
{
    CHK_HANDLE(s);
    if (!out) return fail_thread(SISPH_EINVAL, "NULL out");
    return s->e->fetch_field((int)f, out, count, false);
}
int sisph_fetch_field_f32(sisph_t* s, sisph_field f, float* out, int64_t count)
{
    CHK_HANDLE(s);
    if (!out) return fail_thread(SISPH_EINVAL, "NULL out");
    return s->e->fetch_field((int)f, out, count, true);
}
int sisph_fetch_wait(sisph_t* s)
{
    CHK_HANDLE(s);
    return s->e->fetch_wait();
}
int sisph_get_order(sisph_t* s, int64_t* ids, int64_t n)
{
    CHK_HANDLE(s);
    if (!ids || n != s->e->n) {
        s->e->err = "get_order: n must equal the particle count";
        return SISPH_EINVAL;
    }
    return s->e->get_order(ids);
}
int sisph_get_neighbors(sisph_t* s, int64_t* offsets, int64_t* ids, int64_t cap, int64_t* total)
{
    CHK_HANDLE(s);
    if (!offsets || !total) return fail_thread(SISPH_EINVAL, "NULL offsets/total");
    return s->e->get_neighbors(offsets, ids, cap, total);
}
int sisph_get_neighbors_of(sisph_t* s, const int64_t* ids_in, int64_t m, int64_t* offsets, int64_t* ids,
                           int64_t cap, int64_t* total)
{
    CHK_HANDLE(s);
    if (!ids_in || m < 0 || !offsets || !total) return fail_thread(SISPH_EINVAL, "NULL or bad argument");
    return s->e->get_neighbors_of(ids_in, m, offsets, ids, cap, total);
}
int sisph_get_counts(const sisph_t* s, int64_t* n, int64_t* n_fluid, int64_t* n_wall)
{
    if (!s) return fail_thread(SISPH_EINVAL, "NULL handle");
    if (n) *n = s->e->n;
    if (n_fluid) *n_fluid = s->e->nf;
    if (n_wall) *n_wall = s->e->nw;
    return SISPH_OK;
}
int sisph_get_owned_counts(sisph_t* s, int64_t* n_fluid, int64_t* n_wall)
{
    CHK_HANDLE(s);
    return s->e->owned_counts(n_fluid, n_wall);
}
int sisph_next_dt(sisph_t* s, double* dt_next, double* dt_cfl, double* dt_force)
{
    CHK_HANDLE(s);
    return s->e->next_dt(dt_next, dt_cfl, dt_force);
}
int sisph_sweep_timing(sisph_t* s, double* ms, int* n)
{
    CHK_HANDLE(s);
    return s->e->sweep_timing(ms, n);
}
int sisph_set_timing(sisph_t* s, int enable)
{
    CHK_HANDLE(s);
    s->e->timing = enable ? 1 : 0;
    return SISPH_OK;
}
int sisph_sync(sisph_t* s)
{
    CHK_HANDLE(s);
    return s->e->sync();
}
const char* sisph_last_error(const sisph_t* s)
{
    if (s) return s->e->err.c_str();
    return g_thread_err.c_str();
}

}  // extern "C"
