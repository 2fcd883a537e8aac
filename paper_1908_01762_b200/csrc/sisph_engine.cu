// sisph_engine.cu — host runtime behind the C ABI of include/sisph.h.
//
// One Engine<T, D> per handle (T = float | double, D = 2 | 3).  It owns the
// device state in cell-sorted structure-of-arrays order (fluid slots [0, Nf),
// static wall slots [Nf, Ntot)), runs every step of the hot path as the
// kernels of sisph_kernels.cuh on one stream, and keeps the PPE stop decision
// on the device (the host only polls a pinned copy of the control block
// between speculative batches of sweeps).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/sisph.h"
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
    virtual int get_order(int64_t* ids) = 0;
    virtual int get_neighbors(int64_t* off, int64_t* ids, int64_t cap, int64_t* total) = 0;
    virtual int get_neighbors_of(const int64_t* which, int64_t m, int64_t* off, int64_t* ids, int64_t cap,
                                 int64_t* total) = 0;
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
    int phase = IDLE;
    int min_iter = 2, max_iter = 1000, K = 10;
    double tol = 1e-2;
    double last_dt = 0;

    // device state
    V *pos = nullptr, *pos_alt = nullptr, *vel = nullptr, *vel_alt = nullptr, *us = nullptr, *us_alt = nullptr;
    V *vt = nullptr, *vt_alt = nullptr, *rn = nullptr, *rstar = nullptr, *nrm = nullptr, *nstmp = nullptr;
    V *rkA = nullptr, *rkB = nullptr, *vk = nullptr, *dk = nullptr;
    T *p = nullptr, *p_alt = nullptr, *rho = nullptr, *rho_alt = nullptr, *rhs = nullptr, *diag = nullptr;
    uint8_t *fs = nullptr, *fs_alt = nullptr;
    int *pid = nullptr, *pid_alt = nullptr;
    int *keys = nullptr, *rank = nullptr, *perm0 = nullptr, *perm = nullptr;
    int *ccount = nullptr, *fstart = nullptr, *wstart = nullptr, *bsum = nullptr;
    int *nbr = nullptr, *cnt = nullptr;
    int *nbr_in = nullptr, *cnt_in = nullptr;  // GTVF inner list (h~ < h)
    // single per-step build (R3): loose list at r^n on the skin geometry PS,
    // walls binned for PS through wperm_s / wstart_s (recomputed when PS's grid changes)
    int *nbs = nullptr, *cnt_s = nullptr;
    int cap_s = 0;
    int *wperm_s = nullptr, *wstart_s = nullptr;
    int wnc_s[3] = {-1, -1, -1};
    Params<T> PS;
    int rebuild_mode = 0;
    int matrix_free = 0;    // 1: the sweep recomputes fac_ij from positions; 0: A11 stores it per pair
    T* coef = nullptr;      // stored per-pair part of fac_ij, blocked-ELL layout of nbr (fluid rows)   // 0: single build + filter when the skin fits, 1: always two exact builds
    bool skin_used = false;
    double skin_radius = 0;
    double extent = 0;      // max |coordinate| of the domain (rounding margin of the skin)
    bool use_inner = false, inner_valid = false;
    int64_t gtvf_fallbacks = 0;
    Ctl* ctl = nullptr;
    Ctl* hctl = nullptr;  // pinned host mirror
    double* partials = nullptr;
    double* dtmp = nullptr;  // staging for get/set (n * 3 doubles)
    std::vector<int> tags_host;  // creation-order tags
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

    ~Engine() override
    {
        void* ptrs[] = {pos, pos_alt, vel, vel_alt, us, us_alt, vt, vt_alt, rn, rstar, nrm, nstmp, rkA, rkB, vk, dk,
                        p, p_alt, rho, rho_alt, rhs, diag, fs, fs_alt, pid, pid_alt, keys, rank, perm0, perm,
                        ccount, fstart, wstart, bsum, nbr, cnt, ctl, partials, dtmp, nbr_in, cnt_in,
                        nbs, cnt_s, wperm_s, wstart_s, coef};
        if (st) cudaStreamSynchronize(st);
        for (void* q : ptrs)
            if (q) cudaFree(q);
        if (hctl) cudaFreeHost(hctl);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : sev)
            if (e) cudaEventDestroy(e);
        if (own_stream && st) cudaStreamDestroy(st);
    }

    // ------------------------------------------------------------------ setup
    int init(const double* x, const double* u, const double* m, const double* r0, const int32_t* tags, int64_t n_,
             double h, const sisph_domain* dom, const sisph_params* prm)
    {
        n = n_;
        dim = D;
        tags_host.assign(tags, tags + n);
        std::vector<int> fid, wid;
        for (int64_t k = 0; k < n; k++) (tags[k] == SISPH_TAG_FLUID ? fid : wid).push_back((int)k);
        Nf = (int)fid.size();
        Nw = (int)wid.size();
        Ntot = Nf + Nw;
        nf = Nf;
        nw = Nw;
        if (prm->device >= 0) SCK(cudaSetDevice(prm->device));
        if (prm->stream) {
            st = (cudaStream_t)prm->stream;
        } else {
            SCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own_stream = true;
        }
        for (auto& e : ev) SCK(cudaEventCreate(&e));
        // ------------------------------------------------ parameters
        memset(&P, 0, sizeof(P));
        P.Nf = Nf;
        P.Nw = Nw;
        P.Ntot = Ntot;
        P.dim = D;
        const double R = 3.0 * h;
        for (int a = 0; a < 3; a++) {
            P.nc[a] = 1;
            P.cell[a] = 1.0;
            P.lo[a] = dom->lo[a];
            P.hi[a] = dom->hi[a];
            P.per[a] = 0;
        }
        for (int a = 0; a < D; a++) {
            double L = dom->hi[a] - dom->lo[a];
            int nc = (int)floor(L / R);
            if (nc < 1) nc = 1;
            if (dom->periodic[a] && nc < 3) {
                err = "periodic axis " + std::to_string(a) + " has fewer than 3 cells of size >= 3h";
                return SISPH_EINVAL;
            }
            P.nc[a] = nc;
            P.cell[a] = L / nc;
            P.per[a] = dom->periodic[a] ? 1 : 0;
            P.Ld[a] = L;
            P.halfLd[a] = 0.5 * L;
            P.Lf[a] = (float)L;
            P.halfLf[a] = (float)(0.5 * L);
            P.L[a] = (T)L;
            P.halfL[a] = (T)(0.5 * L);
        }
        long long nc_tot = (long long)P.nc[0] * P.nc[1] * P.nc[2];
        if (nc_tot > (1ll << 30)) {
            err = "cell grid too large";
            return SISPH_EINVAL;
        }
        ncells = (int)nc_tot;
        P.R2d = R * R;
        P.R2lo = (float)(R * R * (1.0 - 1.0 / 4096.0));
        P.R2hi = (float)(R * R * (1.0 + 1.0 / 4096.0));
        const double sigd = D == 2 ? 7.0 / (478.0 * M_PI) : 1.0 / (120.0 * M_PI);
        auto hd = [&](double hh, T& sig, T& dwk, T& inv) {
            sig = (T)(sigd / pow(hh, D));
            dwk = (T)(-5.0 * sigd / pow(hh, D + 1));
            inv = (T)(1.0 / hh);
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
        rebuild_mode = prm->rebuild_mode;
        matrix_free = prm->matrix_free;
        for (int a = 0; a < D; a++) extent = std::max(extent, std::max(fabs(dom->lo[a]), fabs(dom->hi[a])));
        min_iter = prm->min_iter;
        max_iter = prm->max_iter;
        tol = prm->tol;
        K = prm->K;
        // GTVF inner list: worth it when the GTVF kernel support 3 h~ is well inside 3 h
        {
            const double ht = prm->h_tilde_factor * h, skin = 0.25 * h;
            const double rin = 3.0 * ht + skin;
            use_inner = rin < 0.85 * R && prm->p_ref != 0.0 && prm->K > 0;
            P.Rin2f = (float)(rin * rin * (1.0 + 1.0 / 1024.0));
            P.skin_half2 = (T)(0.25 * skin * skin);
        }
        // ------------------------------------------------ allocation
        int rc = 0;
        size_t NT = (size_t)Ntot, NF = (size_t)std::max(Nf, 1), NW = (size_t)std::max(Nw, 1);
#define AL(ptr, Ty, cntx)                    \
    ptr = dalloc<Ty>((cntx), err, rc);       \
    if (rc) return rc;
        AL(pos, V, NT) AL(pos_alt, V, NT) AL(vel, V, NT) AL(vel_alt, V, NT) AL(us, V, NT) AL(us_alt, V, NT)
        AL(vt, V, NF) AL(vt_alt, V, NF) AL(rn, V, NT) AL(rstar, V, NT) AL(nrm, V, NW) AL(nstmp, V, NW)
        AL(rkA, V, NT) AL(rkB, V, NT) AL(vk, V, NF) AL(dk, V, NF)
        AL(p, T, NT) AL(p_alt, T, NT) AL(rho, T, NT) AL(rho_alt, T, NT) AL(rhs, T, NF) AL(diag, T, NF)
        AL(fs, uint8_t, NF) AL(fs_alt, uint8_t, NF) AL(pid, int, NT) AL(pid_alt, int, NT)
        AL(keys, int, NT) AL(rank, int, NT) AL(perm0, int, NT) AL(perm, int, NT)
        AL(ccount, int, (size_t)ncells + 1) AL(fstart, int, (size_t)ncells + 1) AL(wstart, int, (size_t)ncells + 1)
        AL(bsum, int, (size_t)nblk(ncells + 1, SCAN_B) + 1) AL(cnt, int, NT) AL(ctl, Ctl, 1) AL(cnt_in, int, NF)
        AL(cnt_s, int, NT) AL(wperm_s, int, NW) AL(wstart_s, int, (size_t)ncells + 1)
        AL(partials, double, 2 * (size_t)nblk(Nf, SWEEP_T) + 2) AL(dtmp, double, 3 * (size_t)n)
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
        SCK(cudaMemsetAsync(rhs, 0, NF * sizeof(T), st));
        SCK(cudaMemsetAsync(diag, 0, NF * sizeof(T), st));
        // ------------------------------------------------ upload (fluid ids, then wall ids, ascending)
        std::vector<V> hpos(NT), hvel(NT);
        std::vector<T> hrho(NT);
        std::vector<int> hid(NT);
        for (int s = 0; s < Ntot; s++) {
            int k = s < Nf ? fid[s] : wid[s - Nf];
            hid[s] = k;
            const double* xk = x + (size_t)k * D;
            const double* uk = u + (size_t)k * D;
            hpos[s] = mkh(xk[0], xk[1], D == 3 ? xk[2] : 0.0, m[k]);
            hvel[s] = mkh(uk[0], uk[1], D == 3 ? uk[2] : 0.0, 0.0);
            hrho[s] = (T)r0[k];
        }
        SCK(cudaMemcpyAsync(pos, hpos.data(), NT * sizeof(V), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(vel, hvel.data(), NT * sizeof(V), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(vt, hvel.data(), (size_t)Nf * sizeof(V), cudaMemcpyHostToDevice, st));  // R23
        SCK(cudaMemcpyAsync(rho, hrho.data(), NT * sizeof(T), cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(pid, hid.data(), NT * sizeof(int), cudaMemcpyHostToDevice, st));
        SCK(cudaStreamSynchronize(st));  // host vectors go out of scope
        // identity tails of the permutations (walls are gathered in place)
        if (Nw) {
            ++nlaunch, k_iota<<<nblk(Nw, 256), 256, 0, st>>>(perm + Nf, Nw, Nf);
            SCK(cudaGetLastError());
        }
        // ------------------------------------------------ capacity, walls, first build, normals
        int cap = prm->nbr_cap;
        if (cap <= 0) cap = D == 2 ? 48 : 160;
        cap = (cap + 3) / 4 * 4;   // blocked ELL stores 16-byte chunks of 4 entries
        SRET(alloc_list(cap));
        SRET(setup_walls());
        if (prm->nbr_cap <= 0) {
            // automatic capacity: 1.5 x the largest count of the first build
            SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            SCK(cudaStreamSynchronize(st));
            int mc = hctl->max_count;
            int want = std::max((int)ceil(1.5 * mc) + 8, D == 2 ? 48 : 128);
            want = (want + 7) / 8 * 8;
            if (want != P.cap) {
                SRET(alloc_list(want));
                SRET(setup_walls());
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

    int alloc_list(int cap)
    {
        if (nbr) cudaFree(nbr);
        if (nbr_in) cudaFree(nbr_in);
        if (coef) cudaFree(coef);
        nbr = nbr_in = nullptr;
        coef = nullptr;
        int rc = 0;
        nbr = dalloc<int>((size_t)cap * rows32(Ntot), err, rc);
        if (rc) return rc;
        if (!matrix_free) {
            coef = dalloc<T>((size_t)cap * rows32(Nf), err, rc);
            if (rc) return rc;
        }
        P.cap = cap;
        if (use_inner) {
            // the inner list holds a subset of each fluid row: the full capacity is an upper bound
            P.cap_in = cap;
            nbr_in = dalloc<int>((size_t)cap * rows32(Nf), err, rc);
            if (rc) return rc;
        }
        return SISPH_OK;
    }

    static size_t rows32(int n) { return ((size_t)std::max(n, 1) + 31) / 32 * 32; }

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

    // A1 + A2 + A4: stable counting sort of n particles at xs by cell key;
    // writes start[0..ncells] and perm_out[0..n) (relative slots)
    static int ncells_of(const Params<T>& G) { return G.nc[0] * G.nc[1] * G.nc[2]; }

    int sort_set(const V* xs, int nn, int* start, int* perm_out) { return sort_set(P, xs, nn, start, perm_out); }
    int sort_set(const Params<T>& G, const V* xs, int nn, int* start, int* perm_out)
    {
        const int nc = ncells_of(G);
        SCK(cudaMemsetAsync(ccount, 0, ((size_t)nc + 1) * sizeof(int), st));
        if (nn > 0) {
            ++nlaunch, k_hash_count<T, D><<<nblk(nn, 256), 256, 0, st>>>(G, xs, nn, keys, rank, ccount);
            SCK(cudaGetLastError());
        }
        SRET(scan(ccount, start, nc + 1));
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
        SCK(cudaMemsetAsync(&ctl->max_count, 0, 2 * sizeof(int) + 2 * sizeof(unsigned long long), st));
        const int nc = ncells_of(PS);
        ++nlaunch, k_build_loose<T, D><<<nblk(nc, BL_WARPS), 32 * BL_WARPS, 0, st>>>(
            PS, nc, pos, fstart, wstart_s, Nw ? wperm_s : nullptr, nbs, cnt_s, ctl);
        SCK(cudaGetLastError());
        return SISPH_OK;
    }

    // exact sets at the current positions out of the loose list (+ GTVF inner list)
    int filter_list()
    {
        // keep the overflow flag of the loose build; reset the statistics
        SCK(cudaMemsetAsync(&ctl->max_count, 0, sizeof(int), st));
        SCK(cudaMemsetAsync(&ctl->pairs_fluid, 0, 2 * sizeof(unsigned long long), st));
        int* ni = nbr_in;
        ++nlaunch, k_filter<T, D><<<nblk(Ntot, 128), 128, 0, st>>>(P, pos, nbs, cnt_s, cap_s, nbr, cnt, ni, cnt_in, ctl);
        SCK(cudaGetLastError());
        inner_valid = ni != nullptr;
        return SISPH_OK;
    }

    // Decide whether this step can use the single build: skin s = 2 dt max|u~|
    // (+ a rounding margin); the skin geometry has cells >= 3h + s, at least 3
    // per periodic axis, and 3h + s <= 1.3 * 3h (list capacity).  Sets PS.
    int plan_skin(double dt, bool& ok)
    {
        ok = false;
        skin_used = false;
        skin_radius = 0;
        if (rebuild_mode != 0 || Nf == 0) return SISPH_OK;
        SCK(cudaMemsetAsync(&ctl->umax2_bits, 0, sizeof(unsigned long long), st));
        ++nlaunch, k_max_speed<T, D><<<std::min(nblk(Nf, 256), 148 * 8), 256, 0, st>>>(vt, Nf, ctl);
        SCK(cudaGetLastError());
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
            nbs = dalloc<int>((size_t)want * rows32(Ntot), err, rc);
            if (rc) return rc;
            cap_s = want;
        }
        G.cap = cap_s;
        PS = G;
        // walls binned on the skin grid (static: only when the grid changes)
        if (Nw && (G.nc[0] != wnc_s[0] || G.nc[1] != wnc_s[1] || G.nc[2] != wnc_s[2])) {
            SRET(sort_set(G, pos + Nf, Nw, wstart_s, wperm_s));
            for (int a = 0; a < 3; a++) wnc_s[a] = G.nc[a];
        } else if (!Nw) {
            SCK(cudaMemsetAsync(wstart_s, 0, ((size_t)ncells_of(G) + 1) * sizeof(int), st));
        }
        ok = true;
        skin_used = true;
        skin_radius = Rs;
        return SISPH_OK;
    }

    // walls: stable sort by cell (once, or when wall positions change), wall
    // cell table, copies of the wall positions into every position buffer,
    // then a full build and the normals (A0).
    int setup_walls()
    {
        if (Nw > 0) {
            // relative wall slots go to rank[] (free after the sort): gather through it
            int* wp = rank + Nf;
            SRET(sort_set(pos + Nf, Nw, wstart, wp));
            GatherList G{};
            gl_add(G, pos + Nf, pos_alt + Nf, sizeof(V), Nw);
            gl_add(G, vel + Nf, vel_alt + Nf, sizeof(V), Nw);
            gl_add(G, rho + Nf, rho_alt + Nf, sizeof(T), Nw);
            gl_add(G, pid + Nf, pid_alt + Nf, sizeof(int), Nw);
            gl_add(G, p + Nf, p_alt + Nf, sizeof(T), Nw);
            SRET(gather(G, wp, Nw));
            SCK(cudaMemcpyAsync(pos + Nf, pos_alt + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(vel + Nf, vel_alt + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rho + Nf, rho_alt + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(pid + Nf, pid_alt + Nf, Nw * sizeof(int), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(p + Nf, p_alt + Nf, Nw * sizeof(T), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rkA + Nf, pos + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rkB + Nf, pos + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rn + Nf, pos + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            SCK(cudaMemcpyAsync(rstar + Nf, pos + Nf, Nw * sizeof(V), cudaMemcpyDeviceToDevice, st));
            wnc_s[0] = wnc_s[1] = wnc_s[2] = -1;
        } else {
            SCK(cudaMemsetAsync(wstart, 0, ((size_t)ncells + 1) * sizeof(int), st));
        }
        SRET(build_fluid());
        if (Nw > 0) {
            ++nlaunch, k_normals_raw<T, D><<<nblk(Nw, 128), 128, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, nstmp);
            ++nlaunch, k_normals_smooth<T, D><<<nblk(Nw, 128), 128, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, nstmp, nrm);
            SCK(cudaGetLastError());
        }
        return SISPH_OK;
    }

    // build at the current fluid positions: sort, reorder the carried state,
    // neighbour lists.
    int build_fluid(bool loose = false)
    {
        SRET(sort_set(loose ? PS : P, pos, Nf, fstart, perm));
        GatherList G{};
        gl_add(G, pos, pos_alt, sizeof(V), Nf);
        gl_add(G, vel, vel_alt, sizeof(V), Nf);
        gl_add(G, vt, vt_alt, sizeof(V), Nf);
        gl_add(G, p, p_alt, sizeof(T), Nf);
        gl_add(G, pid, pid_alt, sizeof(int), Nf);
        gl_add(G, rho, rho_alt, sizeof(T), Nf);
        gl_add(G, fs, fs_alt, 1, Nf);
        SRET(gather(G, perm, Nf));
        // wall parts of the alternates
        SRET(copy_walls_to_alt());
        std::swap(pos, pos_alt);
        std::swap(vel, vel_alt);
        std::swap(vt, vt_alt);
        std::swap(p, p_alt);
        std::swap(pid, pid_alt);
        std::swap(rho, rho_alt);
        std::swap(fs, fs_alt);
        return loose ? build_loose() : build_list();
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
        SRET(plan_skin(dt, single));
        // A1-A5 at r^n (single build: the loose list on the skin grid)
        SRET(build_fluid(single));
        const int* nb1 = single ? nbs : nbr;
        const int* cn1 = single ? cnt_s : cnt;
        const int cap1 = single ? cap_s : P.cap;
        // A6 (loose pairs beyond 3h contribute exactly 0: W, dW/dr vanish for q >= 3)
        ++nlaunch, k_density<T, D><<<nblk(Ntot, 256), 256, 0, st>>>(P, pos, nb1, cn1, cap1, rho, fs);
        // A7
        if (Nw) ++nlaunch, k_wall_velocity<T, D><<<nblk(Nw, 256), 256, 0, st>>>(P, pos, nb1, cn1, cap1, nrm, vel, 0);
        // A8
        if (Nf) ++nlaunch, k_forces_predict<T, D><<<nblk(Nf, 128), 128, 0, st>>>(P, (T)dt, pos, vel, vt, rho, nb1, cn1, cap1, us, rstar);
        SCK(cudaGetLastError());
        if (single) {
            // A9 (R3): r* becomes the current position set (walls are in every buffer),
            // r^n is kept as rn; exact sets at r* filtered out of the loose list
            std::swap(pos, rstar);
            std::swap(rn, rstar);
            SRET(filter_list());
        } else {
            // A9: build at r*; carry r^n along as rn
            SRET(sort_set(rstar, Nf, fstart, perm));
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
            SRET(gather(G, perm, Nf));
            SRET(copy_walls_to_alt());
            std::swap(pos, pos_alt);
            std::swap(vel, vel_alt);
            std::swap(vt, vt_alt);
            std::swap(us, us_alt);
            std::swap(rho, rho_alt);
            std::swap(fs, fs_alt);
            std::swap(p, p_alt);
            std::swap(pid, pid_alt);
            SRET(build_list(true));   // + GTVF inner list
        }
        // A10
        if (Nw) ++nlaunch, k_wall_velocity<T, D><<<nblk(Nw, 256), 256, 0, st>>>(P, pos, nbr, cnt, P.cap, nrm, us, P.ustar_noslip ? 0 : 1);
        // A11
        SCK(cudaMemsetAsync(&ctl->lambda_bits, 0, sizeof(unsigned long long), st));
        if (Nf) ++nlaunch, k_rhs_diag<T, D><<<nblk(Nf, 128), 128, 0, st>>>(P, (T)(1.0 / dt), pos, us, rho, fs, nbr, cnt, P.cap, rhs, diag, coef, ctl);
        SCK(cudaGetLastError());
        phase = PREDICTED;
        return SISPH_OK;
    }

    static constexpr int MAXREC = 64;
    cudaEvent_t sev[2 * MAXREC] = {};
    int nrec = 0;
    double last_ms_sweeps = 0;
    int last_sweeps_timed = 0;

    int launch_sweeps(int count, double tl, int mi, int mx)
    {
        for (int c = 0; c < count; c++) {
            if (Nw) ++nlaunch, k_wall_pressure<T, D><<<nblk(Nw, 256), 256, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, p, p_alt, ctl);
            bool rec = timing && nrec < MAXREC;
            if (rec) {
                if (!sev[2 * nrec]) {
                    SCK(cudaEventCreate(&sev[2 * nrec]));
                    SCK(cudaEventCreate(&sev[2 * nrec + 1]));
                }
                SCK(cudaEventRecord(sev[2 * nrec], st));
            }
            if (coef)
                ++nlaunch, k_sweep<T, D, true><<<nblk(Nf, SWEEP_T), SWEEP_T, 0, st>>>(
                               P, pos, rho, rhs, diag, fs, nbr, cnt, P.cap, coef, p, p_alt, ctl, partials, tl, mi, mx);
            else
                ++nlaunch, k_sweep<T, D, false><<<nblk(Nf, SWEEP_T), SWEEP_T, 0, st>>>(
                               P, pos, rho, rhs, diag, fs, nbr, cnt, P.cap, nullptr, p, p_alt, ctl, partials, tl, mi, mx);
            if (rec) {
                SCK(cudaEventRecord(sev[2 * nrec + 1], st));
                nrec++;
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
        SCK(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), st));  // ticket, iter, done, nonfinite
        int launched = 0;
        nrec = 0;
        if (Nf > 0) {
            // speculative batches: sweeps after convergence are no-ops on the device
            int batch = std::min(mx, std::max(mi, 2) + 1);
            for (;;) {
                SRET(launch_sweeps(batch, tl, mi, mx));
                launched += batch;
                SCK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
                SCK(cudaStreamSynchronize(st));
                if (hctl->done || launched >= mx) break;
                batch = std::min(mx - launched, std::min(2 * batch, 32));
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
        last_sweeps_timed = std::min(k, nrec);
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

    // K modified-GTVF sub-steps (A14) from r* = pos; returns the final positions in rK
    int gtvf_substeps(T dtau, bool inner, const V*& rK)
    {
        ++nlaunch, k_gtvf_prep<T><<<nblk(Ntot, 256), 256, 0, st>>>(pos, rho, Ntot, rkA, rkB);
        if (inner) SCK(cudaMemsetAsync(&ctl->gtvf_far, 0, sizeof(int), st));
        const V* src = rkB;
        for (int k = 0; k < K; k++) {
            V* dst = (k & 1) ? rkB : rkA;
            if (inner)
                ++nlaunch, k_gtvf_substep<T, D><<<nblk(Nf, 128), 128, 0, st>>>(P, dtau, src, dst, vk, dk, p, nbr_in, P.cap_in,
                                                                               cnt_in, k == 0, pos, 1, ctl);
            else
                ++nlaunch, k_gtvf_substep<T, D><<<nblk(Nf, 128), 128, 0, st>>>(P, dtau, src, dst, vk, dk, p, nbr, P.cap,
                                                                               cnt, k == 0, pos, 0, ctl);
            src = dst;
        }
        SCK(cudaGetLastError());
        rK = dk;
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
        if (Nw) ++nlaunch, k_wall_pressure<T, D><<<nblk(Nw, 256), 256, 0, st>>>(P, pos, rho, nbr, cnt, P.cap, p, p_alt, nullptr);
        if (Nf) ++nlaunch, k_pgrad_correct<T, D><<<nblk(Nf, 128), 128, 0, st>>>(P, (T)dt, pos, rho, p, us, nbr, cnt, P.cap, vel);
        // A14: K sub-steps (p0 = 0 everywhere when p_ref == 0: the shift is exactly zero)
        const V* rK = nullptr;   // GTVF displacement r^K - r^0 (none when p0 = 0)
        if (P.p_ref != T(0) && K > 0 && Nf) {
            SRET(gtvf_substeps((T)(dt / K), inner_valid, rK));
            if (inner_valid) {
                // the inner list is exact only while no particle moved more than skin/2
                SCK(cudaMemcpyAsync(&hctl->gtvf_far, &ctl->gtvf_far, sizeof(int), cudaMemcpyDeviceToHost, st));
                SCK(cudaStreamSynchronize(st));
                if (hctl->gtvf_far) {
                    gtvf_fallbacks++;
                    SRET(gtvf_substeps((T)(dt / K), false, rK));
                }
            }
        }
        // A15
        if (Nf) ++nlaunch, k_advance<T, D><<<nblk(Nf, 256), 256, 0, st>>>(P, (T)dt, rK, rn, vel, pos, vt);
        SCK(cudaGetLastError());
        phase = IDLE;
        return SISPH_OK;
    }

    int step(double dt, sisph_step_report* rep) override
    {
        int64_t l0 = nlaunch;
        if (timing) SCK(cudaEventRecord(ev[0], st));
        SRET(predict(dt));
        if (timing) SCK(cudaEventRecord(ev[1], st));
        int it = 0;
        double res = 0;
        SRET(solve(tol, max_iter, &it, &res));
        if (timing) SCK(cudaEventRecord(ev[2], st));
        SRET(correct(dt));
        if (timing) SCK(cudaEventRecord(ev[3], st));
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
            if (timing) {
                SCK(cudaEventSynchronize(ev[3]));
                float a, b, c;
                cudaEventElapsedTime(&a, ev[0], ev[1]);
                cudaEventElapsedTime(&b, ev[1], ev[2]);
                cudaEventElapsedTime(&c, ev[2], ev[3]);
                rep->ms_predict = a;
                rep->ms_solve = b;
                rep->ms_correct = c;
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
            case SISPH_FIELD_NORMAL: return D;
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

    int get_field(int f, double* out, int64_t count) override
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
        bool mid = phase != IDLE;
        if (f == SISPH_FIELD_RSTAR && !mid) {
            err = "RSTAR is only defined between sisph_predict and sisph_correct";
            return SISPH_EINVAL;
        }
        SCK(cudaMemsetAsync(dtmp, 0, (size_t)count * sizeof(double), st));
        const int B = 256;
        auto vec = [&](const V* src, int base, int cntx) {
            if (cntx > 0) ++nlaunch, k_to_ids_vec<T><<<nblk(cntx, B), B, 0, st>>>(src + base, pid + base, cntx, D, dtmp);
        };
        auto sc = [&](const auto* src, int base, int cntx) {
            if (cntx > 0) ++nlaunch, k_to_ids_sc<<<nblk(cntx, B), B, 0, st>>>(src + base, pid + base, cntx, dtmp);
        };
        switch (f) {
            case SISPH_FIELD_POSITION:
                vec(mid ? rn - 0 : pos, 0, Nf);
                vec(pos, Nf, Nw);
                break;
            case SISPH_FIELD_RSTAR:
                vec(pos, 0, Ntot);
                break;
            case SISPH_FIELD_VELOCITY: vec(vel, 0, Ntot); break;
            case SISPH_FIELD_TRANSPORT_VELOCITY: vec(vt, 0, Nf); break;
            case SISPH_FIELD_USTAR: vec(us, 0, Ntot); break;
            case SISPH_FIELD_NORMAL:
                if (Nw) ++nlaunch, k_to_ids_vec<T><<<nblk(Nw, B), B, 0, st>>>(nrm, pid + Nf, Nw, D, dtmp);
                break;
            case SISPH_FIELD_PRESSURE: sc(p, 0, Ntot); break;
            case SISPH_FIELD_DENSITY: sc(rho, 0, Ntot); break;
            case SISPH_FIELD_RHS: sc(rhs, 0, Nf); break;
            case SISPH_FIELD_DIAG: sc(diag, 0, Nf); break;
            case SISPH_FIELD_FREE_SURFACE: sc(fs, 0, Nf); break;
            case SISPH_FIELD_MASS:
                if (Ntot) ++nlaunch, k_to_ids_w<T><<<nblk(Ntot, B), B, 0, st>>>(pos, pid, Ntot, dtmp);
                break;
        }
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(out, dtmp, (size_t)count * sizeof(double), cudaMemcpyDefault, st));
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    int set_field(int f, const double* in, int64_t count) override
    {
        int nc = ncomp(f);
        if (nc < 0 || count != (int64_t)nc * n || f == SISPH_FIELD_TAG || f == SISPH_FIELD_RSTAR) {
            err = "set_field: unknown or read-only field, or count != n * components";
            return SISPH_EINVAL;
        }
        SCK(cudaMemcpyAsync(dtmp, in, (size_t)count * sizeof(double), cudaMemcpyDefault, st));
        const int B = 256;
        auto vec = [&](V* dst, int base, int cntx, int keep_w) {
            if (cntx > 0) ++nlaunch, k_from_ids_vec<T><<<nblk(cntx, B), B, 0, st>>>(dtmp, pid + base, cntx, D, dst + base, keep_w);
        };
        auto sc = [&](auto* dst, int base, int cntx) {
            using S = std::remove_pointer_t<decltype(dst)>;
            if (cntx > 0) ++nlaunch, k_from_ids_sc<T, S><<<nblk(cntx, B), B, 0, st>>>(dtmp, pid + base, cntx, dst + base);
        };
        switch (f) {
            case SISPH_FIELD_POSITION: {
                bool mid = phase != IDLE;
                vec(mid ? rn : pos, 0, Nf, 1);
                if (Nw) {
                    // wall geometry is static; re-sort walls + normals only if it changed
                    std::vector<double> oldw((size_t)count);
                    SRET(get_field_walls_pos(oldw.data()));
                    bool changed = false;
                    for (int64_t k = 0; k < n && !changed; k++)
                        if (tags_host[k] == SISPH_TAG_WALL)
                            for (int a = 0; a < D; a++)
                                if ((T)in[k * D + a] != (T)oldw[k * D + a]) changed = true;
                    if (changed) {
                        SCK(cudaMemcpyAsync(dtmp, in, (size_t)count * sizeof(double), cudaMemcpyDefault, st));
                        vec(pos, Nf, Nw, 1);
                        SRET(setup_walls());
                        phase = IDLE;
                    }
                }
            } break;
            case SISPH_FIELD_VELOCITY: vec(vel, 0, Ntot, 0); break;
            case SISPH_FIELD_TRANSPORT_VELOCITY: vec(vt, 0, Nf, 0); break;
            case SISPH_FIELD_USTAR: vec(us, 0, Ntot, 0); break;
            case SISPH_FIELD_NORMAL:
                if (Nw) ++nlaunch, k_from_ids_vec<T><<<nblk(Nw, B), B, 0, st>>>(dtmp, pid + Nf, Nw, D, nrm, 0);
                break;
            case SISPH_FIELD_PRESSURE: sc(p, 0, Ntot); break;
            case SISPH_FIELD_DENSITY: sc(rho, 0, Ntot); break;
            case SISPH_FIELD_RHS: sc(rhs, 0, Nf); break;
            case SISPH_FIELD_DIAG: sc(diag, 0, Nf); break;
            case SISPH_FIELD_FREE_SURFACE: sc(fs, 0, Nf); break;
            case SISPH_FIELD_MASS:
                if (Ntot) ++nlaunch, k_from_ids_w<T><<<nblk(Ntot, B), B, 0, st>>>(dtmp, pid, Ntot, pos);
                break;
        }
        SCK(cudaGetLastError());
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    int get_field_walls_pos(double* out)
    {
        SCK(cudaMemsetAsync(dtmp, 0, (size_t)n * D * sizeof(double), st));
        if (Nw) ++nlaunch, k_to_ids_vec<T><<<nblk(Nw, 256), 256, 0, st>>>(pos + Nf, pid + Nf, Nw, D, dtmp);
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(out, dtmp, (size_t)n * D * sizeof(double), cudaMemcpyDefault, st));
        SCK(cudaStreamSynchronize(st));
        return SISPH_OK;
    }

    int get_order(int64_t* ids) override
    {
        std::vector<int> h(Ntot);
        SCK(cudaMemcpyAsync(h.data(), pid, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        for (int s = 0; s < Ntot; s++) ids[s] = h[s];
        return SISPH_OK;
    }

    int get_neighbors(int64_t* off, int64_t* ids, int64_t cap, int64_t* total) override
    {
        std::vector<int> hc(Ntot), hp(Ntot), hn((size_t)P.cap * rows32(Ntot));
        SCK(cudaMemcpyAsync(hc.data(), cnt, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(hp.data(), pid, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(hn.data(), nbr, hn.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        std::vector<int> slot_of(n);
        for (int s = 0; s < Ntot; s++) slot_of[hp[s]] = s;
        off[0] = 0;
        for (int64_t k = 0; k < n; k++) off[k + 1] = off[k] + hc[slot_of[k]];
        *total = off[n];
        if (cap < off[n]) {
            err = "get_neighbors: cap < total";
            return SISPH_EINVAL;
        }
        for (int64_t k = 0; k < n; k++) {
            int s = slot_of[k];
            int64_t* row = ids + off[k];
            // blocked ELL (see sisph_kernels.cuh): (s / 32) 32 cap + (q / 4) 128 + (s % 32) 4 + q % 4
            const size_t b = (size_t)(s >> 5) * ((size_t)P.cap << 5) + ((s & 31) << 2);
            for (int q = 0; q < hc[s]; q++) row[q] = hp[hn[b + ((size_t)(q >> 2) << 7) + (q & 3)]];
            std::sort(row, row + hc[s]);
        }
        return SISPH_OK;
    }

    // rows of the listed particles only (large problems): each row's 16-byte
    // chunks sit 512 bytes apart in the blocked layout -> one 2D copy per row
    int get_neighbors_of(const int64_t* which, int64_t m, int64_t* off, int64_t* ids, int64_t cap,
                         int64_t* total) override
    {
        std::vector<int> hc(Ntot), hp(Ntot);
        SCK(cudaMemcpyAsync(hc.data(), cnt, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaMemcpyAsync(hp.data(), pid, Ntot * sizeof(int), cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        std::vector<int> slot_of(n);
        for (int s = 0; s < Ntot; s++) slot_of[hp[s]] = s;
        off[0] = 0;
        for (int64_t q = 0; q < m; q++) {
            if (which[q] < 0 || which[q] >= n) {
                err = "get_neighbors_of: id out of range";
                return SISPH_EINVAL;
            }
            off[q + 1] = off[q] + hc[slot_of[which[q]]];
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
            const size_t b = (size_t)(s >> 5) * ((size_t)P.cap << 5) + ((s & 31) << 2);
            SCK(cudaMemcpy2DAsync(rows.data() + (size_t)q * P.cap, 16, nbr + b, 512, 16, nch, cudaMemcpyDeviceToHost,
                                  st));
        }
        SCK(cudaStreamSynchronize(st));
        for (int64_t q = 0; q < m; q++) {
            const int s = slot_of[which[q]];
            int64_t* row = ids + off[q];
            for (int k = 0; k < hc[s]; k++) row[k] = hp[rows[(size_t)q * P.cap + k]];
            std::sort(row, row + hc[s]);
        }
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

extern "C" {

void sisph_params_default(sisph_params* p)
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
    p->device = -1;
}

static int fail_thread(int code, const std::string& m)
{
    g_thread_err = m;
    return code;
}

int sisph_create(const double* positions, const double* velocities, const double* masses, const double* densities,
                 const int32_t* tags, int64_t n, double h, const sisph_domain* domain, const sisph_params* params,
                 sisph_t** out)
{
    if (!out) return fail_thread(SISPH_EINVAL, "out is NULL");
    *out = nullptr;
    if (!positions || !velocities || !masses || !densities || !tags || !domain)
        return fail_thread(SISPH_EINVAL, "NULL input array");
    if (n <= 0 || n > (1ll << 30)) return fail_thread(SISPH_EINVAL, "n must be in [1, 2^30]");
    if (!(h > 0) || !std::isfinite(h)) return fail_thread(SISPH_EINVAL, "h must be finite and > 0");
    int dim = domain->dim;
    if (dim != 2 && dim != 3) return fail_thread(SISPH_EINVAL, "dim must be 2 or 3");
    sisph_params prm;
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
        if (tags[k] != 0 && tags[k] != 1) return fail_thread(SISPH_EINVAL, "tag must be 0 (fluid) or 1 (wall)");
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
    EngineBase* e = nullptr;
    int rc;
    if (prm.precision == 32) {
        if (dim == 2) {
            auto* x = new Engine<float, 2>();
            e = x;
            rc = x->init(positions, velocities, masses, densities, tags, n, h, domain, &prm);
        } else {
            auto* x = new Engine<float, 3>();
            e = x;
            rc = x->init(positions, velocities, masses, densities, tags, n, h, domain, &prm);
        }
    } else {
        if (dim == 2) {
            auto* x = new Engine<double, 2>();
            e = x;
            rc = x->init(positions, velocities, masses, densities, tags, n, h, domain, &prm);
        } else {
            auto* x = new Engine<double, 3>();
            e = x;
            rc = x->init(positions, velocities, masses, densities, tags, n, h, domain, &prm);
        }
    }
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
