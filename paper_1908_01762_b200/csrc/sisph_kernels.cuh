// sisph_kernels.cuh — the hand-written sm_100a kernels of the SISPH per-step
// hot path.  One thread per destination particle for the neighbour passes
// (particles are cell-sorted, so a warp's neighbour rows overlap and the
// gathers hit L1/L2); warp-shuffle + block reductions with a last-block
// finish for the device-wide sums.  Citations: PAPER.md lines (P:a-b) and
// DESIGN.md readings (Rn).
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "sisph_device.cuh"

namespace cg = cooperative_groups;

namespace sb {

// device-side control block of one handle
struct Ctl {
    unsigned int ticket;       // last-block election of the sweep reduction
    int iter;                  // sweeps completed in the current solve
    int done;                  // 1 once eq:convergence holds or max_iter is reached
    int nonfinite;             // a non-finite p^{k+1} was produced
    double residual;           // last value of eq:convergence's left side
    unsigned long long lambda_bits;  // Lambda as ordered bits of a non-negative double
    int max_count;             // largest neighbour count of the last build
    int overflow;              // a row exceeded the list capacity
    unsigned long long pairs_fluid;  // sum of neighbour counts over fluid rows of the last build
    unsigned long long pairs_inner;  // sum of GTVF inner-list counts of the last build
    int gtvf_far;              // a particle moved more than skin/2 during the GTVF sub-steps
    unsigned int gbar;         // arrivals at the persistent PPE kernel's grid barrier (reset per launch)
    unsigned long long umax2_bits;   // max |u~|^2 over fluid (ordered bits of a non-negative double)
    double red[4];             // slab ranks: local (sum |dp|, sum |p|, nonfinite) of a sweep, allreduced
    unsigned long long fmax2_bits;   // max |f^n|^2 of the last correct (adaptive dt)
    unsigned long long vmax2_bits;   // max |u^{n+1}|^2 of the last correct
    int max_count_s;           // largest row of the last loose build (k_build_loose, k_build_loose_m)
    int overflow_s;            // a loose row exceeded the loose capacity
};

// block max of a non-negative double, one atomic per block (every thread of
// the block calls it; blockDim.x a multiple of 32, at most 1024)
__device__ __forceinline__ void warp_max_to(double v, unsigned long long* dst)
{
    __shared__ double sm_max[32];
    v = warp_max(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sm_max[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sm_max[lane] : 0.0;
        v = warp_max(v);
        if (lane == 0 && v > 0.0) atomicMax(dst, (unsigned long long)__double_as_longlong(v));
    }
}

// ===========================================================================
// max |u~_i|^2 over fluid particles: sizes the skin of the single per-step
// build (R3: |r*_ij| <= |r^n_ij| + dt |u~_i| + dt |u~_j|, eq:int:rnp1).
// ===========================================================================
template <class T, int D>
__global__ void __launch_bounds__(256) k_max_speed(const V4<T>* __restrict__ vt, int n, Ctl* ctl)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    for (; i < n; i += gridDim.x * blockDim.x) {
        V4<T> u = ld4(vt + i);
        double a = (double)u.x * u.x + (double)u.y * u.y + (D == 3 ? (double)u.z * u.z : 0.0);
        v = fmax(v, a);
    }
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0 && v > 0.0) atomicMax(&ctl->umax2_bits, (unsigned long long)__double_as_longlong(v));
}

// ===========================================================================
// A1: cell hash + per-cell counts.  rank = arrival order inside the cell
// (made deterministic later by the stable fix-up, A2).  Warp-aggregated:
// lanes with equal keys elect one atomic.
// ===========================================================================
// Slab halos: particles at i >= nown are ghosts; their key is offset by the
// cell count, so a stable sort keeps the owned set first (and both sets
// cell-sorted) and the cell table has 2 x ncells + 1 entries.
template <class T, int D>
__global__ void k_hash_count(Params<T> P, const V4<T>* __restrict__ pos, int n, int nown,
                             int* __restrict__ keys, int* __restrict__ rank, int* __restrict__ ccount)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool act = i < n;
    int key = -1;
    if (act) {
        V4<T> x = ld4(pos + i);
        int c[3];
        cell_of<T, D>(P, x, c);
        key = cell_key(P, c) + (i >= nown ? P.nc[0] * P.nc[1] * P.nc[2] : 0);
        keys[i] = key;
    }
    unsigned mask = __ballot_sync(0xffffffffu, act);
    if (!act) return;
    unsigned peers = __match_any_sync(mask, key);
    int lane = threadIdx.x & 31;
    int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(ccount + key, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    rank[i] = base + __popc(peers & ((1u << lane) - 1u));
}

// ===========================================================================
// exclusive scan of ints (3-phase: per-block scan, scan of block sums,
// add-back).  1024 items per block of 256 threads.
// ===========================================================================
constexpr int SCAN_T = 256, SCAN_IPT = 4, SCAN_B = SCAN_T * SCAN_IPT;

__device__ __forceinline__ int block_excl_scan(int v, int* sm, int& total)
{
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < (blockDim.x >> 5) ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < (blockDim.x >> 5)) sm[lane] = s;
    }
    __syncthreads();
    total = sm[(blockDim.x >> 5) - 1];
    int pre = (w > 0 ? sm[w - 1] : 0) + x - v;
    __syncthreads();
    return pre;
}

__global__ void k_scan_local(const int* __restrict__ in, int* __restrict__ out, int n, int* __restrict__ bsum)
{
    __shared__ int sm[32];
    int base = blockIdx.x * SCAN_B + threadIdx.x * SCAN_IPT;
    int v[SCAN_IPT];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; k++) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    int tot;
    int pre = block_excl_scan(s, sm, tot);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; k++) {
        if (base + k < n) out[base + k] = pre;
        pre += v[k];
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// single block: exclusive scan of nb block sums (loops over chunks)
__global__ void k_scan_sums(int* __restrict__ bsum, int nb)
{
    __shared__ int sm[32];
    int carry = 0;
    for (int c0 = 0; c0 < nb; c0 += blockDim.x) {
        int i = c0 + threadIdx.x;
        int v = i < nb ? bsum[i] : 0;
        int tot;
        int pre = block_excl_scan(v, sm, tot);
        if (i < nb) bsum[i] = pre + carry;
        carry += tot;
    }
}

__global__ void k_scan_add(int* __restrict__ out, int n, const int* __restrict__ bsum)
{
    int base = blockIdx.x * SCAN_B + threadIdx.x * SCAN_IPT;
    int add = bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_IPT; k++)
        if (base + k < n) out[base + k] += add;
}

// ===========================================================================
// A2: counting sort by the full cell key (a single radix pass, radix =
// number of cells), then a stable per-cell fix-up: within a cell, elements
// are re-ranked by their previous slot, so the result equals a stable sort
// of the current order by key (bit-exact with the oracle's counting sort).
// ===========================================================================
__global__ void k_scatter(const int* __restrict__ keys, const int* __restrict__ rank,
                          const int* __restrict__ start, int* __restrict__ perm, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) perm[start[keys[i]] + rank[i]] = i;
}

__global__ void k_stabilize(const int* __restrict__ perm, const int* __restrict__ keys,
                            const int* __restrict__ start, int* __restrict__ perm2, int n)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int o = perm[t];
    int key = keys[o];
    int a = start[key], b = start[key + 1];
    int r = 0;
    for (int u = a; u < b; u++) r += perm[u] < o;
    perm2[a + r] = o;
}

// ===========================================================================
// A3: reorder (gather) of the per-particle state by the permutation.
// ===========================================================================
struct GatherList {
    int nf;
    const void* src[14];
    void* dst[14];
    int size[14];   // element bytes
    int n[14];      // elements to move (fluid only, or fluid + walls with an identity tail)
};

__global__ void k_gather(GatherList G, const int* __restrict__ perm, int n)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int o = perm[t];
#pragma unroll 1
    for (int f = 0; f < G.nf; f++) {
        if (t >= G.n[f]) continue;
        switch (G.size[f]) {
            case 32: {
                const double2* s = (const double2*)G.src[f] + 2 * (size_t)o;
                double2* d = (double2*)G.dst[f] + 2 * (size_t)t;
                d[0] = __ldg(s);
                d[1] = __ldg(s + 1);
            } break;
            case 16: ((float4*)G.dst[f])[t] = __ldg((const float4*)G.src[f] + o); break;
            case 8: ((double*)G.dst[f])[t] = __ldg((const double*)G.src[f] + o); break;
            case 4: ((int*)G.dst[f])[t] = __ldg((const int*)G.src[f] + o); break;
            case 1: ((uint8_t*)G.dst[f])[t] = ((const uint8_t*)G.src[f])[o]; break;
        }
    }
}

// ===========================================================================
// A5: neighbour lists.  Destination i scans the 3^d stencil of its cell; in
// each stencil row the cells (cx-1 .. cx+1) are consecutive keys, so their
// fluid particles form ONE contiguous slot range (likewise the walls').
//
// Storage: blocked ELL.  Rows in groups of 32; inside a group the entries k
// .. k+3 of each row form one 16-byte chunk and the 32 rows' chunks are
// contiguous:
//     index(i, k) = (i / 32) 32 cap + (k / 4) 128 + (i % 32) 4 + k % 4
// (cap a multiple of 4, rows padded to a multiple of 32).  A warp of 32
// consecutive destinations reads 4 entries each with ONE coalesced 512-byte
// int4 load; a builder lane fills its own row's chunks in order, so every
// 16-byte chunk is written by one lane and every 512-byte block by one warp
// (the L2 merges them before write-back: no partial-sector traffic).
// ===========================================================================
#ifdef SISPH_LIST_LDG
#define LDLIST __ldg      // A/B: the default read-only path (lists stay L2-resident on small problems)
#else
#define LDLIST __ldcs
#endif
// List (and stored-coefficient) loads use the streaming cache policy
// (__ldcs: evict-first in L1 and L2): each list is read once per pass and is
// far larger than L2, so it must not evict the gathered per-particle arrays.
__device__ __forceinline__ size_t nb_base(int i, int cap)
{
    return (size_t)(i >> 5) * ((size_t)cap << 5) + (size_t)((i & 31) << 2);
}
// offset of entry k + 1 relative to entry k
__device__ __forceinline__ int nb_adv(int k) { return (k & 3) == 3 ? 125 : 1; }

// for every neighbour j of row i (n entries), in list order
template <class F>
__device__ __forceinline__ void for_nbrs(const int* __restrict__ nbr, int cap, int i, int n, F&& f)
{
    const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, cap));
    for (int c = 0; c < n; c += 4) {
        const int4 v = LDLIST(q + (size_t)(c >> 2) * 32);
        f(v.x);
        if (c + 1 < n) f(v.y);
        if (c + 2 < n) f(v.z);
        if (c + 3 < n) f(v.w);
    }
}

// same, with the index chunks of the next PD chunks in flight (register ring)
template <int PD, class F>
__device__ __forceinline__ void for_nbrs_pf(const int* __restrict__ nbr, int cap, int i, int n, F&& f)
{
    const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, cap));
    int4 r[PD];
#pragma unroll
    for (int k = 0; k < PD; k++) r[k] = 4 * k < n ? LDLIST(q + (size_t)k * 32) : make_int4(0, 0, 0, 0);
    for (int c = 0; c < n; c += 4) {
        const int cn = c + 4 * PD;
        const int4 nx = cn < n ? LDLIST(q + (size_t)(cn >> 2) * 32) : make_int4(0, 0, 0, 0);
        const int4 v = r[0];
        f(v.x);
        if (c + 1 < n) f(v.y);
        if (c + 2 < n) f(v.z);
        if (c + 3 < n) f(v.w);
#pragma unroll
        for (int k = 0; k < PD - 1; k++) r[k] = r[k + 1];
        r[PD - 1] = nx;
    }
}

// for_nbrs_k with the index chunks of the next PD chunks in flight
template <int PD, class F>
__device__ __forceinline__ void for_nbrs_k_pf(const int* __restrict__ nbr, int cap, int i, int n, F&& f)
{
    if constexpr (PD == 0) {
        for_nbrs_k(nbr, cap, i, n, f);
    } else {
        const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, cap));
        int4 r[PD];
#pragma unroll
        for (int k = 0; k < PD; k++) r[k] = 4 * k < n ? LDLIST(q + (size_t)k * 32) : make_int4(0, 0, 0, 0);
        for (int c = 0; c < n; c += 4) {
            const int cn = c + 4 * PD;
            const int4 nx = cn < n ? LDLIST(q + (size_t)(cn >> 2) * 32) : make_int4(0, 0, 0, 0);
            const int4 v = r[0];
            f(v.x, c);
            if (c + 1 < n) f(v.y, c + 1);
            if (c + 2 < n) f(v.z, c + 2);
            if (c + 3 < n) f(v.w, c + 3);
#pragma unroll
            for (int k = 0; k < PD - 1; k++) r[k] = r[k + 1];
            r[PD - 1] = nx;
        }
    }
}
// B200, C5 (us per launch, PD 0 / 1 / 2): A11 1105 / 1100 / 1059, wall velocity 46.7 / 39.3 / 39.5
#ifndef SISPH_RHS_PF
#define SISPH_RHS_PF 2
#endif
#ifndef SISPH_WALLV_PF
#define SISPH_WALLV_PF 1
#endif

// PD = 0: for_nbrs; PD > 0: for_nbrs_pf<PD> (per-pass prefetch switches, tuned by A/B builds)
template <int PD, class F>
__device__ __forceinline__ void for_nbrs_pfx(const int* __restrict__ nbr, int cap, int i, int n, F&& f)
{
    if constexpr (PD == 0) for_nbrs(nbr, cap, i, n, f);
    else for_nbrs_pf<PD>(nbr, cap, i, n, f);
}
// B200, C5 (us per launch, PD 0 / 1 / 2): density 435 / 415 / 430, forces 1350 / 1367 / 1278,
// f_p 513 / 500 / 504, wall pressure 46.7 / 42.9 / 41.4
#ifndef SISPH_DENS_PF
#define SISPH_DENS_PF 1
#endif
#ifndef SISPH_FORCES_PF
#define SISPH_FORCES_PF 2
#endif
#ifndef SISPH_PGRAD_PF
#define SISPH_PGRAD_PF 1
#endif

// same, also passing the entry number k
template <class F>
__device__ __forceinline__ void for_nbrs_k(const int* __restrict__ nbr, int cap, int i, int n, F&& f)
{
    const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, cap));
    for (int c = 0; c < n; c += 4) {
        const int4 v = LDLIST(q + (size_t)(c >> 2) * 32);
        f(v.x, c);
        if (c + 1 < n) f(v.y, c + 1);
        if (c + 2 < n) f(v.z, c + 2);
        if (c + 3 < n) f(v.w, c + 3);
    }
}
__device__ __forceinline__ size_t nb_off(int k) { return ((size_t)(k >> 2) << 7) + (k & 3); }
// store one 4-entry chunk of a per-pair array (16 / 32 bytes, aligned)
__device__ __forceinline__ void st_chunk4(float* p, const float (&f)[4])
{
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
}
__device__ __forceinline__ void st_chunk4(double* p, const double (&f)[4])
{
    reinterpret_cast<double2*>(p)[0] = make_double2(f[0], f[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(f[2], f[3]);
}
// one 4-entry chunk of a per-pair array in the same layout (16 / 32 bytes)
__device__ __forceinline__ void ld_chunk4(const float* p, float (&f)[4])
{
    const float4 v = LDLIST(reinterpret_cast<const float4*>(p));
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
}
__device__ __forceinline__ void ld_chunk4_l1(const float* p, float (&f)[4])
{
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
}
__device__ __forceinline__ void ld_chunk4_s(const float* p, float (&f)[4])
{
    const float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
}
__device__ __forceinline__ void ld_chunk4_s(const double* p, double (&f)[4])
{
    const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
    f[0] = a.x;
    f[1] = a.y;
    f[2] = b.x;
    f[3] = b.y;
}
__device__ __forceinline__ void ld_chunk4_l1(const double* p, double (&f)[4])
{
    const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    f[0] = a.x;
    f[1] = a.y;
    f[2] = b.x;
    f[3] = b.y;
}
__device__ __forceinline__ void ld_chunk4(const double* p, double (&f)[4])
{
    const double2 a = LDLIST(reinterpret_cast<const double2*>(p)), b = LDLIST(reinterpret_cast<const double2*>(p) + 1);
    f[0] = a.x;
    f[1] = a.y;
    f[2] = b.x;
    f[3] = b.y;
}

// a builder lane's append cursor into its row
struct NbCursor {
    int* row;   // nbr + nb_base(i, cap)
    int k;      // entries so far (may exceed cap: overflow is counted, not stored)
    __device__ __forceinline__ void init(int* nbr, int cap, int i)
    {
        row = nbr + nb_base(i, cap);
        k = 0;
    }
    __device__ __forceinline__ void push(bool acc, int j, int cap)
    {
        // entry k sits at (k / 4) 128 + k % 4 = 32 (k & ~3) + (k & 3) ints from the row base;
        // predicated store (no branch: the candidate loop stays straight-line)
        const unsigned off = ((unsigned)(k & ~3) << 5) | (unsigned)(k & 3);
        const int pr = (acc && k < cap) ? 1 : 0;
        asm volatile("{\n\t.reg .pred q;\n\t.reg .b64 a;\n\tsetp.ne.b32 q, %3, 0;\n\t"
                     "mad.wide.u32 a, %1, 4, %0;\n\t@q st.global.b32 [a], %2;\n\t}"
                     :: "l"(row), "r"(off), "r"(j), "r"(pr) : "memory");
        k += acc ? 1 : 0;
    }
};

// an append cursor that collects 4 entries in registers and writes them as one
// 16-byte chunk (the blocked-ELL chunk of its row); flush() writes a partial tail
// chunk (entries past the count are never read)
struct NbCursorV {
    int* row;
    int k;
    int b0, b1, b2, b3;
    __device__ __forceinline__ void init(int* nbr, int cap, int i)
    {
        row = nbr + nb_base(i, cap);
        k = 0;
        b0 = b1 = b2 = b3 = 0;
    }
    __device__ __forceinline__ void push(bool acc, int j, int cap)
    {
        const int s = k & 3;
        b0 = (acc && s == 0) ? j : b0;
        b1 = (acc && s == 1) ? j : b1;
        b2 = (acc && s == 2) ? j : b2;
        b3 = (acc && s == 3) ? j : b3;
        if (acc && s == 3 && k < cap) *reinterpret_cast<int4*>(row + ((k >> 2) << 7)) = make_int4(b0, b1, b2, b3);
        k += acc ? 1 : 0;
    }
    __device__ __forceinline__ void flush(int cap)
    {
        if ((k & 3) != 0 && k < cap) *reinterpret_cast<int4*>(row + ((k >> 2) << 7)) = make_int4(b0, b1, b2, b3);
    }
};

// the same 16-byte append with the entries shifted in (b3 newest): four
// selects per push and no slot compares
struct NbCursorS {
    int* row;
    int k;
    int b0, b1, b2, b3;
    __device__ __forceinline__ void init(int* nbr, int cap, int i)
    {
        row = nbr + nb_base(i, cap);
        k = 0;
        b0 = b1 = b2 = b3 = 0;
    }
    __device__ __forceinline__ void push(bool acc, int j, int cap)
    {
        b0 = acc ? b1 : b0;
        b1 = acc ? b2 : b1;
        b2 = acc ? b3 : b2;
        b3 = acc ? j : b3;
        if (acc && (k & 3) == 3 && k < cap) *reinterpret_cast<int4*>(row + ((k >> 2) << 7)) = make_int4(b0, b1, b2, b3);
        k += acc ? 1 : 0;
    }
    __device__ __forceinline__ void flush(int cap)
    {
        const int s = k & 3;
        if (s != 0 && k < cap) {
            const int4 v = s == 1 ? make_int4(b3, 0, 0, 0) : s == 2 ? make_int4(b2, b3, 0, 0) : make_int4(b1, b2, b3, 0);
            *reinterpret_cast<int4*>(row + ((k >> 2) << 7)) = v;
        }
    }
};

// One warp per cell: the lanes are the cell's destinations; candidates of
// each stencil row are staged 32 at a time in shared memory (with the range's
// periodic image shift applied) and read back as broadcasts, so every lane
// tests the same candidate in lockstep.
//
// Two kernels:
//  * k_build_cells (exact): N(i) = { j != i : r_ij^2 < (3h)^2 } decided as R2
//    prescribes (fp32 prefilter with a rounding-bound band [R2lo, R2hi] decided in fp64 from the
//    unshifted positions with the oracle's minimum-image arithmetic; every
//    pair in fp64 mode), optionally also the GTVF inner list (fluid rows;
//    pairs with r^2 < Rin2f);
//  * k_build_loose: a superset list of every pair with r^2 < Rs2 in working
//    precision (Rs = 3h + skin, inflated), no exact decision: the single
//    per-step build at r^n (R3) whose exact r* sets k_filter extracts.
//    A lane takes up to two destinations (cells of 33..64 particles in one
//    pass over the candidates).
// Walls are static: their slots keep the order of the base geometry, and a
// build on another cell geometry reads them through wperm (wall slots sorted
// by that geometry's key); wperm == nullptr means identity.
constexpr int BL_WARPS = 4;

__device__ __forceinline__ int wslot(const int* __restrict__ wperm, int Nf, int u)
{
    return (wperm && u >= Nf) ? Nf + __ldg(wperm + (u - Nf)) : u;
}

// slot ranges of the 3^d stencil of cell c: lane r < NROW fills row r = (dy, dz)
// with up to 3 ranges for each candidate set (x, y) and the image shift code z
// (2 bits per axis, s + 1 for a shift of s L): entries 0-2 owned fluid, 3-5
// owned walls, 6-8 ghost fluid, 9-11 ghost walls (slab halos: keys + ncells).
// Returns after __syncwarp.
constexpr int RNG_PER_ROW = 12;
template <class T, int D>
__device__ __forceinline__ void stencil_ranges(const Params<T>& P, int c, const int* __restrict__ fstart,
                                               const int* __restrict__ wstart, int4* o12)
{
    constexpr int NROW = D == 3 ? 9 : 3;
    const int lane = threadIdx.x & 31;
    if (lane < NROW) {
        const int NC = P.nc[0] * P.nc[1] * P.nc[2];
        const int c0 = c % P.nc[0], c1 = (c / P.nc[0]) % P.nc[1], c2 = c / (P.nc[0] * P.nc[1]);
        const int dy = lane % 3 - 1, dz = D == 3 ? lane / 3 - 1 : 0;
        int4* o = o12 + RNG_PER_ROW * lane;
        for (int q = 0; q < RNG_PER_ROW; q++) o[q] = make_int4(0, 0, 0, 0);
        int cy = c1 + dy, cz = c2 + dz;
        int code = 1 | (1 << 2) | (1 << 4);
        bool ok = true;
        if (P.per[1]) {
            if (cy < 0) { cy += P.nc[1]; code += (-1) << 2; }        // candidate row is the image below
            else if (cy >= P.nc[1]) { cy -= P.nc[1]; code += 1 << 2; }
        } else ok = ok && cy >= 0 && cy < P.nc[1];
        if (D == 3) {
            if (P.per[2]) {
                if (cz < 0) { cz += P.nc[2]; code += (-1) << 4; }
                else if (cz >= P.nc[2]) { cz -= P.nc[2]; code += 1 << 4; }
            } else ok = ok && cz >= 0 && cz < P.nc[2];
        }
        if (ok) {
            const int row = P.nc[0] * (cy + P.nc[1] * cz);
            const int nset = P.ghosts ? 2 : 1;
            for (int g = 0; g < nset; g++) {
                const int kb = row + g * NC;   // ghost keys are offset by the cell count
                int4* og = o + 6 * g;
                int x0 = c0 - 1, x1 = c0 + 1;
                if (P.per[0] && (x0 < 0 || x1 >= P.nc[0])) {
                    for (int dx = 0; dx < 3; dx++) {
                        int cx = c0 + dx - 1, cd = code;
                        if (cx < 0) { cx += P.nc[0]; cd -= 1; }
                        else if (cx >= P.nc[0]) { cx -= P.nc[0]; cd += 1; }
                        const int key = kb + cx;
                        og[dx] = make_int4(fstart[key], fstart[key + 1], cd, 0);
                        og[3 + dx] = make_int4(P.Nf + wstart[key], P.Nf + wstart[key + 1], cd, 0);
                    }
                } else {
                    x0 = max(x0, 0);
                    x1 = min(x1, P.nc[0] - 1);
                    og[0] = make_int4(fstart[kb + x0], fstart[kb + x1 + 1], code, 0);
                    og[3] = make_int4(P.Nf + wstart[kb + x0], P.Nf + wstart[kb + x1 + 1], code, 0);
                }
            }
        }
    }
    __syncwarp();
}

template <class T>
__device__ __forceinline__ void shift_of(const Params<T>& P, int code, T& sx, T& sy, T& sz)
{
    sx = (T)((code & 3) - 1) * P.L[0];
    sy = (T)(((code >> 2) & 3) - 1) * P.L[1];
    sz = (T)(((code >> 4) & 3) - 1) * P.L[2];
}

// stage candidates [j0, min(j0 + 32, b)) of a range: shifted copy, unshifted
// copy (exact mode only) and slot
template <class T, int D, bool ORIG>
__device__ __forceinline__ void stage32(const V4<T>* __restrict__ pos, const int* __restrict__ wperm, int Nf, int j0,
                                        int b, T sx, T sy, T sz, V4<T>* sm, V4<T>* smo, int* smj)
{
    const int lane = threadIdx.x & 31;
    const int jj = j0 + lane;
    if (jj < b) {
        const int slot = wslot(wperm, Nf, jj);
        V4<T> v = ld4(pos + slot);
        if (ORIG) smo[lane] = v;
        smj[lane] = slot;
        v.x += sx;
        v.y += sy;
        if (D == 3) v.z += sz;
        sm[lane] = v;
    }
    __syncwarp();
}

template <class T, int D>
__global__ void __launch_bounds__(32 * BL_WARPS) k_build_cells(Params<T> P, int ncells, const V4<T>* __restrict__ pos,
                                                              const int* __restrict__ fstart,
                                                              const int* __restrict__ wstart,
                                                              const int* __restrict__ wperm, int* __restrict__ nbr,
                                                              int* __restrict__ cnt, int* __restrict__ nbr_in,
                                                              int* __restrict__ cnt_in, Ctl* ctl)
{
    constexpr int NROW = D == 3 ? 9 : 3;
    constexpr int NRNG = NROW * RNG_PER_ROW;
    __shared__ V4<T> smem[BL_WARPS][32], smemo[BL_WARPS][32];
    __shared__ int smemj[BL_WARPS][32];
    __shared__ int4 rng[BL_WARPS][NRNG];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * BL_WARPS + warp;
    if (c >= ncells) return;
    const int fa = fstart[c], nfc = fstart[c + 1] - fa;
    const int wa = wstart[c], nwc = wstart[c + 1] - wa;
    const int nd = nfc + nwc;
    if (nd == 0) return;
    V4<T>* sm = smem[warp];
    V4<T>* smo = smemo[warp];
    int* smj = smemj[warp];
    stencil_ranges<T, D>(P, c, fstart, wstart, rng[warp]);
    const int Nf = P.Nf, cap = P.cap, cap_in = P.cap_in;
    const int pmask = P.per[0] | (P.per[1] << 1) | (P.per[2] << 2);
    int mmax = 0;
    unsigned sfl = 0, sin_ = 0;
    for (int base = 0; base < nd; base += 32) {
        const int t = base + lane;
        const bool act = t < nd;
        const int i = !act ? -1 : (t < nfc ? fa + t : wslot(wperm, Nf, Nf + wa + (t - nfc)));
        const V4<T> xi = ld4(pos + (act ? i : fa));
        const double xid = (double)xi.x, yid = (double)xi.y, zid = (double)xi.z;
        NbCursor A, B;
        A.init(nbr, cap, act ? i : 0);
        // wall destinations get no inner list
        const bool inner = nbr_in && act && i < Nf;
        B.init(nbr_in ? nbr_in : nbr, cap_in, inner ? i : 0);
        const float Rin2 = inner ? P.Rin2f : -1.f;
#pragma unroll 1
        for (int q = 0; q < NRNG; q++) {
            const int4 ab = rng[warp][q];
            if (ab.x >= ab.y) continue;
            T sx, sy, sz;
            shift_of(P, ab.z, sx, sy, sz);
            for (int j0 = ab.x; j0 < ab.y; j0 += 32) {
                stage32<T, D, true>(pos, wperm, Nf, j0, ab.y, sx, sy, sz, sm, smo, smj);
                const int nn = min(32, ab.y - j0);
                for (int u = 0; u < nn; u++) {
                    const V4<T> xj = sm[u];
                    const int j = smj[u];
                    const float dx = (float)(xi.x - xj.x), dy = (float)(xi.y - xj.y);
                    const float dz = D == 3 ? (float)(xi.z - xj.z) : 0.f;
                    float r2 = dx * dx + dy * dy;
                    if (D == 3) r2 += dz * dz;
                    bool in = r2 < P.R2lo;
                    const bool band = !in && r2 <= P.R2hi;
                    // exact ties (lattices!) are common: the fp64 decision on the unshifted
                    // positions runs inline and predicated, once per candidate for the warp
                    if (__any_sync(0xffffffffu, band)) {
                        const V4<T> o = smo[u];
                        const bool ex = exact_band(xid, yid, zid, (double)o.x, (double)o.y, (double)o.z, P.Ld[0],
                                                   P.Ld[1], P.Ld[2], pmask, D == 3, P.R2d);
                        in = band ? ex : in;
                    }
                    const bool acc = act && in && j != i;
                    A.push(acc, j, cap);
                    B.push(acc && r2 < Rin2, j, cap_in);
                }
                __syncwarp();
            }
        }
        if (act) {
            cnt[i] = min(A.k, cap);
            if (inner) cnt_in[i] = min(B.k, cap_in);
            mmax = max(mmax, max(A.k, inner && B.k > cap_in ? cap + 1 : 0));
            if (i < Nf) {
                sfl += (unsigned)min(A.k, cap);
                sin_ += (unsigned)B.k;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
        sfl += __shfl_xor_sync(0xffffffffu, sfl, o);
        sin_ += __shfl_xor_sync(0xffffffffu, sin_, o);
    }
    if (lane == 0) {
        atomicMax(&ctl->max_count, mmax);
        if (mmax > cap) atomicExch(&ctl->overflow, 1);
        if (sfl) atomicAdd(&ctl->pairs_fluid, (unsigned long long)sfl);
        if (sin_) atomicAdd(&ctl->pairs_inner, (unsigned long long)sin_);
    }
}

// stage one chunk of candidates for the loose build (positions already in
// registers, ok = the lane holds a candidate), keeping only those within
// sqrt(Rc2) of the box [lo, hi] that holds the warp's destinations (order
// preserved): a culled candidate has r^2 >= its box distance^2 >= Rc2 > Rs2
// for every destination, so the loose list is the same set in the same
// order.  Returns the kept count.
template <class T, int D>
__device__ __forceinline__ int cull_compact(V4<T> v, int slot, bool ok, T sx, T sy, T sz, const V4<T>& lo,
                                            const V4<T>& hi, T Rc2, V4<T>* sm, int* smj)
{
    const int lane = threadIdx.x & 31;
    bool keep = false;
    if (ok) {
        v.x += sx;
        v.y += sy;
        if (D == 3) v.z += sz;
        const T bx = max(max(lo.x - v.x, v.x - hi.x), (T)0);
        const T by = max(max(lo.y - v.y, v.y - hi.y), (T)0);
        T d2 = bx * bx + by * by;
        if (D == 3) {
            const T bz = max(max(lo.z - v.z, v.z - hi.z), (T)0);
            d2 += bz * bz;
        }
        keep = d2 < Rc2;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
        const int q = __popc(m & ((1u << lane) - 1u));
        sm[q] = v;
        smj[q] = slot;
    }
    __syncwarp();
    return __popc(m);
}

// loose candidate loop over one staged chunk for DPL destinations per lane
template <class T, int D, int DPL, class Cur>
__device__ __forceinline__ void loose_chunk(const V4<T>* sm, const int* smj, int nn, const V4<T> (&xi)[2],
                                            const int (&i)[2], const bool (&act)[2], Cur (&A)[2], T Rs2, int cap)
{
#pragma unroll 4
    for (int u = 0; u < nn; u++) {
        const V4<T> xj = sm[u];
        const int j = smj[u];
#pragma unroll
        for (int d = 0; d < DPL; d++) {
            const T dx = xi[d].x - xj.x, dy = xi[d].y - xj.y;
            T r2 = dx * dx + dy * dy;
            if (D == 3) {
                const T dz = xi[d].z - xj.z;
                r2 += dz * dz;
            }
            A[d].push(act[d] && r2 < Rs2 && j != i[d], j, cap);
        }
    }
}

#ifndef SISPH_BUILD_CULL
// B200, C5 k_build_loose (profiles/r1_variants.md §11): plain 1766 us; culled 1788 us
// (36 % fewer instructions, the staging load latency exposed); culled + 16-byte
// appends 1642 us (adopted); + next-chunk prefetch 1664 us; shift-in appends 1767 us
#define SISPH_BUILD_CULL 1   // cull staged candidates against the destinations' box
#endif
#ifndef SISPH_BUILD_PF
#define SISPH_BUILD_PF 0     // load the next chunk's candidates while testing this one
#endif
#ifndef SISPH_BUILD_VST
#define SISPH_BUILD_VST 1   // unculled: 1770 -> 2355 us with the register-buffered append; culled: 1788 -> 1642 us
#endif
// 3D only: on C3 (2D, a 3 x 3 stencil, short candidate loops) the loose build takes 192 us with
// the cull and 16-byte appends against 155 us without
template <int D>
struct BlCfg {
    static constexpr bool cull = SISPH_BUILD_CULL && D == 3;
    static constexpr bool vst = SISPH_BUILD_VST != 0 && D == 3;
    using Cur = typename std::conditional<!vst, NbCursor,
                                          typename std::conditional<SISPH_BUILD_VST == 2, NbCursorS, NbCursorV>::type>::type;
};
#ifdef SISPH_BUILD_MINB
#define BL_LOOSE_BOUNDS __launch_bounds__(32 * BL_WARPS, SISPH_BUILD_MINB)
#else
#define BL_LOOSE_BOUNDS __launch_bounds__(32 * BL_WARPS)
#endif
template <class T, int D>
__global__ void BL_LOOSE_BOUNDS k_build_loose(Params<T> P, int ncells, const V4<T>* __restrict__ pos,
                                                              const int* __restrict__ fstart,
                                                              const int* __restrict__ wstart,
                                                              const int* __restrict__ wperm, int* __restrict__ nbr,
                                                              int* __restrict__ cnt, Ctl* ctl)
{
    constexpr int NROW = D == 3 ? 9 : 3;
    constexpr int NRNG = NROW * RNG_PER_ROW;
    __shared__ V4<T> smem[BL_WARPS][32];
    __shared__ int smemj[BL_WARPS][32];
    __shared__ int4 rng[BL_WARPS][NRNG];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * BL_WARPS + warp;
    if (c >= ncells) return;
    const int fa = fstart[c], nfc = fstart[c + 1] - fa;
    const int wa = wstart[c], nwc = wstart[c + 1] - wa;
    const int nd = nfc + nwc;
    if (nd == 0) return;
    V4<T>* sm = smem[warp];
    int* smj = smemj[warp];
    stencil_ranges<T, D>(P, c, fstart, wstart, rng[warp]);
    const int Nf = P.Nf, cap = P.cap;
    const T Rs2 = P.Rs2;
    int mmax = 0;
    for (int base = 0; base < nd; base += 64) {
        const bool two = nd - base > 32;   // warp-uniform
        V4<T> xi[2];
        int i[2];
        bool act[2];
        typename BlCfg<D>::Cur A[2];
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const int t = base + 32 * d + lane;
            act[d] = t < nd;
            i[d] = !act[d] ? -1 : (t < nfc ? fa + t : wslot(wperm, Nf, Nf + wa + (t - nfc)));
            xi[d] = ld4(pos + (act[d] ? i[d] : fa));
            A[d].init(nbr, cap, act[d] ? i[d] : 0);
        }
        if constexpr (BlCfg<D>::cull) {
        // box of this pass's destinations (warp-wide)
        V4<T> lo, hi;
        {
            const T big = (T)3.0e38;
            lo.x = lo.y = lo.z = big;
            hi.x = hi.y = hi.z = -big;
#pragma unroll
            for (int d = 0; d < 2; d++)
                if (act[d]) {
                    lo.x = min(lo.x, xi[d].x); lo.y = min(lo.y, xi[d].y); lo.z = min(lo.z, xi[d].z);
                    hi.x = max(hi.x, xi[d].x); hi.y = max(hi.y, xi[d].y); hi.z = max(hi.z, xi[d].z);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo.x = min(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
                lo.y = min(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
                hi.x = max(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
                hi.y = max(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
                if (D == 3) {
                    lo.z = min(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
                    hi.z = max(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
                }
            }
        }
        // margin over Rs2 for the rounding of the two distance evaluations
        const T Rc2 = Rs2 * (T)(1.0 + 1.0 / 4096.0);
        // flattened walk over the 32-candidate chunks of the stencil ranges; the
        // next chunk's slots and positions are loaded while this one is tested
        int q = -1, j0 = 0, b = 0, code = 0;
        auto advance = [&]() -> bool {
            j0 += 32;
            if (j0 < b) return true;
            while (++q < NRNG) {
                const int4 ab = rng[warp][q];
                if (ab.x < ab.y) {
                    j0 = ab.x;
                    b = ab.y;
                    code = ab.z;
                    return true;
                }
            }
            return false;
        };
        V4<T> vn;
        vn.x = vn.y = vn.z = vn.w = (T)0;
        int sn = 0;
        auto fetch = [&]() {
            if (j0 + lane < b) {
                sn = wslot(wperm, Nf, j0 + lane);
                vn = ld4(pos + sn);
            }
        };
        bool more = advance();
#if SISPH_BUILD_PF
        if (more) fetch();
#endif
#pragma unroll 1
        while (more) {
#if !SISPH_BUILD_PF
            fetch();
#endif
            const V4<T> v0 = vn;
            const int s0 = sn, code0 = code;
            const bool ok0 = j0 + lane < b;
            more = advance();
#if SISPH_BUILD_PF
            if (more) fetch();
#endif
            T sx, sy, sz;
            shift_of(P, code0, sx, sy, sz);
            const int nn = cull_compact<T, D>(v0, s0, ok0, sx, sy, sz, lo, hi, Rc2, sm, smj);
            if (nn == 0) continue;
            if (two)
                loose_chunk<T, D, 2>(sm, smj, nn, xi, i, act, A, Rs2, cap);
            else
                loose_chunk<T, D, 1>(sm, smj, nn, xi, i, act, A, Rs2, cap);
            __syncwarp();
        }
        } else {
#pragma unroll 1
        for (int q = 0; q < NRNG; q++) {
            const int4 ab = rng[warp][q];
            if (ab.x >= ab.y) continue;
            T sx, sy, sz;
            shift_of(P, ab.z, sx, sy, sz);
            for (int j0 = ab.x; j0 < ab.y; j0 += 32) {
                stage32<T, D, false>(pos, wperm, Nf, j0, ab.y, sx, sy, sz, sm, nullptr, smj);
                const int nn = min(32, ab.y - j0);
                if (two)
                    loose_chunk<T, D, 2>(sm, smj, nn, xi, i, act, A, Rs2, cap);
                else
                    loose_chunk<T, D, 1>(sm, smj, nn, xi, i, act, A, Rs2, cap);
                __syncwarp();
            }
        }
        }
#pragma unroll
        for (int d = 0; d < 2; d++) {
            if constexpr (BlCfg<D>::vst) A[d].flush(cap);
            if (act[d]) {
                cnt[i[d]] = min(A[d].k, cap);
                mmax = max(mmax, A[d].k);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
    if (lane == 0) {
        atomicMax(&ctl->max_count_s, mmax);
        if (mmax > cap) atomicExch(&ctl->overflow_s, 1);
    }
}

// ===========================================================================
// k_build_loose_m (round 2): the loose list of k_build_loose, entry for entry
// and in the same order, with the candidate test and the append split.
// k_build_loose tests a candidate and appends it in one step, so every lane
// pays the append (register buffer selects + predicated 16-byte store, ~12
// instructions) for every candidate, accepted or not — ~28 instructions per
// candidate, 1/3 of which are accepted on a lattice.  Here:
//  * the culled candidates are packed densely into a 64-entry shared ring
//    (order kept), and every full 32-candidate chunk is tested by all lanes
//    at once into one 32-bit acceptance mask per destination (~10
//    instructions per candidate: distance, compare, a predicated OR);
//  * after BM_QM chunks (or at the end of the stencil) each lane walks its
//    own masks lowest bit first and appends only the accepted slots (the
//    walk diverges, but every lane's total is about the same row length).
// Same candidates (the box cull), same test expression, same order: the
// list is the one k_build_loose writes.
// ===========================================================================
constexpr int BM_WARPS = 4;
#ifndef SISPH_BM_QM
#define SISPH_BM_QM 16
#endif
constexpr int BM_QM = SISPH_BM_QM;

// acceptance masks of nn staged candidates (ring entries t0 .. t0 + nn - 1, t0 in {0, 32})
// for DPL destinations per lane
template <class T, int D, int DPL, bool FULL>
__device__ __forceinline__ void bm_test(const V4<T>* ring, const int* rslot, int t0, int nn, const V4<T> (&xi)[2],
                                        const int (&i)[2], T Rs2, unsigned (&m)[2])
{
    m[0] = m[1] = 0u;
    auto one = [&](int u) {
        const V4<T> xj = ring[t0 + u];
        const int j = rslot[t0 + u];
#pragma unroll
        for (int d = 0; d < DPL; d++) {
            const T dx = xi[d].x - xj.x, dy = xi[d].y - xj.y;
            T r2 = dx * dx + dy * dy;
            if (D == 3) {
                const T dz = xi[d].z - xj.z;
                r2 += dz * dz;
            }
            if (r2 < Rs2 && j != i[d]) m[d] |= 1u << u;
        }
    };
    if constexpr (FULL) {
#pragma unroll
        for (int u = 0; u < 32; u++) one(u);
    } else {
#pragma unroll 4
        for (int u = 0; u < nn; u++) one(u);
    }
}

// append the accepted slots of masks 0 .. nq - 1 (chunk q's slots in cs[q], lowest bit first)
// to a lane's row at entry k: single entries up to a 4-aligned count, then 16-byte chunks (the
// last one padded; entries past the count are never read).  (Measured on C5 against a
// per-lane list of the non-empty masks, with a branched and a branch-free step to the next
// mask: 1193 / 1290 / 1219 us.)
__device__ __forceinline__ void bm_walk(const unsigned (*msk)[2][32], const int (*cs)[32], int d, int nq, int* row,
                                        int& k, int cap)
{
    const int lane = threadIdx.x & 31;
    int qq = 0;
    unsigned mm = msk[0][d][lane];
    auto next = [&](int& j) -> bool {
        while (mm == 0u) {
            if (++qq >= nq) return false;
            mm = msk[qq][d][lane];
        }
        const int bit = __ffs(mm) - 1;
        mm &= mm - 1u;
        j = cs[qq][bit];
        return true;
    };
    while (k & 3) {
        int j;
        if (!next(j)) return;
        if (k < cap) row[((k >> 2) << 7) + (k & 3)] = j;
        k++;
    }
    while (true) {
        int e0, e1, e2, e3;
        if (!next(e0)) return;
        int ne = 1;
        e1 = e2 = e3 = e0;
        if (next(e1)) {
            ne++;
            if (next(e2)) {
                ne++;
                if (next(e3)) ne++;
            }
        }
        if (k < cap) *reinterpret_cast<int4*>(row + ((k >> 2) << 7)) = make_int4(e0, e1, e2, e3);
        k += ne;
        if (ne < 4) return;
    }
}

template <class T, int D>
__global__ void __launch_bounds__(32 * BM_WARPS) k_build_loose_m(Params<T> P, int ncells, const V4<T>* __restrict__ pos,
                                                                 const int* __restrict__ fstart,
                                                                 const int* __restrict__ wstart,
                                                                 const int* __restrict__ wperm, int* __restrict__ nbr,
                                                                 int* __restrict__ cnt, Ctl* ctl)
{
    constexpr int NROW = D == 3 ? 9 : 3;
    constexpr int NRNG = NROW * RNG_PER_ROW;
    __shared__ V4<T> sring[BM_WARPS][64];
    __shared__ int sslot[BM_WARPS][64];
    __shared__ int4 rng[BM_WARPS][NRNG];
    __shared__ unsigned smsk[BM_WARPS][BM_QM][2][32];
    __shared__ int scs[BM_WARPS][BM_QM][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * BM_WARPS + warp;
    if (c >= ncells) return;
    const int fa = fstart[c], nfc = fstart[c + 1] - fa;
    const int wa = wstart[c], nwc = wstart[c + 1] - wa;
    const int nd = nfc + nwc;
    if (nd == 0) return;
    V4<T>* ring = sring[warp];
    int* rslot = sslot[warp];
    unsigned (*msk)[2][32] = smsk[warp];
    int (*cs)[32] = scs[warp];
    stencil_ranges<T, D>(P, c, fstart, wstart, rng[warp]);
    // the non-empty ranges, in order, compacted in place
    int nr = 0;
    for (int q0 = 0; q0 < NRNG; q0 += 32) {
        const int q = q0 + lane;
        const int4 ab = q < NRNG ? rng[warp][q] : make_int4(0, 0, 0, 0);
        const bool ne = ab.x < ab.y;
        const unsigned m = __ballot_sync(0xffffffffu, ne);   // every lane has read its entry
        if (ne) rng[warp][nr + __popc(m & ((1u << lane) - 1u))] = ab;
        nr += __popc(m);
        __syncwarp();
    }
    const int Nf = P.Nf, cap = P.cap;
    const T Rs2 = P.Rs2;
    int mmax = 0;
    for (int base = 0; base < nd; base += 64) {
        const bool two = nd - base > 32;   // warp-uniform
        V4<T> xi[2];
        int i[2], k[2];
        int* row[2];
        bool act[2];
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const int t = base + 32 * d + lane;
            act[d] = t < nd;
            i[d] = !act[d] ? -1 : (t < nfc ? fa + t : wslot(wperm, Nf, Nf + wa + (t - nfc)));
            xi[d] = ld4(pos + (act[d] ? i[d] : fa));
            row[d] = nbr + nb_base(act[d] ? i[d] : 0, cap);
            k[d] = 0;
        }
        // box of this pass's destinations (warp-wide), as k_build_loose
        V4<T> lo, hi;
        {
            const T big = (T)3.0e38;
            lo.x = lo.y = lo.z = big;
            hi.x = hi.y = hi.z = -big;
#pragma unroll
            for (int d = 0; d < 2; d++)
                if (act[d]) {
                    lo.x = min(lo.x, xi[d].x); lo.y = min(lo.y, xi[d].y); lo.z = min(lo.z, xi[d].z);
                    hi.x = max(hi.x, xi[d].x); hi.y = max(hi.y, xi[d].y); hi.z = max(hi.z, xi[d].z);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo.x = min(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
                lo.y = min(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
                hi.x = max(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
                hi.y = max(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
                if (D == 3) {
                    lo.z = min(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
                    hi.z = max(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
                }
            }
        }
        const T Rc2 = Rs2 * (T)(1.0 + 1.0 / 4096.0);
        auto emit = [&](int nq) {
            if (act[0]) bm_walk(msk, cs, 0, nq, row[0], k[0], cap);
            if (act[1]) bm_walk(msk, cs, 1, nq, row[1], k[1], cap);
            __syncwarp();
        };
        // test the 32 (at the end: nn) staged candidates at ring offset t0 as chunk qn (a last
        // chunk padded to 32 far-away candidates: 1231 us against 1193)
        auto test = [&](int t0, int nn, int qn) {
            unsigned m[2];
            if (nn == 32) {
                if (two) bm_test<T, D, 2, true>(ring, rslot, t0, 32, xi, i, Rs2, m);
                else bm_test<T, D, 1, true>(ring, rslot, t0, 32, xi, i, Rs2, m);
            } else {
                if (two) bm_test<T, D, 2, false>(ring, rslot, t0, nn, xi, i, Rs2, m);
                else bm_test<T, D, 1, false>(ring, rslot, t0, nn, xi, i, Rs2, m);
            }
            msk[qn][0][lane] = m[0];
            msk[qn][1][lane] = m[1];
            cs[qn][lane] = lane < nn ? rslot[t0 + lane] : 0;
            __syncwarp();
        };
        int head = 0, tail = 0, nq = 0;
        // (a flattened walk that loads the next chunk while this one is tested: 1237 us against 1193)
#pragma unroll 1
        for (int r = 0; r < nr; r++) {
            const int4 ab = rng[warp][r];
            V4<T> sh;
            shift_of(P, ab.z, sh.x, sh.y, sh.z);
#pragma unroll 1
            for (int j0 = ab.x; j0 < ab.y; j0 += 32) {
                V4<T> v;
                v.x = v.y = v.z = v.w = (T)0;
                int slot = 0;
                const bool ok = j0 + lane < ab.y;
                bool keep = false;
                if (ok) {
                    slot = wslot(wperm, Nf, j0 + lane);
                    v = ld4(pos + slot);
                    // cull against the box (cull_compact's test) into the ring, order kept
                    v.x += sh.x;
                    v.y += sh.y;
                    if (D == 3) v.z += sh.z;
                    const T bx = max(max(lo.x - v.x, v.x - hi.x), (T)0);
                    const T by = max(max(lo.y - v.y, v.y - hi.y), (T)0);
                    T d2 = bx * bx + by * by;
                    if (D == 3) {
                        const T bz = max(max(lo.z - v.z, v.z - hi.z), (T)0);
                        d2 += bz * bz;
                    }
                    keep = d2 < Rc2;
                }
                const unsigned km = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int at = (head + __popc(km & ((1u << lane) - 1u))) & 63;
                    ring[at] = v;
                    rslot[at] = slot;
                }
                head += __popc(km);
                __syncwarp();
                if (head - tail >= 32) {
                    test(tail & 63, 32, nq);
                    tail += 32;
                    if (++nq == BM_QM) {
                        emit(nq);
                        nq = 0;
                    }
                }
            }
        }
        if (head > tail) {
            test(tail & 63, head - tail, nq);
            nq++;
        }
        if (nq) emit(nq);
#pragma unroll
        for (int d = 0; d < 2; d++)
            if (act[d]) {
                cnt[i[d]] = min(k[d], cap);
                mmax = max(mmax, k[d]);
            }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
    if (lane == 0) {
        atomicMax(&ctl->max_count_s, mmax);
        if (mmax > cap) atomicExch(&ctl->overflow_s, 1);
    }
}

// r* = r^n + dt u~^n (eq:int:rnp1) of the slots [0, n): known at the start of the step, so the
// single per-step build takes the r* sets before the stage-1 passes (same expression as
// forces_finish, bit-identical r*)
template <class T, int D>
__global__ void k_rstar(Params<T> P, T dt, int n, const V4<T>* __restrict__ pos, const V4<T>* __restrict__ vt,
                        V4<T>* __restrict__ rstar)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V4<T> xi = ld4(pos + i), uti = ld4(vt + i);
    T rx = xi.x + dt * uti.x, ry = xi.y + dt * uti.y, rz = D == 3 ? xi.z + dt * uti.z : xi.z;
    if (P.per[0]) { if (rx >= P.hi[0]) rx -= P.L[0]; else if (rx < P.lo[0]) rx += P.L[0]; }
    if (P.per[1]) { if (ry >= P.hi[1]) ry -= P.L[1]; else if (ry < P.lo[1]) ry += P.L[1]; }
    if (D == 3 && P.per[2]) { if (rz >= P.hi[2]) rz -= P.L[2]; else if (rz < P.lo[2]) rz += P.L[2]; }
    rstar[i] = mk4<T>(rx, ry, rz, xi.w);
}

// ===========================================================================
// A9 (single-build form, R3): the exact neighbour sets at r* filtered out of
// the loose list built at r^n.  Every pair with |r*_ij| < 3h has
// |r^n_ij| < 3h + dt|u~_i| + dt|u~_j| <= Rs, so it is in the loose list; the
// decision itself is R2's (fp32 prefilter + fp64 band, as the exact build).
// r* = r^n + dt u~^n is known at the start of the step (eq:int:rnp1, k_rstar),
// so the filter runs right after the build.  The filtered rows keep the loose
// list's order (deterministic; band cases last); also writes the GTVF inner
// list of fluid rows.  The warp walks to its longest row so that the fp64
// band decision can be taken warp-wide.
// ===========================================================================
#ifdef SISPH_FILTER_MINB
#define FILTER_BOUNDS __launch_bounds__(128, SISPH_FILTER_MINB)
#else
#define FILTER_BOUNDS __launch_bounds__(128)
#endif
#ifndef SISPH_FILTER_PF
#define SISPH_FILTER_PF 1   // B200, C5: PD 1 / 2 / 3 -> 1214 / 1204 / 1201 us
#endif
// INNER: the GTVF inner list is written too (h~ well inside h); without it the instance has no
// second append in the entry loop
template <class T, int D, bool INNER = true>
__global__ void FILTER_BOUNDS k_filter(Params<T> P, int nrows, const V4<T>* __restrict__ pos,
                                       const int* __restrict__ nbs, const int* __restrict__ cnts, int cap_s,
                                       int* __restrict__ nbr, int* __restrict__ cnt, int* __restrict__ nbr_in,
                                       int* __restrict__ cnt_in, Ctl* ctl)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int Nf = P.Nf, cap = P.cap, cap_in = P.cap_in;
    // every owned row: fluid [0, Nfo), then walls [Nf, Nf + Nwo)
    const bool act = t < nrows;
    const int i = !act ? 0 : (t < P.Nfo ? t : Nf + (t - P.Nfo));
    const bool inner = act && nbr_in && i < Nf;
    const V4<T> xi = ld4(pos + i);
    const int n = act ? cnts[i] : 0;
    int nmax = n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    const float Rin2 = inner ? P.Rin2f : -1.f;
    // fp32 band cases (|r^2 - R^2| within the prefilter's rounding bound, R37: lattice
    // near-ties) are queued per lane and decided in fp64 after the row, so the warp runs the
    // fp64 path max-over-lanes times instead of once per entry any lane has in the band; they
    // are appended after the row's other entries (the set is the same).  Band pairs lie at
    // ~3h, beyond every inner-list radius (3 h~ + 0.1 h <= 0.85 x 3h).
    constexpr int FQ = 48;
    __shared__ int bq[FQ][128];
    int nq = 0;
    const int pmask = P.per[0] | (P.per[1] << 1) | (P.per[2] << 2);
    NbCursorV A, B;
    A.init(nbr, cap, i);
    B.init(nbr_in ? nbr_in : nbr, cap_in, inner ? i : 0);
    const int4* __restrict__ src = reinterpret_cast<const int4*>(nbs + nb_base(i, cap_s));
    // the index chunks of the next SISPH_FILTER_PF chunks stay in flight while one is tested
    int4 vr[SISPH_FILTER_PF];
#pragma unroll
    for (int q = 0; q < SISPH_FILTER_PF; q++) vr[q] = 4 * q < n ? LDLIST(src + (size_t)q * 32) : make_int4(i, i, i, i);
    // one 4-entry chunk of the row: entries e < nv are valid (B200, C5: 1164 -> 1129 us against the
    // same body inline in the chunk loop)
    auto chunk = [&](const int4 v, int nv) {
        const int c = 0;
        const int n = nv;
        // the queue can take this chunk's band cases on every lane: no fp64 decision inside it
        const bool roomy = __all_sync(0xffffffffu, nq <= FQ - 4);
        V4<T> xj4[4];
        int j4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; e++) xj4[e] = ld4(pos + (c + e < n ? j4[e] : i));
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const bool valid = c + e < n;
            const int j = j4[e];
            const V4<T> xj = xj4[e];
            float r2;
            bool in;
            if constexpr (std::is_same<T, float>::value) {
                float d0 = xi.x - xj.x, d1 = xi.y - xj.y, d2 = D == 3 ? xi.z - xj.z : 0.f;
                if (P.per[0]) d0 = wrapd(d0, P.Lf[0], P.halfLf[0]);
                if (P.per[1]) d1 = wrapd(d1, P.Lf[1], P.halfLf[1]);
                if (D == 3 && P.per[2]) d2 = wrapd(d2, P.Lf[2], P.halfLf[2]);
                r2 = d0 * d0 + d1 * d1;
                if (D == 3) r2 += d2 * d2;
                in = r2 < P.R2lo;
                const bool band = valid && !in && r2 <= P.R2hi;
                const bool queued = band && nq < FQ;
                if (queued) bq[nq++][threadIdx.x] = j;
                const bool now = band && !queued;   // queue full: decide here
                if (!roomy && __any_sync(0xffffffffu, now)) {
                    const bool ex = exact_band((double)xi.x, (double)xi.y, (double)xi.z, (double)xj.x, (double)xj.y,
                                               (double)xj.z, P.Ld[0], P.Ld[1], P.Ld[2], pmask, D == 3, P.R2d);
                    in = now ? ex : in;
                }
            } else {
                in = nb_test<D>(P, xi, xj, r2);
            }
            in = in && valid;
            A.push(in, j, cap);
            if constexpr (INNER) B.push(in && r2 < Rin2, j, cap_in);
        }
    };
    for (int c = 0; c < nmax; c += 4) {
        const int4 v = vr[0];
        {
            const int cn = c + 4 * SISPH_FILTER_PF;
            const int4 nx = cn < n ? LDLIST(src + (size_t)(cn >> 2) * 32) : make_int4(i, i, i, i);
#pragma unroll
            for (int q = 0; q < SISPH_FILTER_PF - 1; q++) vr[q] = vr[q + 1];
            vr[SISPH_FILTER_PF - 1] = nx;
        }
        chunk(v, n - c);
    }
    // the queued band cases, in fp64 (R2)
    for (int q = 0; q < nq; q++) {
        const int j = bq[q][threadIdx.x];
        const V4<T> xj = ld4(pos + j);
        const bool ex = exact_band((double)xi.x, (double)xi.y, (double)xi.z, (double)xj.x, (double)xj.y, (double)xj.z,
                                   P.Ld[0], P.Ld[1], P.Ld[2], pmask, D == 3, P.R2d);
        A.push(ex, j, cap);
    }
    A.flush(cap);
    if (INNER) B.flush(cap_in);
    if (act) {
        cnt[i] = min(A.k, cap);
        if (INNER && inner) cnt_in[i] = min(B.k, cap_in);
    }
    int mmax = act ? max(A.k, INNER && inner && B.k > cap_in ? cap + 1 : 0) : 0;
    unsigned sfl = act && i < Nf ? (unsigned)min(A.k, cap) : 0u, sin_ = INNER && inner ? (unsigned)B.k : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
        sfl += __shfl_xor_sync(0xffffffffu, sfl, o);
        sin_ += __shfl_xor_sync(0xffffffffu, sin_, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&ctl->max_count, mmax);
        if (mmax > cap) atomicExch(&ctl->overflow, 1);
        if (sfl) atomicAdd(&ctl->pairs_fluid, (unsigned long long)sfl);
        if (sin_) atomicAdd(&ctl->pairs_inner, (unsigned long long)sin_);
    }
}

// ===========================================================================
// Joint per-particle records for the pair passes: rec[i] = {a[i], b[i]} (8 working-
// precision values), so that a neighbour's position + mass and velocity + density
// arrive with ONE 256-bit gather instead of two 128-bit ones from two arrays (the
// pair passes are bound by L1 requests).  A8 reads {r^n, m, u, rho}
// (packed after A7), A11 reads {r*, m, u*, rho} (packed after A10).
// ===========================================================================
template <class T>
__global__ void k_pack_rec(const V4<T>* __restrict__ a, const V4<T>* __restrict__ b, int n, T* __restrict__ rec)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V4<T> x = ld4(a + i), u = ld4(b + i);
    const T r[8] = {x.x, x.y, x.z, x.w, u.x, u.y, u.z, u.w};
    st8(rec + 8 * (size_t)i, r);
}

// ===========================================================================
// A6: summation density, eq:summation_density, self included;
// walls keep rho0 unless wall_rho_summation (R4).  Free surface flag
// rho_i / rho0 < 0.8 for fluid.
// ===========================================================================
template <class T, int D>
__global__ void __launch_bounds__(256) k_density(Params<T> P, const V4<T>* __restrict__ pos,
                                                 const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap,
                                                 T* __restrict__ rho, uint8_t* __restrict__ fs,
                                                 V4<T>* __restrict__ vel)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.Ntot || (i >= P.Nfo && i < P.Nf) || i >= P.Nf + P.Nwo) return;   // owned rows
    V4<T> xi = ld4(pos + i);
    if (i >= P.Nf && !P.wall_rho_summation) {
        rho[i] = P.rho0;
        return;
    }
    T s = 0;
    int n = cnt[i];
    for_nbrs_pfx<SISPH_DENS_PF>(nbr, ncap, i, n, [&](int j) {
        V4<T> xj = ld4(pos + j);
        T d[3], r, ri;
        r_of(pair_vec<T, D>(P, xi, xj, d), r, ri);
        s += xj.w * quintic5(r * P.inv_h);           // W = 0 exactly beyond 3h (loose-list pairs)
    });
    s = xi.w * P.w0 + P.sig * s;
    rho[i] = s;
    if (i < P.Nf) {
        const int ty = P.ptype ? P.ptype[i] : 0;
        // fs: 1 free surface (fluid only, R11); 2 outlet row (R34: p frozen, not a PPE unknown)
        fs[i] = ty == 3 ? 2 : (ty == 0 && s / P.rho0 < P.fs_ratio ? 1 : 0);
        // rho_i rides in the 4th lane of u_i: the force pass gathers one vector less per pair
        reinterpret_cast<T*>(vel + i)[3] = s;
    }
}

// ===========================================================================
// A7 / A10: wall velocities from a Shepard average of a fluid vector field
// with W(r, h/2) (eq:vf), then eq:vg-adami (u_wall = 0) or the
// slip reading (R16), then eq:vg-no-normal's clip.
//   mode 0: mirror (ghost velocity, no-slip u*): u_w = -Shepard
//   mode 1: slip u*: u_w = +Shepard
// ===========================================================================
template <class T, int D>
__global__ void __launch_bounds__(256) k_wall_velocity(Params<T> P, const V4<T>* __restrict__ pos,
                                                       const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap,
                                                       const V4<T>* __restrict__ nrm, const T* __restrict__ rho,
                                                       const V4<T>* __restrict__ uwl, V4<T>* __restrict__ vel,
                                                       int mode)
{
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= P.Nwo) return;
    int i = P.Nf + w;
    V4<T> xi = ld4(pos + i);
    T sw = 0, ax = 0, ay = 0, az = 0;
    int n = cnt[i];
    for_nbrs_pfx<SISPH_WALLV_PF>(nbr, ncap, i, n, [&](int j) {
        if (j >= P.Nf) return;
        V4<T> xj = ld4(pos + j);
        T d[3], r, ri;
        const T r2 = pair_vec<T, D>(P, xi, xj, d);
        if (r2 >= P.R2cut * T(0.25)) return;          // beyond 3 (h/2): W(r, h/2) = 0
        r_of(r2, r, ri);
        T wv = P.sig2 * quintic5(r * P.inv_h2);
        V4<T> uj = ld4(vel + j);
        ax += uj.x * wv;
        ay += uj.y * wv;
        if (D == 3) az += uj.z * wv;
        sw += wv;
    });
    // eq:vg-adami with the wall's prescribed velocity u_wall (uwl); an empty
    // Shepard sum gives u~ = u_wall (R15a)
    const V4<T> uw = ld4(uwl + w);
    T ux = uw.x, uy = uw.y, uz = D == 3 ? uw.z : T(0);
    if (sw > 0) {
        ux = ax / sw;
        uy = ay / sw;
        uz = D == 3 ? az / sw : T(0);
    }
    if (mode == 0) {
        ux = T(2) * uw.x - ux;
        uy = T(2) * uw.y - uy;
        uz = D == 3 ? T(2) * uw.z - uz : T(0);
    }
    V4<T> nn = ld4(nrm + w);
    T un = ux * nn.x + uy * nn.y;
    if (D == 3) un += uz * nn.z;
    if (un < 0) {
        ux -= un * nn.x;
        uy -= un * nn.y;
        if (D == 3) uz -= un * nn.z;
    }
    vel[i] = mk4<T>(ux, uy, uz, rho[i]);   // rho_w in the 4th lane (as the fluid's, see k_density)
}

// ===========================================================================
// A8: non-pressure forces + predictors (Alg. 1 lines 3-5):
//   f_visc  eq:mom:sph:visc, fluid + wall sources (R19)
//   f_avisc eq:mom:sph:av (R20), fluid + wall (ghost velocities)
//   f_astress eq:mom:sph:gtvf:stress (R21), fluid sources
//   u* = u + dt (f_visc + f_avisc + f_astress + g)   (eq:int:vint)
//   r* = r + dt u~                                    (eq:int:rnp1)
// ===========================================================================
// per-pair part of A8 (shared by the list pass and the staged cell pass):
// d = r_i - r_j (already minimum-image / shifted), r2 = |d|^2
template <class T, int D>
__device__ __forceinline__ void forces_pair(const Params<T>& P, const V4<T>& ui, T rhoi, T irhoi, T dux, T duy, T duz,
                                            const V4<T>& xj, const V4<T>& uj, const V4<T>& utj, bool fluid_j,
                                            const T (&d)[3], T r2, T& ax, T& ay, T& az)
{
    const T nu4 = T(4) * P.nu;
    const T avf2 = T(2) * P.alpha * P.h * P.c_ref;   // Pi = -avf phi / rhobar, rhobar = (rho_i + rho_j) / 2
    T rhoj = uj.w;                                   // k_density / k_wall_velocity put rho_j there
    T r, ri;
    r_of(r2, r, ri);
    T dwdr = P.dwk * quintic4(r * P.inv_h);
    T gf = dwdr * ri;                                // grad_i W_ij = gf * r_ij
    T mj = xj.w;
    T uijx = ui.x - uj.x, uijy = ui.y - uj.y, uijz = D == 3 ? ui.z - uj.z : T(0);
    T iden = frcp((rhoi + rhoj) * (r2 + P.eta_h2));  // shared by f_visc and f_avisc
    if (P.nu > T(0)) {
        T f = mj * nu4 * (r * dwdr) * iden;          // eq:mom:sph:visc
        ax += f * uijx;
        ay += f * uijy;
        if (D == 3) az += f * uijz;
    }
    if (P.alpha > T(0)) {
        T vr = uijx * d[0] + uijy * d[1];
        if (D == 3) vr += uijz * d[2];
        if (vr < T(0)) {                             // eq:mom:sph:av:params (R20)
            T Pi = -avf2 * vr * iden;
            T f = mj * Pi * gf;
            ax -= f * d[0];
            ay -= f * d[1];
            if (D == 3) az -= f * d[2];
        }
    }
    if (fluid_j) {                                   // eq:mom:sph:gtvf:stress (R21)
        T gx = gf * d[0], gy = gf * d[1], gz = D == 3 ? gf * d[2] : T(0);
        T ai = (dux * gx + duy * gy + (D == 3 ? duz * gz : T(0))) * irhoi;
        T aj = ((utj.x - uj.x) * gx + (utj.y - uj.y) * gy + (D == 3 ? (utj.z - uj.z) * gz : T(0))) * frcp(rhoj);
        ax += mj * (ui.x * ai + uj.x * aj);
        ay += mj * (ui.y * ai + uj.y * aj);
        if (D == 3) az += mj * (ui.z * ai + uj.z * aj);
    }
}

// per-particle part of A8: u* = u + dt a (eq:int:vint), r* = r + dt u~ (eq:int:rnp1)
template <class T, int D>
__device__ __forceinline__ void forces_finish(const Params<T>& P, int i, T dt, const V4<T>& xi, const V4<T>& ui,
                                              const V4<T>& uti, T rhoi, T ax, T ay, T az, V4<T>* __restrict__ us,
                                              V4<T>* __restrict__ rstar, V4<T>* __restrict__ fnp)
{
    us[i] = mk4<T>(ui.x + dt * ax, ui.y + dt * ay, D == 3 ? ui.z + dt * az : T(0), rhoi);   // rho_i in lane 4
    fnp[i] = mk4<T>(ax, ay, D == 3 ? az : T(0), T(0));   // f_visc + f_avisc + f_astress + f_body (adaptive dt)
    if (!rstar) return;                                  // single build: k_rstar computed r* (same expression)
    T rx = xi.x + dt * uti.x, ry = xi.y + dt * uti.y, rz = D == 3 ? xi.z + dt * uti.z : xi.z;
    if (P.per[0]) { if (rx >= P.hi[0]) rx -= P.L[0]; else if (rx < P.lo[0]) rx += P.L[0]; }
    if (P.per[1]) { if (ry >= P.hi[1]) ry -= P.L[1]; else if (ry < P.lo[1]) ry += P.L[1]; }
    if (D == 3 && P.per[2]) { if (rz >= P.hi[2]) rz -= P.L[2]; else if (rz < P.lo[2]) rz += P.L[2]; }
    rstar[i] = mk4<T>(rx, ry, rz, xi.w);
}

template <class T, int D>
__global__ void __launch_bounds__(128) k_forces_predict(Params<T> P, T dt, const V4<T>* __restrict__ pos,
                                                        const V4<T>* __restrict__ vel, const V4<T>* __restrict__ vt,
                                                        const T* __restrict__ rho, const int* __restrict__ nbr,
                                                        const int* __restrict__ cnt, int ncap, V4<T>* __restrict__ us,
                                                        V4<T>* __restrict__ rstar, V4<T>* __restrict__ fnp,
                                                        const T* __restrict__ rec)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.Nfo) return;
    V4<T> xi = ld4(pos + i), ui = ld4(vel + i), uti = ld4(vt + i);
    T rhoi = rho[i];
    T ax = P.g[0], ay = P.g[1], az = D == 3 ? P.g[2] : T(0);
    T dux = uti.x - ui.x, duy = uti.y - ui.y, duz = D == 3 ? uti.z - ui.z : T(0);
    const T irhoi = frcp(rhoi);
    int n = cnt[i];
    if (P.ptype && P.ptype[i] != 0) {
        // R34: inlet (prescribed) / outlet (frozen) velocity: u* = u, only r* = r + dt u~
        ax = ay = az = T(0);
        n = 0;
    }
    for_nbrs_pfx<SISPH_FORCES_PF>(nbr, ncap, i, n, [&](int j) {
        // (loose-list pairs beyond 3h contribute exactly 0: dW/dr = 0 for q >= 3)
        T q[8];
        ld8(rec + 8 * (size_t)j, q);                 // {r_j, m_j, u_j, rho_j} (k_pack_rec)
        const V4<T> xj = mk4<T>(q[0], q[1], q[2], q[3]), uj = mk4<T>(q[4], q[5], q[6], q[7]);
        const bool fl = j < P.Nf;
        V4<T> utj = fl ? ld4(vt + j) : uj;
        T d[3];
        T r2 = pair_vec<T, D>(P, xi, xj, d);
        forces_pair<T, D>(P, ui, rhoi, irhoi, dux, duy, duz, xj, uj, utj, fl, d, r2, ax, ay, az);
    });
    forces_finish<T, D>(P, i, dt, xi, ui, uti, rhoi, ax, ay, az, us, rstar, fnp);
}


// ===========================================================================
// A11: RHS_i (eq:sph-ppe right side, R8), D_ii (eq:coeff, R6/R7) and the
// device-wide Lambda = max |RHS_i / D_ii| over non-free-surface fluid with
// D_ii != 0 (eq:convergence, R12).
// ===========================================================================
//
// pin != nullptr: the FIRST Jacobi sweep (eq:p-sor from p^0 = pin, walls
// already refreshed from p^0, R14) is fused in: p^0_j is gathered with each
// pair, so sum_j fac_ij p^0_j needs no second pass over the list; p^1 goes
// to pout and the residual sums of eq:convergence are reduced as a deferred
// sweep (k_decide takes the decision in the solve, once Lambda is complete).
constexpr int RHS_T = 128;

// ---------------------------------------------------------------------------
// The sweep's 16-bit list (round 2).  The stored sweep streams, per pair, the
// neighbour index and the stored factor: 4 + 4 bytes.  In code mode A11
// writes each fluid row's S list as SLOTS of (16-bit code, factor) instead:
// the code is the difference to the previous entry (the row index i before
// the first one).  The list runs through the stencil rows in cell order, so
// inside a stencil row and between y-rows the steps fit in 15 bits; a longer
// step (between z-rows, into the wall / halo ranges, across a periodic image)
// takes two slots: A = high part, factor 0, gathers p_i; B = low 16 bits and
// the factor.  Slot codes: bit 0 = 0: d = (short)c >> 1; bit 0 = 1: slot A,
// hi = (short)c >> 1, and the next slot's 16 bits complete d = hi * 2^16 + lo.
// Every slot is decoded and gathered without a branch (fixed rate: one code,
// one factor); the row is padded with (0, 0) slots to a multiple of 8.
// Layout: row group g = i / 32, chunk c of 8 codes at uint4 index
// (g * cc8 + c) * 32 + i % 32 (coalesced like the 32-bit list); factors in
// the blocked-ELL layout of the list with the slot capacity 8 cc8; the slot
// count per row in nslot.  The decoded entries are the list's, in its order,
// and a (0-factor) slot adds +-0: the results are bit-equal.
// ---------------------------------------------------------------------------
__device__ __forceinline__ size_t code_at(int i, int cc8, int c)
{
    return ((size_t)(i >> 5) * cc8 + c) * 32 + (i & 31);
}

// the factors of slots k .. k + 7 (two blocked-ELL chunks), zeros if !ok
template <class T>
__device__ __forceinline__ void ld_slots8(const T* __restrict__ crow, int k, bool ok, T (&f)[8])
{
    T a[4] = {T(0), T(0), T(0), T(0)}, b[4] = {T(0), T(0), T(0), T(0)};
    if (ok) {
        ld_chunk4(crow + nb_off(k), a);
        ld_chunk4(crow + nb_off(k + 4), b);
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
        f[e] = a[e];
        f[4 + e] = b[e];
    }
}

template <class T> struct CodeWriter {
    uint4* code;
    T* crow;            // coef + nb_base(i, 8 cc8)
    int cc8, i, prev, ns;
    unsigned w0, w1, w2, w3;
    T f0, f1, f2, f3;
    __device__ CodeWriter(uint4* c, T* coef, int cc, int row)
        : code(c), crow(coef ? coef + nb_base(row, 8 * cc) : nullptr), cc8(cc), i(row), prev(row), ns(0),
          w0(0), w1(0), w2(0), w3(0), f0(0), f1(0), f2(0), f3(0)
    {
    }
    __device__ __forceinline__ void emit(unsigned c, T f)
    {
        w0 = __funnelshift_r(w0, w1, 16);
        w1 = __funnelshift_r(w1, w2, 16);
        w2 = __funnelshift_r(w2, w3, 16);
        w3 = (w3 >> 16) | (c << 16);
        f0 = f1;
        f1 = f2;
        f2 = f3;
        f3 = f;
        ns++;
        if ((ns & 3) == 0) {
            const T fb[4] = {f0, f1, f2, f3};
            st_chunk4(crow + nb_off(ns - 4), fb);
        }
        if ((ns & 7) == 0) code[code_at(i, cc8, (ns >> 3) - 1)] = make_uint4(w0, w1, w2, w3);
    }
    __device__ __forceinline__ void push(int j, T f)
    {
        const int d = j - prev;
        prev = j;
        if (d >= -16384 && d <= 16383) {
            emit(((unsigned)d << 1) & 0xFFFFu, f);
        } else {
            emit((((unsigned)(d >> 16) << 1) | 1u) & 0xFFFFu, T(0));
            emit((unsigned)d & 0xFFFFu, f);
        }
    }
    __device__ __forceinline__ void finish(int* nslot)
    {
        nslot[i] = ns;
        while (ns & 7) emit(0u, T(0));
    }
};

// CODE: the opt-in 16-bit step-code list (SISPH_SWEEP_CODES) is written too; the plain instance
// carries no CodeWriter state through the pair loop
template <class T, int D, bool CODE = false>
__global__ void __launch_bounds__(RHS_T) k_rhs_diag(Params<T> P, T inv_dt, const V4<T>* __restrict__ pos,
                                                    const V4<T>* __restrict__ us, const T* __restrict__ rho,
                                                    const uint8_t* __restrict__ fs, const int* __restrict__ nbr,
                                                    const int* __restrict__ cnt, int ncap, T* __restrict__ rhs,
                                                    T* __restrict__ diag, T* __restrict__ coef, Ctl* ctl,
                                                    const T* __restrict__ pin, T* __restrict__ pout,
                                                    double* __restrict__ partials, const T* __restrict__ rec,
                                                    uint4* __restrict__ code, int* __restrict__ nslot, int cc8)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double lam = 0.0, dn = 0.0, dd = 0.0;
    bool bad = false;
    if (i < P.Nfo) {
        V4<T> xi = ld4(pos + i), ui = ld4(us + i);
        T rhoi = rho[i];
        T sr = 0, sd = 0, sp = 0;
        int n = cnt[i];
        T* __restrict__ crow = coef ? coef + nb_base(i, ncap) : nullptr;
        // code mode (sweep_row): the factors go out as (code, factor) slots instead of in list order
        CodeWriter<T> cw(CODE ? code : nullptr, coef, cc8, i);
        if (CODE) crow = nullptr;
#ifndef SISPH_RHS_VST
#define SISPH_RHS_VST 1   // B200, C5: 1061 -> 904 us per launch
#endif
        T fb[4] = {T(0), T(0), T(0), T(0)};             // SISPH_RHS_VST: one 16/32-byte store per chunk
        for_nbrs_k_pf<SISPH_RHS_PF>(nbr, ncap, i, n, [&](int j, int k) {
            T q[8];
            ld8(rec + 8 * (size_t)j, q);             // {r*_j, m_j, u*_j, rho_j} (k_pack_rec)
            const V4<T> xj = mk4<T>(q[0], q[1], q[2], q[3]), uj = mk4<T>(q[4], q[5], q[6], q[7]);
            T rhoj = uj.w;                           // rho_j rides in u*_j's 4th lane
            T d[3], r, ri;
            T r2 = pair_vec<T, D>(P, xi, xj, d);
            r_of(r2, r, ri);
            T p4 = quintic4(r * P.inv_h);
            T mj = xj.w;
            T ud = (ui.x - uj.x) * d[0] + (ui.y - uj.y) * d[1];
            if (D == 3) ud += (ui.z - uj.z) * d[2];
            sr += mj * frcp(rhoj) * (ud * p4 * ri);                        // * (-dwk / dt) below
            const T f = mj * (r * p4) * frcp((rhoi + rhoj) * (r2 + P.eta_h2));   // * 4 dwk / rho_i below
            sd += f;
            // stored per-pair part of fac_ij (particles do not move during the solve):
            // the sweep then reads it instead of recomputing it (same value, same layout as nbr)
#if SISPH_RHS_VST
            const int e = k & 3;
            fb[0] = e == 0 ? f : fb[0];
            fb[1] = e == 1 ? f : fb[1];
            fb[2] = e == 2 ? f : fb[2];
            fb[3] = e == 3 ? f : fb[3];
            if (crow && (e == 3 || k == n - 1)) st_chunk4(crow + nb_off(k & ~3), fb);
#else
            if (crow) crow[nb_off(k)] = f;
#endif
            if (pin) sp += f * pin[j];                   // first sweep: sum_j fac_ij p^0_j
            if constexpr (CODE) cw.push(j, f);
        });
        if constexpr (CODE) cw.finish(nslot);
        sr *= -P.dwk * inv_dt;
        const T scale = T(4) * P.dwk * frcp(rhoi);
        sd *= scale;
        const bool frozen = fs[i] == 2;                 // R34 outlet row: not a PPE unknown
        rhs[i] = frozen ? T(0) : sr;
        diag[i] = frozen ? T(0) : sd;
        const bool live = !fs[i] && sd != T(0);
        if (live) lam = (double)fabs(sr / sd);
        if (pin) {
            // eq:p-sor with p^k = p^0, exactly as k_sweep (same expression order)
            const T pold = pin[i];
            T pnew = frozen ? pold : T(0);
            if (live) {
                sp *= scale;
                pnew = P.omega * (sr + sp) * frcp(sd) + (T(1) - P.omega) * pold;
            }
            pout[i] = pnew;
            if (P.mean_free) {
                // R32: reduce (sum, count) of the live rows; k_mean_fix removes the mean
                dn = live ? (double)pnew : 0.0;
                dd = live ? 1.0 : 0.0;
            } else {
                dn = fabs((double)pnew - (double)pold);
                dd = frozen ? 0.0 : fabs((double)pnew);
            }
            bad = !isfinite((double)pnew);
        }
    }
    lam = warp_max(lam);
    if ((threadIdx.x & 31) == 0 && lam > 0.0)
        atomicMax(&ctl->lambda_bits, (unsigned long long)__double_as_longlong(lam));
    if (!pin) return;
    // deferred sweep reduction (fixed order): block partials, the last block sums them
    __shared__ double sn[RHS_T / 32], sdd[RHS_T / 32];
    __shared__ int last;
    dn = warp_sum(dn);
    dd = warp_sum(dd);
    const int anybad = __any_sync(0xffffffffu, bad);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        sn[w] = dn;
        sdd[w] = dd;
        if (anybad) atomicExch(&ctl->nonfinite, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < RHS_T / 32; q++) {
            a += sn[q];
            b += sdd[q];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
        __threadfence();
        const unsigned t = atomicAdd(&ctl->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double a = 0, b = 0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) {
        a += ((volatile double*)partials)[2 * q];
        b += ((volatile double*)partials)[2 * q + 1];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
        sn[w] = a;
        sdd[w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double num = 0, den = 0;
        for (int q = 0; q < RHS_T / 32; q++) {
            num += sn[q];
            den += sdd[q];
        }
        ctl->red[0] = num;
        ctl->red[1] = den;
        ctl->red[2] = ctl->nonfinite ? 1.0 : 0.0;
        ctl->ticket = 0;
    }
}

// ===========================================================================
// A12(i): wall pressure, eq:p-shepard (R14): fluid sources, a_w = 0,
// sum W = 0 -> 0, optional clamp of negative values.  In a solve it reads
// p^k from the buffer selected by the device iteration counter.
// ===========================================================================
// Per-solve state of the PPE iteration that changes between solves (buffer
// rotation, list reallocation, the caller's tolerance): the sweep kernels
// read it from device memory, so the captured graph of the loop (a WHILE
// conditional node) is reused across steps.
template <class T> struct PpeDesc {
    const V4<T>* pos;
    const T* rho;
    const uint8_t* fs;
    const int* nbr;
    const T* coef;      // stored per-pair factor (nullptr: matrix-free)
    const uint4* code;  // the sweep's 16-bit list (CodeWriter; nullptr: the 32-bit list)
    const int* nslot;   // its slot count per row
    int cc8;            // 8-slot chunks per row
    T* pA;
    T* pB;
    double tol;
    double cscale;      // R12b: 1 / (global fluid count) for means, 1 for the printed sums
    int min_it, max_it;
};

// a pressure read inside a kernel that also writes p (the persistent and cluster PPE loops:
// other SMs' writes of the previous iteration): L2-coherent (ld.global.cg) instead of the
// read-only path, whose L1 lines could still hold an older iterate
template <bool COH, class T> __device__ __forceinline__ T ldp(const T* p) { return COH ? __ldcg(p) : __ldg(p); }

// WL lanes share a wall row (lane `sub` takes its chunks sub, sub + WL, ...; the sums
// meet by shuffles): walls are few (configs[1]: 3.1k) and each row is long, so one
// lane per row left the pass bound by a ~45-deep chain of dependent loads
constexpr int WL = 8;
// the body-force part of eq:p-shepard's numerator, g . sum_f rho_f W (r_w - r_f), with its fused
// multiply-adds written out (the grouping the compiler chose in k_ppe_wall, either precision)
template <class T, int D>
__device__ __forceinline__ T wall_gr(const Params<T>& P, T sx, T sy, T sz)
{
    T gr = fma(sx, P.g[0], sy * P.g[1]);
    if (D == 3) gr = fma(sz, P.g[2], gr);
    return gr;
}
template <class T, int D, bool COH = false>
__device__ __forceinline__ void wall_pressure_row(const Params<T>& P, int w, const V4<T>* __restrict__ pos,
                                                  const T* __restrict__ rho, const int* __restrict__ nbr,
                                                  const int* __restrict__ cnt, int ncap, T* p, int sub)
{
    int i = P.Nf + w;
    V4<T> xi = ld4(pos + i);
    T sw = 0, sp = 0, sx = 0, sy = 0, sz = 0;
    int n = cnt[i];
    const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, ncap));
    auto one = [&](int j) {
        if (j >= P.Nf) return;
        V4<T> xj = ld4(pos + j);
        T d[3], r, ri;
        r_of(pair_vec<T, D>(P, xi, xj, d), r, ri);
        T wv = P.sig * quintic5(r * P.inv_h);
        T rw = __ldg(rho + j) * wv;
        sp += ldp<COH>(p + j) * wv;
        sx += rw * d[0];
        sy += rw * d[1];
        if (D == 3) sz += rw * d[2];
        sw += wv;
    };
    for (int c = 4 * sub; c < n; c += 4 * WL) {
        const int4 v = LDLIST(q + (size_t)(c >> 2) * 32);
        one(v.x);
        if (c + 1 < n) one(v.y);
        if (c + 2 < n) one(v.z);
        if (c + 3 < n) one(v.w);
    }
    const unsigned gm = ((1u << WL) - 1u) << ((threadIdx.x & 31) & ~(WL - 1));
#pragma unroll
    for (int o = WL / 2; o > 0; o >>= 1) {
        sw += __shfl_xor_sync(gm, sw, o, WL);
        sp += __shfl_xor_sync(gm, sp, o, WL);
        sx += __shfl_xor_sync(gm, sx, o, WL);
        sy += __shfl_xor_sync(gm, sy, o, WL);
        if (D == 3) sz += __shfl_xor_sync(gm, sz, o, WL);
    }
    if (sub) return;
    T pw = 0;
    if (sw > T(0)) {
        const T gr = wall_gr<T, D>(P, sx, sy, sz);
        pw = (sp + gr) / sw;
    }
    if (P.clamp_wall_p && pw < T(0)) pw = T(0);
    p[i] = pw;
}

// The persistent loop's wall cache: positions do not move during the solve, so a wall row's
// Shepard weights W_wf, their sum and the body-force term are constants of the solve; only
// sum_f p_f W_wf changes per sweep.  Lane `sub` of wall row w stores its fluid entries (index,
// weight; at most WCE, slot e of thread t at [e * SWEEP_T + t]) in list order and the row's
// constants; returns the number of entries, or -1 when its share of the row is longer.
// Same expressions and order as wall_pressure_row.
constexpr int WCE = 8;
template <class T, int D, int NT>
__device__ __forceinline__ int wall_row_cache(const Params<T>& P, int w, const V4<T>* __restrict__ pos,
                                              const T* __restrict__ rho, const int* __restrict__ nbr,
                                              const int* __restrict__ cnt, int ncap, int sub, int* cj, T* cwv,
                                              T& c_sw, T& c_gr)
{
    const int i = P.Nf + w;
    const int n = cnt[i];
    if (n > WCE * WL) return -1;          // a lane would take more than WCE / 4 chunks
    V4<T> xi = ld4(pos + i);
    T sw = 0, sx = 0, sy = 0, sz = 0;
    int m = 0;
    const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, ncap));
    auto one = [&](int j) {
        if (j >= P.Nf) return;
        V4<T> xj = ld4(pos + j);
        T d[3], r, ri;
        r_of(pair_vec<T, D>(P, xi, xj, d), r, ri);
        T wv = P.sig * quintic5(r * P.inv_h);
        T rw = __ldg(rho + j) * wv;
        cj[m * NT] = j;
        cwv[m * NT] = wv;
        m++;
        sx += rw * d[0];
        sy += rw * d[1];
        if (D == 3) sz += rw * d[2];
        sw += wv;
    };
    for (int c = 4 * sub; c < n; c += 4 * WL) {
        const int4 v = LDLIST(q + (size_t)(c >> 2) * 32);
        one(v.x);
        if (c + 1 < n) one(v.y);
        if (c + 2 < n) one(v.z);
        if (c + 3 < n) one(v.w);
    }
    const unsigned gm = ((1u << WL) - 1u) << ((threadIdx.x & 31) & ~(WL - 1));
#pragma unroll
    for (int o = WL / 2; o > 0; o >>= 1) {
        sw += __shfl_xor_sync(gm, sw, o, WL);
        sx += __shfl_xor_sync(gm, sx, o, WL);
        sy += __shfl_xor_sync(gm, sy, o, WL);
        if (D == 3) sz += __shfl_xor_sync(gm, sz, o, WL);
    }
    c_sw = sw;
    c_gr = wall_gr<T, D>(P, sx, sy, sz);
    return m;
}
// one sweep's wall pressure of a cached row from the pressures in p (L2-coherent reads)
template <class T, int NT>
__device__ __forceinline__ void wall_row_cached(const Params<T>& P, int w, int m, const int* cj, const T* cwv, T c_sw,
                                                T c_gr, T* p, int sub)
{
    T pj[WCE];
#pragma unroll
    for (int e = 0; e < WCE; e++) pj[e] = e < m ? __ldcg(p + cj[e * NT]) : T(0);
    T sp = 0;
#pragma unroll
    for (int e = 0; e < WCE; e++)
        if (e < m) sp = fma(pj[e], cwv[e * NT], sp);
    const unsigned gm = ((1u << WL) - 1u) << ((threadIdx.x & 31) & ~(WL - 1));
#pragma unroll
    for (int o = WL / 2; o > 0; o >>= 1) sp += __shfl_xor_sync(gm, sp, o, WL);
    if (sub) return;
    T pw = 0;
    if (c_sw > T(0)) pw = (sp + c_gr) / c_sw;
    if (P.clamp_wall_p && pw < T(0)) pw = T(0);
    p[P.Nf + w] = pw;
}

// standalone wall pressure from the pressures in p (before A11's fused sweep, A13)
template <class T, int D>
__global__ void __launch_bounds__(256) k_wall_pressure(Params<T> P, const V4<T>* __restrict__ pos,
                                                       const T* __restrict__ rho, const int* __restrict__ nbr,
                                                       const int* __restrict__ cnt, int ncap, T* p)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x, w = t / WL;
    if (w >= P.Nwo) return;
    wall_pressure_row<T, D>(P, w, pos, rho, nbr, cnt, ncap, p, t % WL);
}

// in a solve: from p^k, the buffer selected by the device iteration counter
template <class T, int D>
__global__ void __launch_bounds__(256) k_ppe_wall(Params<T> P, const PpeDesc<T>* __restrict__ dsc,
                                                  const int* __restrict__ cnt, int ncap, const Ctl* ctl)
{
    pdl_trigger();
    pdl_wait();
    if (ctl->done) return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, w = t / WL;
    if (w >= P.Nwo) return;
    T* p = (ctl->iter & 1) ? dsc->pB : dsc->pA;
    wall_pressure_row<T, D>(P, w, dsc->pos, dsc->rho, dsc->nbr, cnt, ncap, p, t % WL);
}

// ===========================================================================
// A12(ii, iii): one damped-Jacobi sweep, eq:p-sor with
// fac_ij = 4 m_j / (rho_i (rho_i + rho_j)) r_ij.gradW_ij / (r^2 + eta h^2)
// recomputed matrix-free from the positions, the special cases
// of P:530-534, and the fused device-wide fp64 reduction of eq:convergence
// (sum |p^{k+1} - p^k|, sum |p^{k+1}|) finished by the last block, which also
// takes the stop decision (R12, R13) on the device.
// ===========================================================================
#ifndef SISPH_SWEEP_T
#define SISPH_SWEEP_T 256   // B200, C5: 128 / 256 / 512 -> 298 / 274 / 272 us
#endif
constexpr int SWEEP_T = SISPH_SWEEP_T;
// stored sweep: prefetch distance (chunks of 4 entries; 0 = none) and the minimum
// resident blocks per SM of the fp32 kernel (a 64-register cap: 4 x 256 threads).
// Tuned on B200 with A/B builds (build.py --out ... -DSISPH_SWEEP_PF=...):
// PD 0 / 2 / 3 / 4 / 4 capped -> 0.79 / 0.88 / 0.89 / 0.89 / 0.92 of the measured HBM
// bandwidth on C5; PD 5-8 fall off the occupancy cliff (2 blocks per SM).
#ifndef SISPH_SWEEP_PF
#define SISPH_SWEEP_PF 4
#endif
#ifndef SISPH_PERS_B
#define SISPH_PERS_B -4   // the persistent loop's sweep_row form (< 0: batched gathers, no ring)
#endif
#ifndef SISPH_CLUSTER_B
#define SISPH_CLUSTER_B -2
#endif
#ifndef SISPH_PERS_MINB
#define SISPH_PERS_MINB 3
#endif
#ifndef SISPH_SWEEP_G
#define SISPH_SWEEP_G 1   // 2: measured slower on C2 (1.67 -> 1.88 ms), equal on C4 / C5
#endif
#ifndef SISPH_SWEEP_MINB
#define SISPH_SWEEP_MINB 4
#endif
template <class T> constexpr int sweep_minb() { return sizeof(T) == 4 ? SISPH_SWEEP_MINB : 1; }

// eq:p-sor for row i from p^k = pin (the stored or the recomputed fac_ij)
// eq:p-sor for one row from its neighbour sum s = sum_j (stored factor)_ij p_j:
// p_i^{k+1} = omega (rhs_i + 4 dwk s / rho_i) / D_ii + (1 - omega) p_i^k.  The fused
// multiply-adds are written out (the grouping the compiler chose for k_sweep's expression in
// either precision), so every loop form -- and the persistent loop's cached rows, whose
// operands are loop invariants -- rounds identically whatever the surrounding code.
template <class T>
__device__ __forceinline__ T ppe_update(const Params<T>& P, T rhs_i, T s, T di, T rhoi, T pold)
{
    const T k = T(4) * P.dwk * frcp(rhoi);
    const T t = P.omega * fma(s, k, rhs_i);
    const T om1 = T(1) - P.omega;
    if constexpr (sizeof(T) == 4) return fma(frcp(di), t, pold * om1);
    else return fma(pold, om1, frcp(di) * t);
}

template <class T, int D, bool STORED, bool COH = false, int PFD = SISPH_SWEEP_PF, bool CODE = true>
__device__ __forceinline__ T sweep_row(const Params<T>& P, int i, const V4<T>* __restrict__ pos,
                                       const T* __restrict__ rho, const uint8_t* __restrict__ fs,
                                       const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap,
                                       const T* __restrict__ coef, const T* __restrict__ rhs,
                                       const T* __restrict__ diag, const T* pin,
                                       const uint4* __restrict__ code = nullptr,
                                       const int* __restrict__ nslot = nullptr, int cc8 = 0)
{
    const T pold = pin[i];
    T pnew = fs[i] == 2 ? pold : T(0);                 // R34 outlet rows keep their frozen p
    const T di = diag[i];
    if (!fs[i] && di != T(0)) {
        const T rhoi = rho[i];
        T s = 0;
        const int n = cnt[i];
        const size_t b = nb_base(i, ncap);
        bool wide = true;
        if constexpr (STORED && CODE) {
            if (code) {
            // code mode (CodeWriter): 2 + 4 bytes per slot instead of 4 + 4 per pair.  Each
            // iteration decodes 8 slots without a branch, gathers their 8 p_j, then sums in
            // slot order; the code chunk and the two factor chunks of the iteration DIST
            // ahead are in flight meanwhile.
            wide = false;
            constexpr int DIST = (PFD >= 4 && sizeof(T) == 4) ? 2 : 1;
            const int ns = nslot[i];
            const T* __restrict__ crow = coef + nb_base(i, 8 * cc8);
            uint4 cq[DIST];
            T fq[DIST][8];
#pragma unroll
            for (int q = 0; q < DIST; q++) {
                const bool ok = 8 * q < ns;
                cq[q] = ok ? LDLIST(code + code_at(i, cc8, q)) : make_uint4(0, 0, 0, 0);
                ld_slots8(crow, 8 * q, ok, fq[q]);
            }
            int prev = i, hi = 0;
            bool pend = false;
            for (int c = 0; c < ns; c += 8) {
                const int cn = c + 8 * DIST;
                const bool okn = cn < ns;
                const uint4 cx = okn ? LDLIST(code + code_at(i, cc8, cn >> 3)) : make_uint4(0, 0, 0, 0);
                T fx[8];
                ld_slots8(crow, cn, okn, fx);
                const unsigned wv[4] = {cq[0].x, cq[0].y, cq[0].z, cq[0].w};
                int jj[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const unsigned cu = (wv[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
                    const int v = (int)(short)cu >> 1;
                    const bool isA = !pend && (cu & 1u);
                    const int jr = prev + (pend ? (int)(((unsigned)hi << 16) | cu) : v);
                    jj[u] = isA ? i : jr;
                    prev = isA ? prev : jr;
                    hi = v;
                    pend = isA;
                }
                T pj[8];
#pragma unroll
                for (int u = 0; u < 8; u++) pj[u] = ldp<COH>(pin + jj[u]);
#pragma unroll
                for (int u = 0; u < 8; u++) s += fq[0][u] * pj[u];
#pragma unroll
                for (int q = 0; q < DIST - 1; q++) {
                    cq[q] = cq[q + 1];
#pragma unroll
                    for (int e = 0; e < 8; e++) fq[q][e] = fq[q + 1][e];
                }
                cq[DIST - 1] = cx;
#pragma unroll
                for (int e = 0; e < 8; e++) fq[DIST - 1][e] = fx[e];
            }
            }
        }
        if (STORED && wide) {
            const int4* __restrict__ qi = reinterpret_cast<const int4*>(nbr + b);
            if constexpr (PFD < 0) {
            // latency-bound form (persistent / cluster loops, L2-resident lists): the list and
            // factor chunks are read through L1 (__ldg: a block's rows are re-read every
            // sweep and stay L1-resident on small problems); B = -PFD
            // chunks per iteration, their 4B gathers all issued before the sums consume them
            // in entry order; entries past the row end gather p_i with a zero factor
            constexpr int B = -PFD;
            for (int c = 0; c < n; c += 4 * B) {
                int4 v[B];
                T f[B][4];
#pragma unroll
                for (int g = 0; g < B; g++) {
                    const int cg0 = c + 4 * g;
                    v[g] = cg0 < n ? __ldg(qi + (size_t)(cg0 >> 2) * 32) : make_int4(i, i, i, i);
                    f[g][0] = f[g][1] = f[g][2] = f[g][3] = T(0);
                    if (cg0 < n) ld_chunk4_l1(coef + b + ((size_t)(cg0 >> 2) * 32 << 2), f[g]);
                }
                T pv[B][4];
#pragma unroll
                for (int g = 0; g < B; g++) {
                    const int cg0 = c + 4 * g;
                    pv[g][0] = ldp<COH>(pin + (cg0 < n ? v[g].x : i));
                    pv[g][1] = ldp<COH>(pin + (cg0 + 1 < n ? v[g].y : i));
                    pv[g][2] = ldp<COH>(pin + (cg0 + 2 < n ? v[g].z : i));
                    pv[g][3] = ldp<COH>(pin + (cg0 + 3 < n ? v[g].w : i));
                }
#pragma unroll
                for (int g = 0; g < B; g++) {
                    const int cg0 = c + 4 * g;
#pragma unroll
                    for (int e = 0; e < 4; e++) s += (cg0 + e < n ? f[g][e] : T(0)) * pv[g][e];
                }
            }
            } else if constexpr (PFD > 0) {
            // software pipelining: a register ring keeps the index + factor loads of the next
            // PD chunks in flight while this chunk's p_j are gathered (B200: the streamed
            // HBM traffic needs more bytes in flight per SM than one chunk per row gives;
            // PD = 4 at a 64-register cap measured best, 0.92 of the measured HBM bandwidth)
            // G chunks per iteration: their 4G gathers are all issued before the sums
            // consume them (in entry order, so the result is unchanged): the dependent
            // chain of a row is n / 4G gather latencies, not n / 4
            constexpr int PD = PFD;
            constexpr int G = (PD >= 4 && PD % SISPH_SWEEP_G == 0) ? SISPH_SWEEP_G : 1;
            int4 vr[PD];
            T fr[PD][4];
#pragma unroll
            for (int q = 0; q < PD; q++) {
                const int c = 4 * q;
                vr[q] = c < n ? LDLIST(qi + (size_t)(c >> 2) * 32) : make_int4(i, i, i, i);
                if (c < n) ld_chunk4(coef + b + ((size_t)(c >> 2) * 32 << 2), fr[q]);
                else fr[q][0] = fr[q][1] = fr[q][2] = fr[q][3] = T(0);
            }
            for (int c = 0; c < n; c += 4 * G) {
                int4 vnew[G];
                T fnew[G][4];
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const int cn = c + 4 * (PD + g);
                    vnew[g] = cn < n ? LDLIST(qi + (size_t)(cn >> 2) * 32) : make_int4(i, i, i, i);
                    fnew[g][0] = fnew[g][1] = fnew[g][2] = fnew[g][3] = T(0);
                    if (cn < n) ld_chunk4(coef + b + ((size_t)(cn >> 2) * 32 << 2), fnew[g]);
                }
                // entries past the row end gather p_i (a valid slot) with a zero factor:
                // adding +-0 leaves s unchanged, and the loads issue without predicates
                T pv[G][4];
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const int cg0 = c + 4 * g;
                    pv[g][0] = ldp<COH>(pin + (cg0 < n ? vr[g].x : i));
                    pv[g][1] = ldp<COH>(pin + (cg0 + 1 < n ? vr[g].y : i));
                    pv[g][2] = ldp<COH>(pin + (cg0 + 2 < n ? vr[g].z : i));
                    pv[g][3] = ldp<COH>(pin + (cg0 + 3 < n ? vr[g].w : i));
                }
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const int cg0 = c + 4 * g;
#pragma unroll
                    for (int e = 0; e < 4; e++) s += (cg0 + e < n ? fr[g][e] : T(0)) * pv[g][e];
                }
#pragma unroll
                for (int q = 0; q < PD - G; q++) {
                    vr[q] = vr[q + G];
#pragma unroll
                    for (int e = 0; e < 4; e++) fr[q][e] = fr[q + G][e];
                }
#pragma unroll
                for (int g = 0; g < G; g++) {
                    vr[PD - G + g] = vnew[g];
#pragma unroll
                    for (int e = 0; e < 4; e++) fr[PD - G + g][e] = fnew[g][e];
                }
            }
            } else {
            for (int c = 0; c < n; c += 4) {
                const size_t o = (size_t)(c >> 2) * 32;
                const int4 v = LDLIST(qi + o);
                T f[4];
                ld_chunk4(coef + b + (o << 2), f);
                s += f[0] * ldp<COH>(pin + v.x);
                if (c + 1 < n) s += f[1] * ldp<COH>(pin + v.y);
                if (c + 2 < n) s += f[2] * ldp<COH>(pin + v.z);
                if (c + 3 < n) s += f[3] * ldp<COH>(pin + v.w);
            }
            }
        } else if (!STORED) {
            const V4<T> xi = ld4(pos + i);
            for_nbrs(nbr, ncap, i, n, [&](int j) {
                V4<T> xj = ld4(pos + j);
                T rhoj = __ldg(rho + j);
                T pj = ldp<COH>(pin + j);
                T d[3], r, ri;
                T r2 = pair_vec<T, D>(P, xi, xj, d);
                r_of(r2, r, ri);
                // fac_ij / (4 dW/dr-scale / rho_i): m_j r poly4(q) / ((rho_i + rho_j)(r^2 + eta h^2))
                // (the expression of k_rhs_diag's stored value, so both modes agree bit for bit)
                s += xj.w * (r * quintic4(r * P.inv_h)) * frcp((rhoi + rhoj) * (r2 + P.eta_h2)) * pj;
            });
        }
        pnew = ppe_update(P, rhs[i], s, di, rhoi, pold);   // S_i = 4 dwk s / rho_i = -sum_j OD_ij p_j
    }
    return pnew;
}

// STORED: the per-pair part of fac_ij written by k_rhs_diag is streamed
// alongside the neighbour index (an ELL SpMV: 4 + 4 bytes per pair from HBM,
// p_j gathered); otherwise it is recomputed from the positions every sweep,
// as the paper's listing does.
//
// The per-solve pointers and the tolerance / bounds come from dsc (device
// memory).  use_h: the kernel runs inside the WHILE body of the solve's CUDA
// graph and sets the loop condition (continue = not done) from the last
// block; a sweep launched after the decision only clears it.
// CODE: rows may come as the opt-in 16-bit step-code list (SISPH_SWEEP_CODES); the plain
// instance has no code path
template <class T, int D, bool STORED, bool CODE = false>
__global__ void __launch_bounds__(SWEEP_T, sweep_minb<T>()) k_sweep(Params<T> P, const PpeDesc<T>* __restrict__ dsc,
                                                   const T* __restrict__ rhs, const T* __restrict__ diag,
                                                   const int* __restrict__ cnt, int ncap, Ctl* ctl,
                                                   double* __restrict__ partials, int defer,
                                                   cudaGraphConditionalHandle hcond, int use_h)
{
    pdl_trigger();
    pdl_wait();
    if (ctl->done) {
        if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(hcond, 0u);
        return;
    }
    const V4<T>* __restrict__ pos = dsc->pos;
    const T* __restrict__ rho = dsc->rho;
    const uint8_t* __restrict__ fs = dsc->fs;
    const int* __restrict__ nbr = dsc->nbr;
    const T* __restrict__ coef = dsc->coef;
    const uint4* __restrict__ code = dsc->code;
    const int* __restrict__ nslot = dsc->nslot;
    const int cc8 = dsc->cc8;
    T* pA = dsc->pA;
    T* pB = dsc->pB;
    const int kit = ctl->iter;
    const T* __restrict__ pin = (kit & 1) ? pB : pA;
    T* __restrict__ pout = (kit & 1) ? pA : pB;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double dn = 0.0, dd = 0.0;
    bool bad = false;
    if (i < P.Nfo) {
        const T pold = pin[i];
        const T pnew = sweep_row<T, D, STORED, false, SISPH_SWEEP_PF, CODE>(P, i, pos, rho, fs, nbr, cnt, ncap, coef, rhs,
                                                                          diag, pin, code, nslot, cc8);
        pout[i] = pnew;
        if (P.mean_free) {
            // R32: (sum, count) of the live rows; k_mean_fix removes the mean and decides
            const bool live = !fs[i] && diag[i] != T(0);
            dn = live ? (double)pnew : 0.0;
            dd = live ? 1.0 : 0.0;
        } else {
            dn = fabs((double)pnew - (double)pold);
            dd = fs[i] == 2 ? 0.0 : fabs((double)pnew);   // eq:convergence over the unknown rows
        }
        bad = !isfinite((double)pnew);
    }
    // block reduction (fixed order)
    __shared__ double sn[SWEEP_T / 32], sd[SWEEP_T / 32];
    __shared__ int last;
    dn = warp_sum(dn);
    dd = warp_sum(dd);
    int anybad = __any_sync(0xffffffffu, bad);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        sn[w] = dn;
        sd[w] = dd;
        if (anybad) atomicExch(&ctl->nonfinite, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < SWEEP_T / 32; q++) {
            a += sn[q];
            b += sd[q];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
        __threadfence();
        unsigned t = atomicAdd(&ctl->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last block: fixed-assignment sum of all partials -> deterministic
    double a = 0, b = 0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) {
        a += ((volatile double*)partials)[2 * q];
        b += ((volatile double*)partials)[2 * q + 1];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
        sn[w] = a;
        sd[w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double num = 0, den = 0;
        for (int q = 0; q < SWEEP_T / 32; q++) {
            num += sn[q];
            den += sd[q];
        }
        if (defer || P.mean_free) {
            // slab ranks: the local sums go through an allreduce, k_decide finishes
            // (mean-free: the live-row sum and count go to k_mean_fix)
            ctl->red[0] = num;
            ctl->red[1] = den;
            ctl->red[2] = ctl->nonfinite ? 1.0 : 0.0;
            ctl->ticket = 0;
            return;
        }
        num *= dsc->cscale;
        den *= dsc->cscale;
        double lam = __longlong_as_double((long long)ctl->lambda_bits);
        double dmax = den > lam ? den : lam;
        double res = num == 0.0 ? 0.0 : (dmax > 0.0 ? num / dmax : INFINITY);
        int k1 = kit + 1;
        ctl->residual = res;
        ctl->iter = k1;
        const int done = ((k1 >= dsc->min_it && res < dsc->tol) || k1 >= dsc->max_it || ctl->nonfinite) ? 1 : 0;
        ctl->done = done;
        ctl->ticket = 0;
        if (use_h) cudaGraphSetConditional(hcond, done ? 0u : 1u);
    }
}

// Reading R32 (ppe_mean_free): the sweep (or A11's fused first sweep) left
// p^{k+1} in pout and (sum, count) of its live rows in ctl->red (allreduced
// on slab ranks).  Subtract the mean from the live rows, then the fused
// eq:convergence reduction of k_sweep on the corrected iterate: decide (one
// handle; in the solve's graph it sets the WHILE condition) or defer the two
// sums to an allreduce + k_decide (slab ranks).
template <class T>
__global__ void __launch_bounds__(SWEEP_T) k_mean_fix(Params<T> P, const PpeDesc<T>* __restrict__ dsc,
                                                      const T* __restrict__ diag, Ctl* ctl,
                                                      double* __restrict__ partials, int defer,
                                                      cudaGraphConditionalHandle hcond, int use_h)
{
    pdl_trigger();
    pdl_wait();
    if (ctl->done) {
        if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(hcond, 0u);
        return;
    }
    const uint8_t* __restrict__ fs = dsc->fs;
    const int kit = ctl->iter;
    const T* __restrict__ pin = (kit & 1) ? dsc->pB : dsc->pA;
    T* __restrict__ pout = (kit & 1) ? dsc->pA : dsc->pB;
    const double sum = ctl->red[0], count = ctl->red[1], bad_in = ctl->red[2];
    const double mean = count > 0.0 ? sum / count : 0.0;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double dn = 0.0, dd = 0.0;
    bool bad = false;
    if (i < P.Nfo) {
        T v = pout[i];
        if (!fs[i] && diag[i] != T(0)) {
            v = (T)((double)v - mean);
            pout[i] = v;
        }
        dn = fabs((double)v - (double)pin[i]);
        dd = fs[i] == 2 ? 0.0 : fabs((double)v);
        bad = !isfinite((double)v);
    }
    __shared__ double sn[SWEEP_T / 32], sd[SWEEP_T / 32];
    __shared__ int last;
    dn = warp_sum(dn);
    dd = warp_sum(dd);
    const int anybad = __any_sync(0xffffffffu, bad);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        sn[w] = dn;
        sd[w] = dd;
        if (anybad) atomicExch(&ctl->nonfinite, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < SWEEP_T / 32; q++) {
            a += sn[q];
            b += sd[q];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
        __threadfence();
        const unsigned t = atomicAdd(&ctl->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double a = 0, b = 0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) {
        a += ((volatile double*)partials)[2 * q];
        b += ((volatile double*)partials)[2 * q + 1];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
        sn[w] = a;
        sd[w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double num = 0, den = 0;
        for (int q = 0; q < SWEEP_T / 32; q++) {
            num += sn[q];
            den += sd[q];
        }
        if (bad_in > 0.0) ctl->nonfinite = 1;
        ctl->ticket = 0;
        if (defer) {
            ctl->red[0] = num;
            ctl->red[1] = den;
            ctl->red[2] = ctl->nonfinite ? 1.0 : 0.0;
            return;
        }
        num *= dsc->cscale;
        den *= dsc->cscale;
        const double lam = __longlong_as_double((long long)ctl->lambda_bits);
        const double dmax = den > lam ? den : lam;
        const double res = num == 0.0 ? 0.0 : (dmax > 0.0 ? num / dmax : INFINITY);
        const int k1 = kit + 1;
        ctl->residual = res;
        ctl->iter = k1;
        const int done = ((k1 >= dsc->min_it && res < dsc->tol) || k1 >= dsc->max_it || ctl->nonfinite) ? 1 : 0;
        ctl->done = done;
        if (use_h) cudaGraphSetConditional(hcond, done ? 0u : 1u);
    }
}

// R33: max_i p_i over the owned fluid (one block, fixed order; once per handle);
// with open boundaries (R34) over the fluid proper (not inlet / outlet rows)
template <class T>
__global__ void __launch_bounds__(1024) k_fluid_pmax(const T* __restrict__ p, int nf, const uint8_t* __restrict__ ptype,
                                                     double* out)
{
    __shared__ double sm[32];
    double m = -INFINITY;
    for (int i = threadIdx.x; i < nf; i += blockDim.x)
        if (!ptype || ptype[i] == 0) m = fmax(m, (double)p[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); q++) m = fmax(m, sm[q]);
        *out = fmax(m, sm[0]);
    }
}

// eq:convergence on the allreduced sums (slab ranks; every rank takes the
// same decision from the same bits).  A no-op once the solve is done.
__global__ void k_decide(Ctl* ctl, double tol, int min_it, int max_it, double cscale)
{
    if (ctl->done) return;
    const double num = ctl->red[0] * cscale, den = ctl->red[1] * cscale;
    const double lam = __longlong_as_double((long long)ctl->lambda_bits);
    const double dmax = den > lam ? den : lam;
    const double res = num == 0.0 ? 0.0 : (dmax > 0.0 ? num / dmax : INFINITY);
    const int k1 = ctl->iter + 1;
    if (ctl->red[2] > 0.0) ctl->nonfinite = 1;
    ctl->residual = res;
    ctl->iter = k1;
    ctl->done = ((k1 >= min_it && res < tol) || k1 >= max_it || ctl->nonfinite) ? 1 : 0;
}

// sweep_row's batched-gather form with p^k of the block's neighbour span staged in shared
// memory (persistent loop, stored factors): the same loads of the list and the factors, the
// same sums in entry order (pads gather p_i with a zero factor) -- only the p_j come from the
// tile instead of one L2 request per pair.  Slot of particle j in the tile: fluid j - f0,
// wall j - wsh (the wall span follows the fluid span).
#ifndef SISPH_PERS_TILE
#define SISPH_PERS_TILE 2048
#endif
constexpr int PERS_TILE = SISPH_PERS_TILE;
template <class T, int B>
__device__ __forceinline__ T sweep_row_tile(const Params<T>& P, int i, const T* __restrict__ rho,
                                            const uint8_t* __restrict__ fs, const int* __restrict__ nbr,
                                            const int* __restrict__ cnt, int ncap, const T* __restrict__ coef,
                                            const T* __restrict__ rhs, const T* __restrict__ diag,
                                            const T* tile, int f0, int wsh)
{
    const int nf = P.Nf;
    const T pold = tile[i - f0];
    T pnew = fs[i] == 2 ? pold : T(0);                 // R34 outlet rows keep their frozen p
    const T di = diag[i];
    if (!fs[i] && di != T(0)) {
        const T rhoi = rho[i];
        T s = 0;
        const int n = cnt[i];
        const size_t b = nb_base(i, ncap);
        const int4* __restrict__ qi = reinterpret_cast<const int4*>(nbr + b);
        for (int c = 0; c < n; c += 4 * B) {
            int4 v[B];
            T f[B][4];
#pragma unroll
            for (int g = 0; g < B; g++) {
                const int cg0 = c + 4 * g;
                v[g] = cg0 < n ? __ldg(qi + (size_t)(cg0 >> 2) * 32) : make_int4(i, i, i, i);
                f[g][0] = f[g][1] = f[g][2] = f[g][3] = T(0);
                if (cg0 < n) ld_chunk4_l1(coef + b + ((size_t)(cg0 >> 2) * 32 << 2), f[g]);
            }
            T pv[B][4];
#pragma unroll
            for (int g = 0; g < B; g++) {
                const int cg0 = c + 4 * g;
                const int j0 = cg0 < n ? v[g].x : i, j1 = cg0 + 1 < n ? v[g].y : i;
                const int j2 = cg0 + 2 < n ? v[g].z : i, j3 = cg0 + 3 < n ? v[g].w : i;
                pv[g][0] = tile[j0 - (j0 < nf ? f0 : wsh)];
                pv[g][1] = tile[j1 - (j1 < nf ? f0 : wsh)];
                pv[g][2] = tile[j2 - (j2 < nf ? f0 : wsh)];
                pv[g][3] = tile[j3 - (j3 < nf ? f0 : wsh)];
            }
#pragma unroll
            for (int g = 0; g < B; g++) {
                const int cg0 = c + 4 * g;
#pragma unroll
                for (int e = 0; e < 4; e++) s += (cg0 + e < n ? f[g][e] : T(0)) * pv[g][e];
            }
        }
        pnew = ppe_update(P, rhs[i], s, di, rhoi, pold);   // S_i = 4 dwk s / rho_i = -sum_j OD_ij p_j
    }
    return pnew;
}

// ===========================================================================
// The whole PPE loop in ONE cooperative launch (small problems, where the
// per-sweep launches and their latency dominate: BASELINE configs[0-1]).
// Per sweep: walls from p^k (grid-stride), grid barrier, fluid rows (grid-
// stride) + block partials (per parity), grid barrier, then every block sums
// the partials in block order and takes the same eq:convergence decision (no
// third barrier; block 0 publishes it to ctl).  Same row arithmetic as
// k_sweep; the sums are grouped per block of the grid-stride loop (rounding-
// level differences in the residual only).
// ===========================================================================
#ifdef SISPH_PERS_PROF
__device__ unsigned long long g_pers_prof[4096 * 6];   // debug build: per-block phase times (ns)
#endif
// Grid barrier of the persistent PPE kernel: a monotone arrival counter (reset
// before the launch), thread 0 of every block adds 1 with release semantics and
// spins until the counter reaches (barrier number) x (blocks) with acquire
// loads.  Unlike cg::grid_group::sync it does not invalidate L1: every value
// another block wrote during the kernel (pressures, partials, the non-finite
// flag) is read L2-coherent (ldp<true>, __ldcg), the rest is read-only.
__device__ __forceinline__ void pgrid_sync(unsigned int* cnt, unsigned int target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if ((int)(v - target) >= 0) break;
        }
    }
    __syncthreads();
}

template <class T, int D, bool STORED>
__global__ void __launch_bounds__(SWEEP_T, SISPH_PERS_MINB) k_ppe_persistent(Params<T> P, const PpeDesc<T>* __restrict__ dsc,
                                                            const T* __restrict__ rhs, const T* __restrict__ diag,
                                                            const int* __restrict__ cnt, int ncap, Ctl* ctl,
                                                            double* __restrict__ partials, int csm)
{
    unsigned int* gbar = &ctl->gbar;
    unsigned int nbar = 0;
    const V4<T>* __restrict__ pos = dsc->pos;
    const T* __restrict__ rho = dsc->rho;
    const uint8_t* __restrict__ fs = dsc->fs;
    const int* __restrict__ nbr = dsc->nbr;
    const T* __restrict__ coef = dsc->coef;
    const uint4* __restrict__ code = dsc->code;
    const int* __restrict__ nslot = dsc->nslot;
    const int cc8 = dsc->cc8;
    T* pA = dsc->pA;
    T* pB = dsc->pB;
    const double tol = dsc->tol;
    const int min_it = dsc->min_it, max_it = dsc->max_it;
    volatile Ctl* vc = ctl;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // wall rows block-cyclic (every block takes its share, WL lanes each): the wall phase
    // runs beside the decision in every block instead of in the first blocks only
    const int wq0 = (threadIdx.x / WL) * gridDim.x + blockIdx.x, wqs = (blockDim.x / WL) * gridDim.x;
    __shared__ double sn[SWEEP_T / 32], sd[SWEEP_T / 32];
    __shared__ int done_s;
    // two grid barriers per iteration: walls | sweep + block partials (per parity) | every
    // block sums the partials in block order and takes the (identical) stop decision itself
    int kit = vc->iter;
    bool done = vc->done != 0;
    const double lam = __longlong_as_double((long long)vc->lambda_bits);
#ifdef SISPH_PERS_PROF
    unsigned long long tp[6] = {0, 0, 0, 0, 0, 0}, tq0 = 0, tq1 = 0;
#define PPROF(k) if (threadIdx.x == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq1)); if (k) tp[k - 1] += tq1 - tq0; tq0 = tq1; }
#else
#define PPROF(k)
#endif
    // the neighbour span of this block's rows (once per solve: the lists do not change): when the
    // fluid span [f0, f0 + nfs) and the wall span [w0, w0 + nws) fit the tile, every sweep stages
    // their p^k in shared memory (one coalesced L2 read per value instead of one L2 request per
    // pair: the gathers bypass L1, and on configs[1] their sectors were the sweep phase's bound)
    __shared__ T tile[STORED ? PERS_TILE : 1];
    __shared__ int span_s[4];
    int f0 = 0, w0 = 0, nfs = 0, nws = 0;
    bool tiled = false;
    if constexpr (STORED) {
        // (only with the row cache, csm > 0: the tile alone measured slower than plain gathers)
        if (!done && code == nullptr && csm > 0) {
            if (threadIdx.x == 0) {
                span_s[0] = span_s[2] = 0x7fffffff;
                span_s[1] = span_s[3] = -1;
            }
            __syncthreads();
            int fmn = 0x7fffffff, fmx = -1, wmn = 0x7fffffff, wmx = -1;
            for (int i = gt; i < P.Nfo; i += gs) {
                fmn = min(fmn, i);
                fmx = max(fmx, i);
                if (!fs[i] && diag[i] != T(0))
                    for_nbrs(nbr, ncap, i, cnt[i], [&](int j) {
                        if (j < P.Nf) {
                            fmn = min(fmn, j);
                            fmx = max(fmx, j);
                        } else {
                            wmn = min(wmn, j);
                            wmx = max(wmx, j);
                        }
                    });
            }
            fmn = __reduce_min_sync(0xffffffffu, fmn);
            fmx = __reduce_max_sync(0xffffffffu, fmx);
            wmn = __reduce_min_sync(0xffffffffu, wmn);
            wmx = __reduce_max_sync(0xffffffffu, wmx);
            if (lane == 0) {
                atomicMin(&span_s[0], fmn);
                atomicMax(&span_s[1], fmx);
                atomicMin(&span_s[2], wmn);
                atomicMax(&span_s[3], wmx);
            }
            __syncthreads();
            f0 = span_s[0];
            nfs = span_s[1] >= f0 ? span_s[1] - f0 + 1 : 0;
            w0 = span_s[2];
            nws = span_s[3] >= w0 ? span_s[3] - w0 + 1 : 0;
            tiled = nfs > 0 && (long long)nfs + nws <= PERS_TILE;
        }
    }
    const int wsh = w0 - nfs;
    // the row cache (csm > 0: the launch carries csm 4-entry chunks per thread of dynamic shared
    // memory): the first row of every thread keeps its first csm chunks -- tile slots as 16-bit
    // values and the stored factors, pads as (own slot, 0) -- and its row constants in registers
    // for the whole solve.  On configs[1] the lists of an SM's rows exceed its L1 (ncu: 2 % hit
    // rate), so every sweep re-read them from L2; now a sweep reads the tile and nothing else.
    extern __shared__ __align__(16) unsigned char pers_dsm[];
    T* const cfac = reinterpret_cast<T*>(pers_dsm);                                    // [csm][SWEEP_T][4]
    unsigned short* const cidx = reinterpret_cast<unsigned short*>(cfac + (size_t)csm * SWEEP_T * 4);
    const bool cached = STORED && tiled && csm > 0 && gt < P.Nfo;
    int cn = 0;                // entries of the cached row that are summed (0: the row does not sum)
    T c_di = 0, c_rhs = 0, c_rhoi = 0;
    int c_fs = 0;
    if constexpr (STORED) {
        if (cached) {
            const int i = gt;
            c_fs = fs[i];
            c_di = diag[i];
            c_rhs = rhs[i];
            c_rhoi = rho[i];
            cn = (!c_fs && c_di != T(0)) ? cnt[i] : 0;
            const size_t b = nb_base(i, ncap);
            const int4* __restrict__ qi = reinterpret_cast<const int4*>(nbr + b);
            for (int c = 0; c < csm && 4 * c < cn; c++) {
                const int4 v = __ldg(qi + (size_t)c * 32);
                T f[4];
                ld_chunk4_l1(coef + b + ((size_t)c * 32 << 2), f);
                const int jv[4] = {v.x, v.y, v.z, v.w};
                ushort4 lv;
                unsigned short* lp = &lv.x;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const bool ok = 4 * c + e < cn;
                    const int j = ok ? jv[e] : i;
                    lp[e] = (unsigned short)(j - (j < P.Nf ? f0 : wsh));
                    if (!ok) f[e] = T(0);
                }
                *reinterpret_cast<ushort4*>(cidx + ((size_t)c * SWEEP_T + threadIdx.x) * 4) = lv;
                st_chunk4(cfac + ((size_t)c * SWEEP_T + threadIdx.x) * 4, f);
            }
        }
    }
    // the wall cache (wall_row_cache): this thread's lane of its first wall row
    int* const wcj = reinterpret_cast<int*>(cidx + (size_t)csm * SWEEP_T * 4) + threadIdx.x;
    T* const wcw = reinterpret_cast<T*>(wcj - threadIdx.x + WCE * SWEEP_T) + threadIdx.x;
    int wm = -1;
    T c_wsw = 0, c_wgr = 0;
    if (csm > 0 && !done && wq0 < P.Nwo)
        wm = wall_row_cache<T, D, SWEEP_T>(P, wq0, pos, rho, nbr, cnt, ncap, threadIdx.x % WL, wcj, wcw, c_wsw, c_wgr);
    auto walls = [&](T* pbuf) {
        int q = wq0;
        if (wm >= 0) {
            wall_row_cached<T, SWEEP_T>(P, q, wm, wcj, wcw, c_wsw, c_wgr, pbuf, threadIdx.x % WL);
            q += wqs;
        }
        for (; q < P.Nwo; q += wqs)
            wall_pressure_row<T, D, true>(P, q, pos, rho, nbr, cnt, ncap, pbuf, threadIdx.x % WL);
    };
    // prologue: the walls of p^kit; then per iteration: sweep | walls of p^{k+1} (speculative:
    // after the last sweep they land in the final buffer's wall slots, which the solve's
    // epilogue overwrites with the walls the last sweep used) overlapped with the decision |
    if (!done) {
        T* pin = (kit & 1) ? pB : pA;
        walls(pin);
        pgrid_sync(gbar, (++nbar) * gridDim.x);
    }
    while (!done) {
        PPROF(0);
        const int par = kit & 1;
        T* pin = par ? pB : pA;
        T* pout = par ? pA : pB;
        double dn = 0.0, dd = 0.0;
        bool bad = false;
        if (tiled) {
            for (int t = threadIdx.x; t < nfs; t += blockDim.x) tile[t] = __ldcg(pin + f0 + t);
            for (int t = threadIdx.x; t < nws; t += blockDim.x) tile[nfs + t] = __ldcg(pin + w0 + t);
            __syncthreads();
        }
        int ifirst = gt;
        if constexpr (STORED) {
            if (cached) {
                // the cached row: same sums in entry order as sweep_row (pads add 0 x p_i)
                const int i = gt;
                const T pold = tile[i - f0];
                T pnew = c_fs == 2 ? pold : T(0);
                if (cn > 0) {
                    T s = 0;
                    const int nc = min(csm, (cn + 3) >> 2);
                    for (int c = 0; c < nc; c++) {
                        const ushort4 lv = *reinterpret_cast<const ushort4*>(cidx + ((size_t)c * SWEEP_T + threadIdx.x) * 4);
                        T f[4];
                        ld_chunk4_s(cfac + ((size_t)c * SWEEP_T + threadIdx.x) * 4, f);
                        const T p0 = tile[lv.x], p1 = tile[lv.y], p2 = tile[lv.z], p3 = tile[lv.w];
                        s += f[0] * p0;
                        s += f[1] * p1;
                        s += f[2] * p2;
                        s += f[3] * p3;
                    }
                    if (4 * csm < cn) {
                        // the rest of a long row from the list (tile gathers)
                        const size_t b = nb_base(i, ncap);
                        const int4* __restrict__ qi = reinterpret_cast<const int4*>(nbr + b);
                        for (int c = 4 * csm; c < cn; c += 4) {
                            const int4 v = __ldg(qi + (size_t)(c >> 2) * 32);
                            T f[4];
                            ld_chunk4_l1(coef + b + ((size_t)(c >> 2) * 32 << 2), f);
                            const int j0 = v.x, j1 = c + 1 < cn ? v.y : i, j2 = c + 2 < cn ? v.z : i, j3 = c + 3 < cn ? v.w : i;
                            s += f[0] * tile[j0 - (j0 < P.Nf ? f0 : wsh)];
                            s += (c + 1 < cn ? f[1] : T(0)) * tile[j1 - (j1 < P.Nf ? f0 : wsh)];
                            s += (c + 2 < cn ? f[2] : T(0)) * tile[j2 - (j2 < P.Nf ? f0 : wsh)];
                            s += (c + 3 < cn ? f[3] : T(0)) * tile[j3 - (j3 < P.Nf ? f0 : wsh)];
                        }
                    }
                    pnew = ppe_update(P, c_rhs, s, c_di, c_rhoi, pold);
                }
                pout[i] = pnew;
                dn += fabs((double)pnew - (double)pold);
                dd += c_fs == 2 ? 0.0 : fabs((double)pnew);
                bad = bad || !isfinite((double)pnew);
                ifirst = gt + gs;
            }
        }
        for (int i = ifirst; i < P.Nfo; i += gs) {
            const T pold = pin[i];
            T pnew;
            if constexpr (STORED && SISPH_PERS_B < 0) {
                pnew = tiled ? sweep_row_tile<T, -SISPH_PERS_B>(P, i, rho, fs, nbr, cnt, ncap, coef, rhs, diag, tile, f0, wsh)
                             : sweep_row<T, D, STORED, true, SISPH_PERS_B>(P, i, pos, rho, fs, nbr, cnt, ncap, coef, rhs, diag, pin, code, nslot, cc8);
            } else {
                pnew = sweep_row<T, D, STORED, true, SISPH_PERS_B>(P, i, pos, rho, fs, nbr, cnt, ncap, coef, rhs, diag, pin, code, nslot, cc8);
            }
            pout[i] = pnew;
            dn += fabs((double)pnew - (double)pold);
            dd += fs[i] == 2 ? 0.0 : fabs((double)pnew);
            bad = bad || !isfinite((double)pnew);
        }
        dn = warp_sum(dn);
        dd = warp_sum(dd);
        const int anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            sn[w] = dn;
            sd[w] = dd;
            if (anybad) atomicExch(&ctl->nonfinite, 1);
        }
        __syncthreads();
        double* part = partials + 2 * (size_t)gridDim.x * par;
        if (threadIdx.x == 0) {
            double a = 0, b = 0;
            for (int q = 0; q < SWEEP_T / 32; q++) {
                a += sn[q];
                b += sd[q];
            }
            part[2 * blockIdx.x] = a;
            part[2 * blockIdx.x + 1] = b;
        }
        __syncthreads();
        PPROF(1);
        pgrid_sync(gbar, (++nbar) * gridDim.x);
        PPROF(2);
        // the partials of this parity are next written two iterations on, after two more barriers
        double a = 0, b = 0;
        // the non-finite flag was raised (if at all) before the barrier: its L2 round trip runs
        // beside the wall rows instead of in front of the decision
        const int nonf = threadIdx.x == 0 ? __ldcg(&ctl->nonfinite) : 0;
        for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) {
            a += __ldcg(part + 2 * q);
            b += __ldcg(part + 2 * q + 1);
        }
        walls(pout);
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
            sn[w] = a;
            sd[w] = b;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double num = 0, den = 0;
            for (int q = 0; q < SWEEP_T / 32; q++) {
                num += sn[q];
                den += sd[q];
            }
            num *= dsc->cscale;
            den *= dsc->cscale;
            const double dmax = den > lam ? den : lam;
            const double res = num == 0.0 ? 0.0 : (dmax > 0.0 ? num / dmax : INFINITY);
            const int k1 = kit + 1;
            const int dn_ = ((k1 >= min_it && res < tol) || k1 >= max_it || nonf) ? 1 : 0;
            done_s = dn_;
            if (blockIdx.x == 0) {
                vc->residual = res;
                vc->iter = k1;
                vc->done = dn_;
            }
        }
        __syncthreads();
        done = done_s != 0;
        kit++;
        PPROF(3);
        if (!done) pgrid_sync(gbar, (++nbar) * gridDim.x);   // every block takes the same decision
        PPROF(4);
    }
#ifdef SISPH_PERS_PROF
    if (threadIdx.x == 0)
    {
        for (int k = 0; k < 5; k++) g_pers_prof[blockIdx.x * 6 + k] = tp[k];
        g_pers_prof[blockIdx.x * 6 + 5] = tiled ? (unsigned long long)(nfs + nws) : 0ull;
    }
#endif
#undef PPROF
}

// ===========================================================================
// A12 for small problems: ONE thread-block cluster (up to 16 SMs, one launch per solve)
// runs the whole PPE loop — wall pressures, the sweep, (R32) the live-row mean, the
// fixed-order reduction and the stop decision (R12/R12b, R13) — separated by hardware
// cluster barriers instead of kernel boundaries or a software grid barrier.  The block
// partials meet through distributed shared memory in block-rank order (deterministic);
// the pressures of other SMs are read L2-coherent (ldp<true>).  The row arithmetic is
// sweep_row / wall_pressure_row, the same as every other loop form.
// ===========================================================================
constexpr int CLUSTER_T = 1024;
template <class T, int D, bool STORED>
__global__ void __launch_bounds__(CLUSTER_T) k_ppe_cluster(Params<T> P, const PpeDesc<T>* __restrict__ dsc,
                                                           const T* __restrict__ rhs, const T* __restrict__ diag,
                                                           const int* __restrict__ cnt, int ncap, Ctl* ctl)
{
    cg::cluster_group cl = cg::this_cluster();
    const int nbk = (int)cl.num_blocks(), rk = (int)cl.block_rank();
    const int gt = rk * blockDim.x + threadIdx.x, gs = nbk * blockDim.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ double sa[32], sb[32];
    __shared__ double bp[2][2][2];   // [iteration parity][phase: sweep / R32 pass][a, b]: this block's partials
    __shared__ double red_s[2];      // the cluster sums, identical in every block
    __shared__ int bad_s[2][2];      // [parity][phase]: a non-finite value in this block
    __shared__ int badc_s;           // any block's (identical in every block)
    const V4<T>* __restrict__ pos = dsc->pos;
    const T* __restrict__ rho = dsc->rho;
    const uint8_t* __restrict__ fs = dsc->fs;
    const int* __restrict__ nbr = dsc->nbr;
    const T* __restrict__ coef = dsc->coef;
    const uint4* __restrict__ code = dsc->code;
    const int* __restrict__ nslot = dsc->nslot;
    const int cc8 = dsc->cc8;
    T* pA = dsc->pA;
    T* pB = dsc->pB;
    volatile Ctl* vc = ctl;
    if (threadIdx.x < 4) bad_s[threadIdx.x >> 1][threadIdx.x & 1] = 0;
    // fixed-order block reduction of (a, b) into dst (thread 0 writes); bflag: this phase's flag
    auto block_sum = [&](double a, double b, bool bad, double* dst, int* bflag) {
        a = warp_sum(a);
        b = warp_sum(b);
        const int anyb = __any_sync(0xffffffffu, bad);
        if (threadIdx.x == 0) *bflag = 0;
        __syncthreads();
        if (lane == 0) {
            sa[w] = a;
            sb[w] = b;
            if (anyb) atomicOr(bflag, 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double x = 0, y = 0;
            for (int q = 0; q < nw; q++) {
                x += sa[q];
                y += sb[q];
            }
            dst[0] = x;
            dst[1] = y;
        }
    };
    // after a cluster barrier: every block sums all blocks' partials in block-rank order (the
    // same result everywhere), so every block takes the same decision without a broadcast
    auto cluster_sum = [&](int par, int ph) {
        if (threadIdx.x == 0) {
            double A = 0, B = 0;
            int bad = 0;
            for (int r = 0; r < nbk; r++) {
                const double* q = cl.map_shared_rank(&bp[par][ph][0], r);
                A += q[0];
                B += q[1];
                bad |= *cl.map_shared_rank(&bad_s[par][ph], r);
            }
            red_s[0] = A;
            red_s[1] = B;
            badc_s |= bad;
            if (bad && rk == 0) vc->nonfinite = 1;
        }
        __syncthreads();
    };
    int kit = vc->iter;
    bool done = vc->done != 0;
    const double lam = __longlong_as_double((long long)vc->lambda_bits);
    if (threadIdx.x == 0) badc_s = vc->nonfinite ? 1 : 0;   // e.g. from A11's fused first sweep
    __syncthreads();
#ifdef SISPH_PERS_PROF
    unsigned long long tp[6] = {0, 0, 0, 0, 0, 0}, tq0 = 0, tq1 = 0;
#define CPROF(k) if (threadIdx.x == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq1)); if (k) tp[k - 1] += tq1 - tq0; tq0 = tq1; }
#else
#define CPROF(k)
#endif
    CPROF(0);
    while (!done) {
        const int par = kit & 1;
        const T* pin = par ? pB : pA;
        T* pout = par ? pA : pB;
        if (P.Nwo) {
            for (int t = gt; t < P.Nwo * WL; t += gs)
                wall_pressure_row<T, D, true>(P, t / WL, pos, rho, nbr, cnt, ncap, const_cast<T*>(pin), t % WL);
            cl.sync();
        }
        CPROF(1);
        double dn = 0.0, dd = 0.0;
        bool bad = false;
        auto row_done = [&](int i, T pold, T pnew) {
            pout[i] = pnew;
            if (P.mean_free) {
                const bool live = !fs[i] && diag[i] != T(0);
                dn += live ? (double)pnew : 0.0;
                dd += live ? 1.0 : 0.0;
            } else {
                dn += fabs((double)pnew - (double)pold);
                dd += fs[i] == 2 ? 0.0 : fabs((double)pnew);
            }
            bad = bad || !isfinite((double)pnew);
        };
        for (int i = gt; i < P.Nfo; i += gs) {
            const T pold = pin[i];
            const T pnew = sweep_row<T, D, STORED, true, SISPH_CLUSTER_B>(P, i, pos, rho, fs, nbr, cnt, ncap, coef, rhs,
                                                                         diag, pin, code, nslot, cc8);
            row_done(i, pold, pnew);
        }
        CPROF(2);
        block_sum(dn, dd, bad, &bp[par][0][0], &bad_s[par][0]);
        CPROF(3);
        cl.sync();
        CPROF(4);
        cluster_sum(par, 0);
        CPROF(5);
        double num = red_s[0], den = red_s[1];
        if (P.mean_free) {
            // R32: remove the live-row mean, then the residual sums of the corrected iterate
            const double mean = den > 0.0 ? num / den : 0.0;
            dn = dd = 0.0;
            bad = false;
            for (int i = gt; i < P.Nfo; i += gs) {
                T v = pout[i];
                if (!fs[i] && diag[i] != T(0)) {
                    v = (T)((double)v - mean);
                    pout[i] = v;
                }
                dn += fabs((double)v - (double)pin[i]);
                dd += fs[i] == 2 ? 0.0 : fabs((double)v);
                bad = bad || !isfinite((double)v);
            }
            block_sum(dn, dd, bad, &bp[par][1][0], &bad_s[par][1]);
            cl.sync();
            cluster_sum(par, 1);
            num = red_s[0];
            den = red_s[1];
        }
        num *= dsc->cscale;
        den *= dsc->cscale;
        const double dmax = den > lam ? den : lam;
        const double res = num == 0.0 ? 0.0 : (dmax > 0.0 ? num / dmax : INFINITY);
        kit += 1;
        done = (kit >= dsc->min_it && res < dsc->tol) || kit >= dsc->max_it || badc_s;
        if (rk == 0 && threadIdx.x == 0) {
            vc->residual = res;
            vc->iter = kit;
            vc->done = done ? 1 : 0;
        }
        CPROF(6);
    }
#ifdef SISPH_PERS_PROF
    // phases per iteration: walls | sweep | block sum | cluster barrier | cluster sum | R32 + decision
    if (threadIdx.x == 0)
        for (int k = 0; k < 6; k++) g_pers_prof[rk * 6 + k] = tp[k];
#endif
#undef CPROF
}

// ===========================================================================
// A13: pressure gradient (eq:mom:sph:press:symm / :pij, R18) and corrector
// u^{n+1} = u* + dt f_p (eq:int:vnp1).  Sources fluid + wall.
// ===========================================================================
template <class T, int D>
__global__ void __launch_bounds__(128) k_pgrad_correct(Params<T> P, T dt, const V4<T>* __restrict__ pos,
                                                       const T* __restrict__ rho, const T* __restrict__ p,
                                                       const V4<T>* __restrict__ us, const int* __restrict__ nbr,
                                                       const int* __restrict__ cnt, int ncap, V4<T>* __restrict__ vel,
                                                       const V4<T>* __restrict__ fnp, Ctl* ctl)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double f2 = 0.0;
    if (i < P.Nfo) {
        V4<T> xi = ld4(pos + i);
        T rhoi = rho[i], pi = p[i];
        T irhoi = frcp(rhoi);
        T pir = pi * irhoi * irhoi;
        T ax = 0, ay = 0, az = 0;
        int n = cnt[i];
        if (P.ptype && P.ptype[i] != 0) n = 0;       // R34: inlet / outlet keep u* = u
        for_nbrs_pfx<SISPH_PGRAD_PF>(nbr, ncap, i, n, [&](int j) {
            V4<T> xj = ld4(pos + j);
            T rhoj = __ldg(rho + j), pj = __ldg(p + j);
            T d[3], r, ri;
            r_of(pair_vec<T, D>(P, xi, xj, d), r, ri);
            T gf = quintic4(r * P.inv_h) * ri;       // * dwk below
            T irj = frcp(rhoj);
            T f = P.pgrad == 0 ? xj.w * (pir + pj * irj * irj) : xj.w * irhoi * irj * (pj - pi);
            f *= gf;
            ax -= f * d[0];
            ay -= f * d[1];
            if (D == 3) az -= f * d[2];
        });
        ax *= P.dwk;
        ay *= P.dwk;
        az *= P.dwk;
        V4<T> u = ld4(us + i);
        vel[i] = mk4<T>(u.x + dt * ax, u.y + dt * ay, D == 3 ? u.z + dt * az : T(0), T(0));
        // f^n = f_p + f_visc + f_body + f_avisc + f_astress for the adaptive dt
        const V4<T> a = ld4(fnp + i);
        const double fx = (double)(a.x + ax), fy = (double)(a.y + ay), fz = D == 3 ? (double)(a.z + az) : 0.0;
        f2 = fx * fx + fy * fy + fz * fz;
    }
    warp_max_to(f2, &ctl->fmax2_bits);
}

// ===========================================================================
// A14: one modified-GTVF sub-step (eq:int:gtvf:pos, eq:int:gtvf:vel:tmp) with
// f_GTVF(r^k) = -p0_i sum_j m_j / rho_j^2 gradW(r^k_ij, h~) (eq:mom:sph:gtvf)
// over the pair set frozen at r* (P:454-456).  p0 per P:389-390 / R22.
// ===========================================================================
// rk0 = (r*, m / rho^2) for all particles: the GTVF weight of a source is
// constant through the sub-steps (rho frozen at stage 1, R5), so it rides in
// the position vector's 4th lane and costs no extra gather.
template <class T>
__global__ void k_gtvf_prep(const V4<T>* __restrict__ pos, const T* __restrict__ rho, int n, T* __restrict__ a,
                            T* __restrict__ b)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V4<T> x = ld4(pos + i);
    const T r = rho[i];
    // {r^0 = r*, m / rho^2 (eq:mom:sph:gtvf), delta^0 = 0, 0}
    const T z[8] = {x.x, x.y, x.z, x.w / (r * r), T(0), T(0), T(0), T(0)};
    st8(a + 8 * (size_t)i, z);
    if (b) st8(b + 8 * (size_t)i, z);
}

#ifndef SISPH_GTVF_PF
#define SISPH_GTVF_PF 1   // B200, C5: PD 0 / 1 / 2 / 3 -> 113 / 107 / 125 / 120 us per sub-step
#endif
// fp32 GTVF sub-steps on fixed-point positions (round 2): the sub-step record is 16 bytes,
// {x, y, z as 32-bit fixed point of the local box, m / rho^2}, so a neighbour costs one 128-bit
// gather; the pair difference is an exact integer subtraction of the fixed-point r^k converted
// with the axis scale (quantisation 2e-7 h on C5: the GTVF force sums, which cancel to ~1e-3
// of their terms on near-lattices, keep ~1e-6 relative).  r^k_fix = r*_fix + round(delta^k /
// fxs); delta^k (fp32, the recursion of eq:int:gtvf:pos) and the velocity live per particle.
__device__ __forceinline__ unsigned fix_coord(double x, double lo, double s)
{
    return (unsigned)(unsigned long long)(long long)llrint((x - lo) / s);
}

template <int D>
__global__ void k_gtvf_prep_fx(Params<float> P, const float4* __restrict__ pos, const float* __restrict__ rho, int n,
                               int4* __restrict__ a, int4* __restrict__ b, int4* __restrict__ fix0,
                               float4* __restrict__ dk)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 x = ld4(pos + i);
    const float r = rho[i];
    const int4 f = make_int4((int)fix_coord(x.x, P.lo[0], P.fxs[0]), (int)fix_coord(x.y, P.lo[1], P.fxs[1]),
                             D == 3 ? (int)fix_coord(x.z, P.lo[2], P.fxs[2]) : 0, __float_as_int(x.w / (r * r)));
    a[i] = f;
    b[i] = f;
    fix0[i] = f;
    dk[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ISO (every axis has the same fixed-point unit, e.g. a periodic cube): the pair sum is taken in
// fixed-point units, d / r is the same direction and q = r_units * (unit / h~), three multiplies
// per pair fewer.  Rows are walked in whole 4-entry chunks: entries past the row end are the row
// itself, d = 0, q = 0 and quintic4(0) = 81 - 6 * 16 + 15 = 0 exactly, so they add +0 and the
// loop has no per-entry branch (B200, C4 TGV-3D with h~ = h: 408 us per sub-step before).
template <int D, bool ISO>
__global__ void __launch_bounds__(128) k_gtvf_substep_fx(Params<float> P, float dtau, const int4* __restrict__ rk,
                                                         int4* __restrict__ rk1, const int4* __restrict__ fix0,
                                                         float4* __restrict__ dk, float4* __restrict__ vk,
                                                         const float* __restrict__ p, const int* __restrict__ nbr,
                                                         int ncap, const int* __restrict__ cnt, int first, int check,
                                                         Ctl* ctl, const int* __restrict__ rows,
                                                         const int* __restrict__ nrows)
{
    // rows == nullptr: every owned fluid row; else the rows rows[0 .. *nrows) (slab ranks)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (nrows ? *nrows : P.Nfo)) return;
    const int i = rows ? rows[t] : t;
    const int4 ri = __ldg(rk + i);
    float ax = 0.f, ay = 0.f, az = 0.f;
    int n = cnt[i];
    if (P.ptype && P.ptype[i] != 0) n = 0;           // R34: no GTVF shift for inlet / outlet
    const float s0 = ISO ? 1.f : P.fxf[0], s1 = ISO ? 1.f : P.fxf[1], s2 = ISO ? 1.f : P.fxf[2];
    const float qs = ISO ? P.fxf[0] * P.inv_ht : P.inv_ht;
    auto pair = [&](int j) {
        const int4 rj = __ldg(rk + j);
        const float d0 = (float)(ri.x - rj.x) * s0, d1 = (float)(ri.y - rj.y) * s1;
        const float d2 = D == 3 ? (float)(ri.z - rj.z) * s2 : 0.f;
        float r2 = d0 * d0 + d1 * d1;
        if (D == 3) r2 += d2 * d2;
        float r, rinv;
        r_of(r2, r, rinv);
        const float f = __int_as_float(rj.w) * quintic4(r * qs) * rinv;   // m_j / rho_j^2 |gradW| / r
        ax += f * d0;
        ay += f * d1;
        if (D == 3) az += f * d2;
    };
    {
        const int4* __restrict__ q = reinterpret_cast<const int4*>(nbr + nb_base(i, ncap));
        int4 nx = n > 0 ? LDLIST(q) : make_int4(i, i, i, i);
        for (int c = 0; c < n; c += 4) {
            const int4 v = nx;
            nx = c + 4 < n ? LDLIST(q + (size_t)((c + 4) >> 2) * 32) : make_int4(i, i, i, i);
            pair(v.x);
            pair(c + 1 < n ? v.y : i);
            pair(c + 2 < n ? v.z : i);
            pair(c + 3 < n ? v.w : i);
        }
    }
    float p0 = P.p_ref;
    if (P.pref_external) {
        const float v = 10.f * fabsf(p[i]);
        p0 = v < P.p_ref ? v : P.p_ref;
    }
    const float sc = -p0 * P.dwkt;
    ax *= sc;
    ay *= sc;
    az *= sc;
    const float4 v = first ? make_float4(0.f, 0.f, 0.f, 0.f) : ld4(vk + i);
    const float4 dl = ld4(dk + i);
    const float h2 = 0.5f * dtau * dtau;
    const float4 dn = make_float4(dl.x + dtau * v.x + h2 * ax, dl.y + dtau * v.y + h2 * ay,
                                  D == 3 ? dl.z + dtau * v.z + h2 * az : 0.f, 0.f);
    dk[i] = dn;
    vk[i] = make_float4(v.x + dtau * ax, v.y + dtau * ay, D == 3 ? v.z + dtau * az : 0.f, 0.f);
    const int4 f0 = __ldg(fix0 + i);
    rk1[i] = make_int4(f0.x + __float2int_rn(dn.x / P.fxf[0]), f0.y + __float2int_rn(dn.y / P.fxf[1]),
                       D == 3 ? f0.z + __float2int_rn(dn.z / P.fxf[2]) : 0, ri.w);
    if (check && dn.x * dn.x + dn.y * dn.y + dn.z * dn.z > P.skin_half2) atomicExch(&ctl->gtvf_far, 1);
}

// slab ranks: flag[idx[t]] = 1 (the rows of the halo send lists)
__global__ void k_set_flag(const int* __restrict__ idx, int n, int* __restrict__ flag)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) flag[idx[t]] = 1;
}
// stable split of [0, n) by flag (pre = exclusive scan of flag): flagged rows to brow, the
// others to irow; cnt = {#flagged, #others}
__global__ void k_split_rows(const int* __restrict__ f, const int* __restrict__ pre, int n, int* __restrict__ brow,
                             int* __restrict__ irow, int* __restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (f[i]) brow[pre[i]] = i;
    else irow[i - pre[i]] = i;
    if (i == n - 1) {
        cnt[0] = pre[i] + f[i];
        cnt[1] = n - cnt[0];
    }
}

// slab ranks: the ghosts' fixed-point r^k from their owners' delta^k (halo-exchanged)
__global__ void k_gtvf_ghost_fx(int base, int n, const int4* __restrict__ fix0, const float4* __restrict__ dk,
                                const int4* __restrict__ rk, int4* __restrict__ rk1, float s0, float s1, float s2,
                                int three)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = base + q;
    const int4 f0 = fix0[i];
    const float4 dn = dk[i];
    rk1[i] = make_int4(f0.x + __float2int_rn(dn.x / s0), f0.y + __float2int_rn(dn.y / s1),
                       three ? f0.z + __float2int_rn(dn.z / s2) : 0, rk[i].w);
}

// slab ranks, fused: the received delta^k records of both faces (face 0 first,
// slot grecv[t]) go to dk and straight into the ghosts' fixed-point r^k
__global__ void k_unpack_gtvf_fx(const int* __restrict__ map, int n0, int n1, const float4* __restrict__ buf0,
                                 const float4* __restrict__ buf1, const int4* __restrict__ fix0,
                                 float4* __restrict__ dk, const int4* __restrict__ rk, int4* __restrict__ rk1, float s0,
                                 float s1, float s2, int three)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n0 + n1) return;
    const float4 dn = t < n0 ? buf0[t] : buf1[t - n0];
    const int i = map[t];
    dk[i] = dn;
    const int4 f0 = fix0[i];
    rk1[i] = make_int4(f0.x + __float2int_rn(dn.x / s0), f0.y + __float2int_rn(dn.y / s1),
                       three ? f0.z + __float2int_rn(dn.z / s2) : 0, rk[i].w);
}

// nbr/stride/cnt select the full r* list or the inner list (pairs with
// r* < 3 h~ + skin).  With the inner list, a particle that has moved more
// than skin/2 from r* raises ctl->gtvf_far and the host repeats the
// sub-steps on the full list (exact either way).
// A particle's sub-step record is {r^0 = r*, m / rho^2, delta^k = r^k - r^0, 0}
// (the recursion of eq:int:gtvf:pos carried on delta), read with ONE 256-bit
// load per neighbour.  A pair's r^k_ij is (r^0_i - r^0_j) + (delta^k_i - delta^k_j):
// the difference of the two r* is exact for neighbours (Sterbenz), so the GTVF
// force sees the geometry to the working precision of r_ij itself, not to the
// ulp of the coordinates (fp32 at |x| ~ 3 with h = 1/256: 6e-5 h), and
// eq:int:vhatnp2's (r^K - r^0)/dt keeps its digits.
template <class T, int D>
__global__ void __launch_bounds__(128) k_gtvf_substep(Params<T> P, T dtau, const T* __restrict__ rk,
                                                      T* __restrict__ rk1, V4<T>* __restrict__ vk,
                                                      const T* __restrict__ p, const int* __restrict__ nbr, int ncap,
                                                      const int* __restrict__ cnt, int first, int check, Ctl* ctl)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.Nfo) return;
    T ri8[8];
    ld8(rk + 8 * (size_t)i, ri8);
    const V4<T> xi = mk4<T>(ri8[0], ri8[1], ri8[2], ri8[3]);
    T ax = 0, ay = 0, az = 0;
    int n = cnt[i];
    if (P.ptype && P.ptype[i] != 0) n = 0;           // R34: no GTVF shift for inlet / outlet
    for_nbrs_pf<SISPH_GTVF_PF>(nbr, ncap, i, n, [&](int j) {
        T rj8[8];
        ld8(rk + 8 * (size_t)j, rj8);
        const V4<T> xj = mk4<T>(rj8[0], rj8[1], rj8[2], rj8[3]);
        T d[3], r, ri;
        pair_vec<T, D>(P, xi, xj, d);
        d[0] += ri8[4] - rj8[4];
        d[1] += ri8[5] - rj8[5];
        d[2] = D == 3 ? d[2] + (ri8[6] - rj8[6]) : T(0);
        T r2 = d[0] * d[0] + d[1] * d[1];
        if (D == 3) r2 += d[2] * d[2];
        r_of(r2, r, ri);
        T f = rj8[3] * quintic4(r * P.inv_ht) * ri;   // m_j / rho_j^2 * |gradW| / r (dwkt below)
        ax += f * d[0];
        ay += f * d[1];
        if (D == 3) az += f * d[2];
    });
    T p0 = P.p_ref;
    if (P.pref_external) {
        T v = T(10) * fabs(p[i]);
        p0 = v < P.p_ref ? v : P.p_ref;
    }
    const T s = -p0 * P.dwkt;
    ax *= s;
    ay *= s;
    az *= s;
    const V4<T> zero = mk4<T>(T(0), T(0), T(0), T(0));
    const V4<T> v = first ? zero : ld4(vk + i);
    const T h2 = T(0.5) * dtau * dtau;
    const T o8[8] = {ri8[0], ri8[1], ri8[2], ri8[3], ri8[4] + dtau * v.x + h2 * ax, ri8[5] + dtau * v.y + h2 * ay,
                     D == 3 ? ri8[6] + dtau * v.z + h2 * az : T(0), T(0)};
    st8(rk1 + 8 * (size_t)i, o8);
    vk[i] = mk4<T>(v.x + dtau * ax, v.y + dtau * ay, D == 3 ? v.z + dtau * az : T(0), T(0));
    if (check && o8[4] * o8[4] + o8[5] * o8[5] + o8[6] * o8[6] > P.skin_half2) atomicExch(&ctl->gtvf_far, 1);
}

// ===========================================================================
// A15: transport velocity (eq:int:vhatnp2) and positions from r^n
// (eq:int:rnp2, R24), periodic wrap.
// ===========================================================================
template <class T, int D>
__global__ void k_advance(Params<T> P, T dt, const T* __restrict__ dK, int dstride, const V4<T>* __restrict__ rn,
                          const V4<T>* __restrict__ vel, V4<T>* __restrict__ pos, V4<T>* __restrict__ vt, Ctl* ctl,
                          const T* __restrict__ uout)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double v2 = 0.0;
    const int ptp = (P.ptype && i < P.Nfo) ? P.ptype[i] : 0;
    if (ptp == 2) {
        // R34 inlet: r^{n+1} = r^n + dt u (prescribed), u~ = u
        const V4<T> x = ld4(rn + i), u = ld4(vel + i);
        T X = x.x + dt * u.x, Y = x.y + dt * u.y, Z = D == 3 ? x.z + dt * u.z : x.z;
        if (P.per[1]) { if (Y >= P.hi[1]) Y -= P.L[1]; else if (Y < P.lo[1]) Y += P.L[1]; }
        if (D == 3 && P.per[2]) { if (Z >= P.hi[2]) Z -= P.L[2]; else if (Z < P.lo[2]) Z += P.L[2]; }
        pos[i] = mk4<T>(X, Y, Z, x.w);
        vt[i] = mk4<T>(u.x, u.y, D == 3 ? u.z : T(0), T(0));
    } else if (ptp == 3) {
        // R34 outlet: moved along x with the extrapolated fluid u_x; u, p frozen
        const V4<T> x = ld4(rn + i);
        const T ux = uout[i];
        pos[i] = mk4<T>(x.x + dt * ux, x.y, x.z, x.w);
        vt[i] = mk4<T>(ux, T(0), T(0), T(0));
    } else if (i < P.Nfo) {
        V4<T> x = ld4(rn + i), u = ld4(vel + i), ut = ld4(vt + i);
        // r^K - r^0: the second half of the GTVF record (k_gtvf_substep)
        // r^K - r^0: fp32 the delta array (stride 4), fp64 the second half of the GTVF record (stride 8)
        const V4<T> dl = dK ? ld4(reinterpret_cast<const V4<T>*>(dK + (size_t)dstride * i + (dstride - 4)))
                            : mk4<T>(T(0), T(0), T(0), T(0));
        T tx = u.x + dl.x / dt, ty = u.y + dl.y / dt;
        T tz = D == 3 ? u.z + dl.z / dt : T(0);
        T hd = T(0.5) * dt;
        T X = x.x + hd * (tx + ut.x), Y = x.y + hd * (ty + ut.y), Z = D == 3 ? x.z + hd * (tz + ut.z) : x.z;
        if (P.per[0]) { if (X >= P.hi[0]) X -= P.L[0]; else if (X < P.lo[0]) X += P.L[0]; }
        if (P.per[1]) { if (Y >= P.hi[1]) Y -= P.L[1]; else if (Y < P.lo[1]) Y += P.L[1]; }
        if (D == 3 && P.per[2]) { if (Z >= P.hi[2]) Z -= P.L[2]; else if (Z < P.lo[2]) Z += P.L[2]; }
        pos[i] = mk4<T>(X, Y, Z, x.w);
        vt[i] = mk4<T>(tx, ty, tz, T(0));
        v2 = (double)u.x * u.x + (double)u.y * u.y + (D == 3 ? (double)u.z * u.z : 0.0);   // |u^{n+1}|^2
    }
    warp_max_to(v2, &ctl->vmax2_bits);
}

// ===========================================================================
// R34 open boundaries
// ===========================================================================
// the outlet's advection velocity: Shepard_h of the fluid's u_x^{n+1} at r* (the
// exact r* list; none in the support: the frozen u_x)
template <class T, int D>
__global__ void k_outlet_velocity(Params<T> P, const V4<T>* __restrict__ rn, const V4<T>* __restrict__ vel,
                                  const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap,
                                  T* __restrict__ uout)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.Nfo || P.ptype[i] != 3) return;
    const V4<T> xi = ld4(rn + i);
    T sw = 0, su = 0;
    for_nbrs(nbr, cnt ? ncap : 0, i, cnt ? cnt[i] : 0, [&](int j) {
        if (j >= P.Nf || P.ptype[j] != 0) return;
        T d[3], r, ri;
        const T r2 = pair_vec<T, D>(P, xi, ld4(rn + j), d);
        if (r2 >= P.R2cut) return;                    // W = 0 beyond 3h (loose list)
        r_of(r2, r, ri);
        const T w = P.sig * quintic5(r * P.inv_h);
        su += vel[j].x * w;
        sw += w;
    });
    uout[i] = sw > T(0) ? su / sw : vel[i].x;
}

// conversions after the position update, on the pre-step types:
//   outlet with x >= x_end -> deleted (flag 1); fluid with x >= x_outlet -> outlet;
//   inlet with x >= x_inlet -> fluid and spawns one inlet particle (flag 2)
template <class T>
__global__ void k_open_classify(Params<T> P, const V4<T>* __restrict__ pos, uint8_t* __restrict__ ptype,
                                int* __restrict__ flag)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.Nfo) return;
    const int ty = ptype[i];
    const T x = pos[i].x;
    int f = 0;
    if (ty == 3 && x >= P.x_end) {
        f = 1;
    } else if (ty == 0 && x >= P.x_outlet) {
        ptype[i] = 3;
    } else if (ty == 2 && x >= P.x_inlet) {
        ptype[i] = 0;
        f = 2;
    }
    flag[i] = f;
}

// new inlet rows [base, base + n): copies of the spawning rows src[k] (pre-compaction
// arrays), one inlet length upstream, with the ids drawn from the pool
template <class T>
__global__ void k_open_spawn(Params<T> P, int base, int n, const int* __restrict__ src,
                             const int* __restrict__ newid, const V4<T>* __restrict__ pos0,
                             const V4<T>* __restrict__ vel0, const T* __restrict__ p0, const T* __restrict__ rho0,
                             V4<T>* __restrict__ pos, V4<T>* __restrict__ vel, V4<T>* __restrict__ vt,
                             T* __restrict__ p, T* __restrict__ rho, int* __restrict__ pid, uint8_t* __restrict__ ptype)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = src[k], d = base + k;
    V4<T> x = pos0[s];
    x.x = x.x - P.inlet_length;
    pos[d] = x;
    const V4<T> u = vel0[s];
    vel[d] = u;
    vt[d] = mk4<T>(u.x, u.y, u.z, T(0));
    p[d] = p0[s];
    rho[d] = rho0[s];
    pid[d] = newid[k];
    ptype[d] = 2;
}

// ===========================================================================
// A0: wall normals (§3.4.1, eq:normal-approx / eq:normal, R17), at create.
// ===========================================================================
template <class T, int D>
__global__ void k_normals_raw(Params<T> P, const V4<T>* __restrict__ pos, const T* __restrict__ rho,
                              const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap, V4<T>* __restrict__ ns)
{
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= P.Nwo) return;
    int i = P.Nf + w;
    V4<T> xi = ld4(pos + i);
    T ax = 0, ay = 0, az = 0;
    int n = cnt[i];
    for_nbrs(nbr, ncap, i, n, [&](int j) {
        if (j < P.Nf) return;
        V4<T> xj = ld4(pos + j);
        T d[3];
        T r = my_sqrt(pair_vec<T, D>(P, xi, xj, d));
        T gf = r > T(0) ? P.dwk * quintic4(r * P.inv_h) / r : T(0);
        T v = xj.w / rho[j] * gf;
        ax -= v * d[0];
        ay -= v * d[1];
        if (D == 3) az -= v * d[2];
    });
    T mag = my_sqrt(ax * ax + ay * ay + az * az);
    if (mag < T(1) / (T(4) * P.h)) ax = ay = az = T(0);
    else {
        ax /= mag;
        ay /= mag;
        az /= mag;
    }
    ns[w] = mk4<T>(ax, ay, az, T(0));
}

template <class T, int D>
__global__ void k_normals_smooth(Params<T> P, const V4<T>* __restrict__ pos, const T* __restrict__ rho,
                                 const int* __restrict__ nbr, const int* __restrict__ cnt, int ncap,
                                 const V4<T>* __restrict__ ns, V4<T>* __restrict__ nrm)
{
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= P.Nwo) return;
    int i = P.Nf + w;
    V4<T> xi = ld4(pos + i);
    T v0 = xi.w / rho[i] * P.w0;
    V4<T> n0 = ns[w];
    T ax = v0 * n0.x, ay = v0 * n0.y, az = v0 * n0.z;
    int n = cnt[i];
    for_nbrs(nbr, ncap, i, n, [&](int j) {
        if (j < P.Nf) return;
        V4<T> xj = ld4(pos + j);
        T d[3];
        T r = my_sqrt(pair_vec<T, D>(P, xi, xj, d));
        T v = xj.w / rho[j] * (P.sig * quintic5(r * P.inv_h));
        V4<T> nj = ns[j - P.Nf];
        ax += v * nj.x;
        ay += v * nj.y;
        az += v * nj.z;
    });
    // R17: a smoothed vector shorter than 0.01 (layers cancelling) has no direction -> 0
    T mag = my_sqrt(ax * ax + ay * ay + az * az);
    if (mag >= T(0.01)) {
        ax /= mag;
        ay /= mag;
        az /= mag;
    } else {
        ax = ay = az = T(0);
    }
    nrm[w] = mk4<T>(ax, ay, az, T(0));
}

// ===========================================================================
// Slab decomposition: classification, compaction and
// pack / unpack of halo and migration records.
// ===========================================================================
// wrap the slab-axis coordinate of owned fluid into the global periodic box
// and classify: 0 stays, 1 leaves across the low face, 2 across the high face
template <class T>
__global__ void k_classify(V4<T>* __restrict__ pos, int n, int axis, double slab_lo, double slab_hi, double glo,
                           double ghi, int gper, int has_lo, int has_hi, int* __restrict__ flag,
                           int* __restrict__ nout)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    // nout[0] / nout[1]: how many leave through face 0 / 1 (warp-aggregated counts)
    int fl = 0;
    if (i < n) {
        const double y = (double)reinterpret_cast<const T*>(pos + i)[axis];
        fl = (has_lo && y < slab_lo) ? 1 : ((has_hi && y >= slab_hi) ? 2 : 0);
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, fl == 1), m2 = __ballot_sync(0xffffffffu, fl == 2);
    if ((threadIdx.x & 31) == 0) {
        if (m1) atomicAdd(nout, __popc(m1));
        if (m2) atomicAdd(nout + 1, __popc(m2));
    }
    if (i >= n) return;
    V4<T> x = ld4(pos + i);
    T* c = reinterpret_cast<T*>(&x);
    // the face is decided on the unwrapped coordinate (a particle leaving the
    // first slab downwards goes to the last slab), the stored position is wrapped
    const double y = (double)c[axis];
    flag[i] = fl;
    if (gper) {
        const T L = (T)(ghi - glo);
        if (y >= ghi) c[axis] -= L;
        else if (y < glo) c[axis] += L;
        pos[i] = x;
    }
}

// halo selection: owned particles within G of the low / high face
template <class T>
__global__ void k_halo_flags(const V4<T>* __restrict__ pos, int n, int axis, double slab_lo, double slab_hi, double G,
                             int has_lo, int has_hi, int* __restrict__ flo, int* __restrict__ fhi)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    V4<T> x = ld4(pos + i);
    const double y = (double)reinterpret_cast<const T*>(&x)[axis];
    flo[i] = has_lo && y < slab_lo + G ? 1 : 0;
    fhi[i] = has_hi && y >= slab_hi - G ? 1 : 0;
}

__global__ void k_flag_eq(const int* __restrict__ flag, int n, int v, int* __restrict__ out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = flag[i] == v ? 1 : 0;
}

// stable compaction: out[pre[i]] = i for flagged i (pre = exclusive scan of f)
__global__ void k_compact(const int* __restrict__ f, const int* __restrict__ pre, int n, int* __restrict__ out,
                          int* __restrict__ count)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (f[i]) out[pre[i]] = i;
    if (i == n - 1) *count = pre[i] + f[i];
}

__global__ void k_invperm(const int* __restrict__ perm, int n, int* __restrict__ inv)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) inv[perm[t]] = t;
}

// out[q] = inv[list ? list[q] : base + q]
__global__ void k_remap(const int* __restrict__ list, int base, int n, const int* __restrict__ inv, int* __restrict__ out)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) out[q] = inv[list ? list[q] : base + q];
}

// records of up to 8 fields (4-byte multiples first, 1-byte fields last);
// a field marked shift is a position vector whose slab-axis component gets
// the face's periodic image shift
struct PackList {
    int nf, rec, axis;
    double shift;
    void* ptr[8];
    int size[8];
    int sh[8];
};

template <class T>
__global__ void k_pack(PackList L, const int* __restrict__ idx, int base, int n, char* __restrict__ buf)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int s = idx ? idx[q] : base + q;
    char* r = buf + (size_t)q * L.rec;
    int off = 0;
    for (int f = 0; f < L.nf; f++) {
        const int sz = L.size[f];
        const char* src = (const char*)L.ptr[f] + (size_t)s * sz;
        if (sz == 1) {
            r[off] = *src;
        } else {
            for (int w = 0; w < sz / 4; w++) reinterpret_cast<int*>(r + off)[w] = reinterpret_cast<const int*>(src)[w];
            if (L.sh[f]) reinterpret_cast<T*>(r + off)[L.axis] += (T)L.shift;
        }
        off += sz;
    }
}

// the wall blocks of up to 16 arrays moved in two launches (to a staging
// buffer and back at the new offset; the ranges may overlap): grid.y = array,
// one thread per 4-byte word
struct MoveList {
    int n;
    char* ptr[16];
    int esz[16];
    size_t toff[16];
};
__global__ void k_move_block(MoveList M, int from, int nw, char* __restrict__ tmp, int to_tmp)
{
    const int a = blockIdx.y;
    if (a >= M.n) return;
    const int words = nw * (M.esz[a] >> 2);
    int* blk = reinterpret_cast<int*>(M.ptr[a] + (size_t)from * M.esz[a]);
    int* stg = reinterpret_cast<int*>(tmp + M.toff[a]);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < words; t += gridDim.x * blockDim.x) {
        if (to_tmp) stg[t] = blk[t];
        else blk[t] = stg[t];
    }
}

// both faces of one exchange in one launch: records q < n0 go to face 0's buffer
// (idx0, periodic shift sh0), the rest to face 1's
template <class T>
__global__ void k_pack2(PackList L, double sh0, double sh1, const int* __restrict__ idx0,
                        const int* __restrict__ idx1, int n0, int n1, char* __restrict__ buf0,
                        char* __restrict__ buf1)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n0 + n1) return;
    const bool f1 = t >= n0;
    const int q = f1 ? t - n0 : t;
    const int* idx = f1 ? idx1 : idx0;
    const int s = idx[q];
    char* r = (f1 ? buf1 : buf0) + (size_t)q * L.rec;
    const T shift = (T)(f1 ? sh1 : sh0);
    int off = 0;
    for (int f = 0; f < L.nf; f++) {
        const int sz = L.size[f];
        const char* src = (const char*)L.ptr[f] + (size_t)s * sz;
        if (sz == 1) {
            r[off] = *src;
        } else {
            for (int w = 0; w < sz / 4; w++) reinterpret_cast<int*>(r + off)[w] = reinterpret_cast<const int*>(src)[w];
            if (L.sh[f]) reinterpret_cast<T*>(r + off)[L.axis] += shift;
        }
        off += sz;
    }
}

// both faces' received records in one launch (face 0's first: slots map[t] or base + t)
template <class T>
__global__ void k_unpack2(PackList L, const int* __restrict__ map, int base, int n0, int n1,
                          const char* __restrict__ buf0, const char* __restrict__ buf1)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n0 + n1) return;
    const bool f1 = t >= n0;
    const int q = f1 ? t - n0 : t;
    const int s = map ? map[t] : base + t;
    const char* r = (f1 ? buf1 : buf0) + (size_t)q * L.rec;
    int off = 0;
    for (int f = 0; f < L.nf; f++) {
        const int sz = L.size[f];
        char* dst = (char*)L.ptr[f] + (size_t)s * sz;
        if (sz == 1) {
            *dst = r[off];
        } else {
            for (int w = 0; w < sz / 4; w++) reinterpret_cast<int*>(dst)[w] = reinterpret_cast<const int*>(r + off)[w];
        }
        off += sz;
    }
}

template <class T>
__global__ void k_unpack(PackList L, const int* __restrict__ map, int base, int n, const char* __restrict__ buf)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int s = map ? map[q] : base + q;
    const char* r = buf + (size_t)q * L.rec;
    int off = 0;
    for (int f = 0; f < L.nf; f++) {
        const int sz = L.size[f];
        char* dst = (char*)L.ptr[f] + (size_t)s * sz;
        if (sz == 1) {
            *dst = r[off];
        } else {
            for (int w = 0; w < sz / 4; w++) reinterpret_cast<int*>(dst)[w] = reinterpret_cast<const int*>(r + off)[w];
        }
        off += sz;
    }
}

// ===========================================================================
// host <-> device marshalling in creation-id order
// ===========================================================================
// vector field: dst[slot] = src[id[slot]] (id order -> internal order)
template <class T, class H>
__global__ void k_from_ids_vec(const H* __restrict__ src, const int* __restrict__ id, int n, int dim,
                               V4<T>* __restrict__ dst, int keep_w)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const H* v = src + (size_t)id[s] * dim;
    V4<T> o = dst[s];
    o.x = (T)v[0];
    o.y = (T)v[1];
    o.z = dim == 3 ? (T)v[2] : T(0);
    if (!keep_w) o.w = T(0);
    dst[s] = o;
}
template <class T, class H>
__global__ void k_to_ids_vec(const V4<T>* __restrict__ src, const int* __restrict__ id, int n, int dim,
                             H* __restrict__ dst)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    V4<T> o = src[s];
    H* v = dst + (size_t)id[s] * dim;
    v[0] = (H)o.x;
    v[1] = (H)o.y;
    if (dim == 3) v[2] = (H)o.z;
}
template <class T, class H>
__global__ void k_from_ids_w(const H* __restrict__ src, const int* __restrict__ id, int n,
                             V4<T>* __restrict__ dst)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    dst[s].w = (T)src[id[s]];
}
template <class T, class H>
__global__ void k_to_ids_w(const V4<T>* __restrict__ src, const int* __restrict__ id, int n, H* __restrict__ dst)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    dst[id[s]] = (H)src[s].w;
}
template <class T, class S, class H>
__global__ void k_from_ids_sc(const H* __restrict__ src, const int* __restrict__ id, int n, S* __restrict__ dst)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    dst[s] = (S)src[id[s]];
}
template <class S, class H>
__global__ void k_to_ids_sc(const S* __restrict__ src, const int* __restrict__ id, int n, H* __restrict__ dst)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    dst[id[s]] = (H)src[s];
}
// has any owned wall's position (creation-id order input, working precision)
// changed?  (set_field(POSITION): the wall geometry is static unless it does)
template <class T, class H>
__global__ void k_walls_changed(const H* __restrict__ src, const int* __restrict__ id, int n, int dim,
                                const V4<T>* __restrict__ wpos, int* __restrict__ flag)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const H* v = src + (size_t)id[s] * dim;
    const V4<T> o = wpos[s];
    bool ch = (T)v[0] != o.x || (T)v[1] != o.y;
    if (dim == 3) ch = ch || (T)v[2] != o.z;
    if (ch) atomicOr(flag, 1);
}
__global__ void k_iota(int* __restrict__ a, int n, int base)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) a[s] = base + s;
}

}  // namespace sb
