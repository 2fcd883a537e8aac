// sisph_device.cuh — device-side types and per-pair arithmetic of the SISPH
// hot path (sm_100a).  Citations "P:a-b" are PAPER.md lines; "Rn" DESIGN.md
// readings.  Nothing here is shared with the oracle (oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sb {

// ---------------------------------------------------------------------------
// Vector types.  Particle positions are packed (x, y, z, m) so one 16-byte
// (fp32) or 32-byte (fp64) load brings everything a neighbour gather needs
// besides rho_j and p_j.
// ---------------------------------------------------------------------------
struct __align__(32) dbl4 {
    double x, y, z, w;
};

template <class T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = dbl4; };
template <class T> using V4 = typename V4T<T>::type;

__device__ __forceinline__ float4 ld4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ dbl4 ld4(const dbl4* p)
{
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return dbl4{a.x, a.y, b.x, b.y};
}
template <class T> __device__ __forceinline__ V4<T> mk4(T x, T y, T z, T w);
template <> __device__ __forceinline__ float4 mk4<float>(float x, float y, float z, float w)
{
    return make_float4(x, y, z, w);
}
template <> __device__ __forceinline__ dbl4 mk4<double>(double x, double y, double z, double w)
{
    return dbl4{x, y, z, w};
}

// 8-element records with one 256-bit access (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256);
// fp64 records are two 256-bit halves.  Read-only (.nc) loads: callers never read a
// record array the same kernel writes.
__device__ __forceinline__ void ld8(const float* p, float (&r)[8])
{
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
        : "l"(p));
}
__device__ __forceinline__ void ld8(const double* p, double (&r)[8])
{
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[4]), "=d"(r[5]), "=d"(r[6]), "=d"(r[7]) : "l"(p + 4));
}
__device__ __forceinline__ void st8(float* p, const float (&r)[8])
{
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
                 "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}
__device__ __forceinline__ void st8(double* p, const double (&r)[8])
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3])
                 : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4), "d"(r[4]), "d"(r[5]), "d"(r[6]), "d"(r[7])
                 : "memory");
}

// ---------------------------------------------------------------------------
// Kernel-argument block: geometry + scheme constants, passed by value.
// ---------------------------------------------------------------------------
template <class T> struct Params {
    // sizes: fluid slots [0, Nf) = owned [0, Nfo) + ghosts [Nfo, Nf); wall slots
    // [Nf, Ntot) = owned [Nf, Nf + Nwo) + ghosts.  Single GPU: Nfo = Nf, Nwo = Nw.
    int Nf, Nw, Ntot, cap;
    int Nfo, Nwo;
    int ghosts;            // 1: keys of ghost particles are offset by the cell count (slab halos)
    // cell grid (R26/R27): decisions in fp64
    int dim;
    int nc[3];
    int per[3];
    double lo[3], hi[3], cell[3], Ld[3], halfLd[3];
    double R2d;            // (3h)^2 in fp64 (R2)
    float R2lo, R2hi;      // fp32 prefilter band around R^2
    float Lf[3], halfLf[3];
    // working-precision constants
    T L[3], halfL[3];
    T h, sig, dwk;         // W = sig * poly5(q), dW/dr = dwk * poly4(q), q = r / h
    T inv_h;
    T h2, sig2, dwk2, inv_h2;   // kernel at h/2 (Shepard of eq:vf)
    T ht, dwkt, inv_ht;         // kernel at h~ (GTVF, eq:mom:sph:gtvf)
    T w0;                  // W(0)
    T eta_h2;              // eta h^2 (R6)
    T rho0, nu, alpha, c_ref, omega, fs_ratio, p_ref;
    T g[3];
    int pgrad, pref_external, ustar_noslip, clamp_wall_p, wall_rho_summation;
    int mean_free;          // R32: remove the live-row mean of every Jacobi iterate
    // R34 open boundaries along x: particle type of each fluid-block slot
    // (0 fluid, 2 inlet, 3 outlet; nullptr without open boundaries)
    const uint8_t* ptype;
    T x_inlet, x_outlet, x_end, inlet_length;
    // GTVF inner list (pairs with r* < 3 h~ + skin; used when h~ < h)
    int cap_in;
    float Rin2f;           // (3 h~ + skin)^2 (1 + 2^-10): generous inclusion
    T skin_half2;          // (skin / 2)^2: allowed squared displacement per particle
    // loose (superset) radius^2 of the single per-step build at r^n (R3):
    // (3h + 2 dt max|u~| + margin)^2 (1 + 2^-10), working precision
    T Rs2;
    // (3h)^2 (1 + 2^-10): a pair at or beyond it contributes exactly 0 to every
    // kernel sum (W, dW/dr vanish for q >= 3): passes over the loose list skip it
    T R2cut;
    // fixed-point coordinates of the fp32 GTVF sub-steps: x_fix = (x - lo) / fxs (mod 2^32),
    // fxs = L / 2^32 per axis (7.5e-10 m on C5's 3.2 m tank: 2e-7 h); a pair difference is an
    // exact int32 subtraction (the minimum image on a periodic axis for free)
    double fxs[3];
    float fxf[3];
};

// ---------------------------------------------------------------------------
// M6 quintic spline (reading R1), branch-free: each truncated power is
// max(k - q, 0)^n, identical to the piecewise definition.
// ---------------------------------------------------------------------------
template <class T> __device__ __forceinline__ T quintic4(T q)
{
    T a = fmax(T(3) - q, T(0)), b = fmax(T(2) - q, T(0)), c = fmax(T(1) - q, T(0));
    T a2 = a * a, b2 = b * b, c2 = c * c;
    return a2 * a2 - T(6) * (b2 * b2) + T(15) * (c2 * c2);
}
template <class T> __device__ __forceinline__ T quintic5(T q)
{
    T a = fmax(T(3) - q, T(0)), b = fmax(T(2) - q, T(0)), c = fmax(T(1) - q, T(0));
    T a2 = a * a, b2 = b * b, c2 = c * c;
    return a2 * a2 * a - T(6) * (b2 * b2 * b) + T(15) * (c2 * c2 * c);
}

__device__ __forceinline__ float my_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double my_sqrt(double x) { return sqrt(x); }

// minimum-image difference on a periodic axis (R26)
template <class T> __device__ __forceinline__ T wrapd(T d, T L, T halfL)
{
    if (d > halfL) d -= L;
    else if (d < -halfL) d += L;
    return d;
}

// r_ij = r_i - r_j in working precision (minimum image), returns r^2
template <class T, int D>
__device__ __forceinline__ T pair_vec(const Params<T>& P, const V4<T>& a, const V4<T>& b, T d[3])
{
    d[0] = a.x - b.x;
    d[1] = a.y - b.y;
    d[2] = D == 3 ? a.z - b.z : T(0);
    if (P.per[0]) d[0] = wrapd(d[0], P.L[0], P.halfL[0]);
    if (P.per[1]) d[1] = wrapd(d[1], P.L[1], P.halfL[1]);
    if (D == 3 && P.per[2]) d[2] = wrapd(d[2], P.L[2], P.halfL[2]);
    T r2 = d[0] * d[0] + d[1] * d[1];
    if (D == 3) r2 += d[2] * d[2];
    return r2;
}

// ---------------------------------------------------------------------------
// Exact neighbour decision (R2): r^2 < R^2 evaluated in fp64 exactly as the
// definition is written (difference, minimum image, products and sums in
// order, no contraction).  Working in fp32, a cheap prefilter decides all
// pairs whose fp32 r^2 is outside a band [R2lo, R2hi] around R^2 that bounds
// the fp32 rounding (a few 2^-24 relative plus the periodic shift terms, set in
// the engine); only the band goes to fp64 (it is also the whole decision in
// fp64 mode).
// ---------------------------------------------------------------------------
// the rare fp32 band case, out of line so the candidate loop stays small;
// scalars by value (a reference to the kernel-parameter block would force
// a local copy of it)
__device__ __forceinline__ double wrap_exact(double d, double L)
{
    double hl = 0.5 * L;
    return d > hl ? __dadd_rn(d, -L) : (d < -hl ? __dadd_rn(d, L) : d);
}
__device__ __forceinline__ bool exact_band(double xi, double yi, double zi, double xj, double yj, double zj, double L0,
                                        double L1, double L2, int pmask, int three, double R2)
{
    double d0 = __dadd_rn(xi, -xj), d1 = __dadd_rn(yi, -yj), d2 = three ? __dadd_rn(zi, -zj) : 0.0;
    if (pmask & 1) d0 = wrap_exact(d0, L0);
    if (pmask & 2) d1 = wrap_exact(d1, L1);
    if (three && (pmask & 4)) d2 = wrap_exact(d2, L2);
    double r2 = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
    if (three) r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
    return r2 < R2;
}

template <int D>
__device__ __forceinline__ bool exact_inside(const Params<double>& P, double xi, double yi, double zi,
                                             double xj, double yj, double zj)
{
    double d0 = __dadd_rn(xi, -xj), d1 = __dadd_rn(yi, -yj), d2 = D == 3 ? __dadd_rn(zi, -zj) : 0.0;
    if (P.per[0]) d0 = d0 > P.halfLd[0] ? __dadd_rn(d0, -P.Ld[0]) : (d0 < -P.halfLd[0] ? __dadd_rn(d0, P.Ld[0]) : d0);
    if (P.per[1]) d1 = d1 > P.halfLd[1] ? __dadd_rn(d1, -P.Ld[1]) : (d1 < -P.halfLd[1] ? __dadd_rn(d1, P.Ld[1]) : d1);
    if (D == 3 && P.per[2])
        d2 = d2 > P.halfLd[2] ? __dadd_rn(d2, -P.Ld[2]) : (d2 < -P.halfLd[2] ? __dadd_rn(d2, P.Ld[2]) : d2);
    double r2 = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
    if (D == 3) r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
    return r2 < P.R2d;
}

// cell coordinates of a position, fp64 with IEEE division (R27): identical
// to floor((x - lo) / cell) then clamp
template <class T>
__device__ __forceinline__ int cell_coord(const Params<T>& P, int a, double x)
{
    double f = floor(__ddiv_rn(__dadd_rn(x, -P.lo[a]), P.cell[a]));
    if (f < 0.0) return 0;
    if (f > (double)(P.nc[a] - 1)) return P.nc[a] - 1;
    return (int)f;
}

template <class T, int D>
__device__ __forceinline__ void cell_of(const Params<T>& P, const V4<T>& x, int c[3])
{
    c[0] = cell_coord(P, 0, (double)x.x);
    c[1] = cell_coord(P, 1, (double)x.y);
    c[2] = D == 3 ? cell_coord(P, 2, (double)x.z) : 0;
}

template <class T>
__device__ __forceinline__ int cell_key(const Params<T>& P, const int c[3])
{
    return c[0] + P.nc[0] * (c[1] + P.nc[1] * c[2]);
}

// ---------------------------------------------------------------------------
// warp / block reductions
// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL): a kernel launched with the programmatic
// stream-serialization attribute may be scheduled while its predecessor runs;
// pdl_wait blocks until the predecessor has completed and its writes are
// visible (a no-op without the attribute), pdl_trigger lets the successor be
// scheduled early.  Every PDL-launched kernel waits before it reads anything.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// Per-pair arithmetic.  fp32: hardware approximations (MUFU rsqrt / rcp,
// relative error ~2^-22), which is well inside the fp32 parity tolerance;
// fp64: correctly rounded operations (parity 1e-10 against the oracle).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float frsqrt(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double frsqrt(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ float frcp(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double frcp(double x) { return 1.0 / x; }

// r and 1/r from r^2 (> 0 for every listed pair; clamped for coincident particles)
__device__ __forceinline__ void r_of(float r2, float& r, float& ri)
{
    float x = fmaxf(r2, 1e-30f);
    ri = frsqrt(x);
    r = x * ri;
}
__device__ __forceinline__ void r_of(double r2, double& r, double& ri)
{
    r = sqrt(r2);
    ri = r > 0.0 ? 1.0 / r : 0.0;
}

// neighbour test that also returns an approximation of r^2 (for the inner list)
template <int D>
__device__ __forceinline__ bool nb_test(const Params<float>& P, const float4& a, const float4& b, float& r2o)
{
    float d0 = a.x - b.x, d1 = a.y - b.y, d2 = D == 3 ? a.z - b.z : 0.f;
    if (P.per[0]) d0 = wrapd(d0, P.Lf[0], P.halfLf[0]);
    if (P.per[1]) d1 = wrapd(d1, P.Lf[1], P.halfLf[1]);
    if (D == 3 && P.per[2]) d2 = wrapd(d2, P.Lf[2], P.halfLf[2]);
    float r2 = d0 * d0 + d1 * d1;
    if (D == 3) r2 += d2 * d2;
    r2o = r2;
    if (r2 < P.R2lo) return true;
    if (r2 > P.R2hi) return false;
    return exact_band((double)a.x, (double)a.y, (double)a.z, (double)b.x, (double)b.y, (double)b.z, P.Ld[0], P.Ld[1],
                      P.Ld[2], P.per[0] | (P.per[1] << 1) | (P.per[2] << 2), D == 3, P.R2d);
}
template <int D>
__device__ __forceinline__ bool nb_test(const Params<double>& P, const dbl4& a, const dbl4& b, float& r2o)
{
    double d0 = a.x - b.x, d1 = a.y - b.y, d2 = D == 3 ? a.z - b.z : 0.0;
    if (P.per[0]) d0 = wrapd(d0, P.Ld[0], P.halfLd[0]);
    if (P.per[1]) d1 = wrapd(d1, P.Ld[1], P.halfLd[1]);
    if (D == 3 && P.per[2]) d2 = wrapd(d2, P.Ld[2], P.halfLd[2]);
    double r2 = d0 * d0 + d1 * d1;
    if (D == 3) r2 += d2 * d2;
    r2o = (float)r2;
    if (r2 < P.R2d * (1.0 - 1e-9)) return true;
    if (r2 > P.R2d * (1.0 + 1e-9)) return false;
    return exact_inside<D>(P, a.x, a.y, a.z, b.x, b.y, b.z);
}

}  // namespace sb
