/*
 * sisph.h — C ABI of the B200-native SISPH hot path (libsisph.so).
 *
 * SISPH is the iterative, matrix-free incompressible SPH scheme of Muta,
 * Ramachandran & Negi (arXiv 1908.01762).  Citations "P:a-b" are lines of the
 * paper's LaTeX source; "Rn" are the readings listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Every pointer argument is a HOST pointer owned by the caller; the library
 *     copies in or out and never keeps it (exception: the pipelined
 *     sisph_stage_field / sisph_fetch_field read / write the caller's buffer
 *     asynchronously until sisph_commit_staged / sisph_fetch_wait returns).
 *     The handle owns all device memory,
 *     its CUDA stream (unless one is supplied in sisph_params.stream), and its
 *     NCCL communicator (distributed handles).
 *   - Vectors are row-major n x dim (dim = domain->dim) doubles.
 *   - Values passed in or returned are in CREATION-ID order: particle k is the
 *     k-th particle given to sisph_create.  Internally particles are kept in
 *     cell-sorted order (fluid and wall sets separately).
 *   - Calls are stream-ordered on the handle's stream; calls that return host
 *     values (solve, step, getters) synchronise the stream.
 *   - One handle per GPU; a handle is not thread-safe.
 *   - Return value: SISPH_OK (0) or one of the error codes below; the message
 *     of the last error is returned by sisph_last_error().  After
 *     SISPH_ENONFINITE or SISPH_ECUDA the state of the handle is undefined.
 */
#ifndef SISPH_H
#define SISPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SISPH_OK 0
#define SISPH_EINVAL 1      /* invalid argument (see each call) */
#define SISPH_ENOMEM 2      /* device or host allocation failed */
#define SISPH_ECUDA 3       /* a CUDA runtime call or kernel failed */
#define SISPH_ENCCL 4       /* an NCCL call failed (distributed handles) */
#define SISPH_ENONFINITE 5  /* a non-finite pressure appeared in the PPE sweep */
#define SISPH_EOVERFLOW 6   /* a particle has more neighbours than the list capacity */

#define SISPH_TAG_FLUID 0
#define SISPH_TAG_WALL 1
/* open boundaries along x (sisph_params.open_x, reading R34): */
#define SISPH_TAG_INLET 2    /* prescribed velocity (its creation velocity), PPE unknown */
#define SISPH_TAG_OUTLET 3   /* u and p frozen, advected with the extrapolated fluid u_x */
#define SISPH_TAG_DORMANT 4  /* not in the flow: the id pool new inlet particles come from */

typedef struct sisph sisph_t;

/* Simulation box.  Axes a < dim are used.  A periodic axis wraps positions
 * into [lo, hi) and uses the minimum image (R26); a bounded axis clamps cell
 * coordinates into the grid (R27). */
typedef struct {
    int dim;            /* 2 or 3 */
    double lo[3];
    double hi[3];
    int periodic[3];    /* 0 or 1 per axis */
} sisph_domain;

/* Scheme parameters.  sisph_params_default() fills the paper's defaults. */
typedef struct {
    int precision;          /* 32: fp32 state and arithmetic; 64: fp64 (default 64) */
    double rho0;            /* rest density rho0 */
    double nu;              /* kinematic viscosity (eq:mom:sph:visc) */
    double g[3];            /* body force per unit mass */
    double alpha;           /* artificial viscosity coefficient (eq:mom:sph:av, R20) */
    double c_ref;           /* reference sound speed c */
    double omega;           /* SOR factor, default 0.5 (eq:p-sor) */
    double eta;             /* regulariser eta h^2 with eta = 0.01 (R6) */
    double fs_ratio;        /* free surface if rho/rho0 < fs_ratio, default 0.8 */
    double h_tilde_factor;  /* GTVF kernel length h~ = factor h */
    double p_ref;           /* GTVF reference background pressure */
    int pgrad;              /* 0 symm (eq:mom:sph:press:symm), 1 asymm (eq:...:pij) */
    int pref_external;      /* 1: p0 = min(10|p|, p_ref); 0: p0 = p_ref */
    int ustar_noslip;       /* 1 no-slip, 0 slip wall u* (R16) */
    int clamp_wall_p;       /* 1: negative wall pressure -> 0 */
    int K;                  /* GTVF sub-steps (R22), default 10 */
    int min_iter;           /* minimum PPE sweeps, default 2 */
    int max_iter;           /* maximum PPE sweeps, default 1000 */
    double tol;             /* epsilon of eq:convergence used by sisph_step, default 1e-2 */
    int wall_rho_summation; /* 1: walls get summation density; 0: walls keep rho0 (R4) */
    int nbr_cap;            /* neighbour-list capacity per particle, 0 = automatic */
    int device;             /* CUDA device ordinal, -1 = current device */
    void* stream;           /* cudaStream_t to run on, NULL = the handle creates one */
    int rebuild_mode;       /* 0 (default): one build per step at r^n with a skin of
                               2 dt max|u~| and the r* sets filtered out of it (R3) when the
                               skin fits the grid; 1: two exact builds (at r^n and r*) */
    int matrix_free;        /* 0 (default): A11 stores the per-pair factor of fac_ij (eq:coeff)
                               once per solve and every sweep streams it (particles do not move
                               during the iterations); 1: every sweep recomputes it from
                               the positions, as the paper's listing */
    int ppe_loop;           /* form of the PPE loop (one handle, timing off; slab ranks and timing
                               always use 1): 0 (default) = auto: 4 for <= 16384 fluid particles,
                               3 for <= 400000 (2 with ppe_mean_free), 1 above; 1 = host-polled
                               speculative batches of
                               sweep launches; 2 = a captured CUDA graph with a device-decided WHILE
                               node; 3 = one persistent cooperative kernel for the whole loop (two
                               grid syncs per sweep, every block takes the stop decision); 4 = one thread-block cluster (<= 16 SMs) for
                               the whole loop, hardware cluster barriers between phases.  Every form
                               runs the same row arithmetic (equal sweep counts and pressures; forms
                               3 and 4 reduce the residual and the R32 mean in another order) */
    int ppe_mean_free;      /* reading R32: 1 = after every Jacobi sweep subtract the
                               mean of the live rows (fluid, not free surface, D_ii != 0) from
                               p^{k+1} before eq:convergence -- the projection onto the range of
                               a PPE with no Dirichlet row (fully periodic / enclosed flows, whose
                               operator has the constant null space: eq:coeff rows sum to zero).
                               0 (default) = eq:p-sor as printed.  Not with ppe_loop = 3. */
    int conv_mean;          /* reading R12b: 1 (default) = eq:convergence compares means over the
                               fluid, mean|p^{k+1} - p^k| / max(Lambda, mean|p^{k+1}|) (the text calls
                               the denominator "the mean pressure" and Lambda "a measure of the mean
                               pressure"; with means the paper's Table 1 sweep counts are
                               reproduced); 0 = the sums as printed */
    int open_x;             /* reading R34: 1 = open boundaries along x (single GPU,
                               bounded x).  After every step, in id order: outlet particles with
                               x >= x_end become dormant; fluid with x >= x_outlet become outlet
                               (u, p frozen); inlet with x >= x_inlet become fluid, and the lowest
                               dormant id becomes a new inlet particle at x - inlet_length with
                               the same velocity.  TAG reads the current types; fields of dormant
                               particles read 0.  SISPH_ENOMEM when the dormant pool runs out. */
    double x_inlet, x_outlet, x_end, inlet_length;
    int pref_auto;          /* reading R33: 1 = the GTVF background pressure p_ref is set to
                               2 max_i p_i over fluid from the handle's first solve (internal
                               flows), then kept; 0 (default) = p_ref as given */
} sisph_params;

/* Per-step report (sisph_step).  Timings are device milliseconds measured
 * with CUDA events on the handle's stream when timing is enabled. */
typedef struct {
    double dt;
    int iters;              /* PPE sweeps executed */
    double residual;        /* final value of eq:convergence's left side */
    double lambda;          /* Lambda = max |RHS_i / D_ii| (eq:convergence, R12) */
    double ms_predict, ms_solve, ms_correct;
    int64_t pairs;          /* directed neighbour pairs with a fluid destination, r* build */
    int max_neighbors;      /* largest neighbour count of the r* build */
    double ms_sweeps;       /* device ms of the Jacobi sweep kernels that did work (timing mode) */
    int sweeps_timed;       /* number of sweep launches ms_sweeps covers */
    int64_t launches;       /* kernel launches this step issued (speculative no-op sweeps included) */
    int single_build;       /* 1 if this step used the single build + filter (R3) */
    double skin_radius;     /* loose radius 3h + skin of that build (0 otherwise) */
    int64_t n_owned_fluid;  /* fluid particles this handle owns (all of them on one GPU) */
    int64_t n_ghost_fluid;  /* halo copies of neighbour slabs' fluid (slab ranks) */
    int64_t halo_bytes;     /* bytes this rank sent in halo / migration exchanges this step */
    /* timing mode, device ms of the pipeline phases: */
    double ms_build;        /* step start -> end of the build at r^n (skin, A1-A5: hash, sort,
                               reorder, list build) */
    double ms_filter;       /* A9: the r* sets (filter of the single build, or the second build) */
    double ms_rhs;          /* A11: wall p^0, RHS_i, D_ii, Lambda (+ the fused first sweep) */
    double ms_ppe;          /* M1's t_PPE: A11 start -> final decision of the solve */
} sisph_step_report;

typedef enum {
    SISPH_FIELD_POSITION = 0,           /* n x dim; r^n (after a step: r^{n+1}) */
    SISPH_FIELD_VELOCITY = 1,           /* n x dim; fluid u, wall ghost velocity u_w */
    SISPH_FIELD_TRANSPORT_VELOCITY = 2, /* n x dim; fluid u~ (walls: 0) */
    SISPH_FIELD_PRESSURE = 3,           /* n; fluid p, wall p_w */
    SISPH_FIELD_DENSITY = 4,            /* n; rho of the last density pass */
    SISPH_FIELD_MASS = 5,               /* n */
    SISPH_FIELD_USTAR = 6,              /* n x dim; u* (walls: wall u*) */
    SISPH_FIELD_RSTAR = 7,              /* n x dim; r* of the last predict (walls: r) */
    SISPH_FIELD_RHS = 8,                /* n; RHS_i of eq:sph-ppe (walls: 0) */
    SISPH_FIELD_DIAG = 9,               /* n; D_ii of eq:coeff (walls: 0) */
    SISPH_FIELD_NORMAL = 10,            /* n x dim; wall unit normals (fluid: 0) */
    SISPH_FIELD_FREE_SURFACE = 11,      /* n; 1 if free-surface fluid particle */
    SISPH_FIELD_TAG = 12,               /* n; 0 fluid, 1 wall (read only) */
    SISPH_FIELD_WALL_VELOCITY = 13      /* n x dim; the prescribed (physical) velocity u_i of a wall
                                           in eq:vg-adami, initially the creation
                                           velocity of the wall particle (fluid: 0; set ignores
                                           fluid entries).  Walls never move (R24): a sliding
                                           wall (a lid) moves along itself */
} sisph_field;

/* Fill *p with the paper's defaults (precision 64, omega 0.5, eta 0.01,
 * fs_ratio 0.8, K 10, min_iter 2, max_iter 1000, tol 1e-2, h~ = h, slip u*,
 * walls keep rho0; everything else 0). */
void sisph_params_default(sisph_params* p);

/* Create a simulation on one GPU.
 *   positions, velocities: n x dim; masses, densities: n; tags: n (0 fluid,
 *   1 wall); h: uniform smoothing length, support 3h.
 * Copies the inputs to the device, computes the cell grid (R26/R27), sorts
 * walls once, builds the neighbour lists, computes the wall normals
 * (§3.4.1) and sets u~ = u (R23), p = 0.
 * Errors: SISPH_EINVAL if n <= 0, h <= 0, dim not 2 or 3, a non-finite input,
 * a tag not 0/1, no fluid particle, a particle outside a bounded axis' box by
 * more than the box size, a periodic axis with fewer than 3 cells (L < 9h),
 * rho <= 0 or m <= 0, precision not 32/64; SISPH_ENOMEM; SISPH_ECUDA. */
int sisph_create(const double* positions, const double* velocities, const double* masses,
                 const double* densities, const int32_t* tags, int64_t n, double h,
                 const sisph_domain* domain, const sisph_params* params, sisph_t** out);

/* Release the handle and all its device memory.  NULL is ignored. */
void sisph_destroy(sisph_t* s);

/* Neighbour build at the current positions (A1-A5): cell hash, counting
 * (radix = cell key) sort with a stable per-cell fix-up, reorder of the fluid
 * state, cell start table, neighbour lists N(i) = { j != i : r_ij^2 < (3h)^2 }
 * (R2, decided in fp64).  Errors: SISPH_ECUDA, SISPH_EOVERFLOW. */
int sisph_build_neighbors(sisph_t* s);

/* Algorithm 1 lines 2-6 plus the PPE set-up: build at r^n,
 * summation density + free-surface flags (A6), wall ghost velocity (A7),
 * forces and predictors u*, r* (A8), neighbour sets at r* (A9: a second exact
 * build, or — default, R3 — the exact r* sets filtered out of a loose list
 * built once at r^n with radius 3h + 2 dt max|u~|), wall u* (A10),
 * RHS_i, D_ii and Lambda (A11).  Errors: SISPH_EINVAL if dt <= 0. */
int sisph_predict(sisph_t* s, double dt);

/* The PPE solve (Algorithm 1 lines 7-10; eq:p-sor, eq:convergence): damped
 * Jacobi from p^0 = current p, walls refreshed from p^k every sweep (R14),
 * until (k >= min(min_iter, max_iter) and residual < tol) or k == max_iter.
 * Needs a preceding sisph_predict.  Non-convergence is NOT an error: it
 * returns SISPH_OK with *iters_out == max_iter and *residual_out >= tol.
 * iters_out / residual_out may be NULL.  Errors: SISPH_EINVAL if tol < 0 or
 * max_iter < 1 or no predict was done; SISPH_ENONFINITE. */
int sisph_ppe_solve(sisph_t* s, double tol, int max_iter, int* iters_out, double* residual_out);

/* Algorithm 1 lines 11-19: final wall pressure, pressure gradient and
 * corrector u^{n+1} (eq:int:vnp1), K GTVF sub-steps with the pair set frozen
 * at r* (eq:int:gtvf:pos/vel:tmp), transport velocity (eq:int:vhatnp2) and
 * positions (eq:int:rnp2).  Errors: SISPH_EINVAL if dt <= 0 or no solve. */
int sisph_correct(sisph_t* s, double dt);

/* One full SISPH step = predict + ppe_solve(params.tol, params.max_iter) +
 * correct.  rep may be NULL. */
int sisph_step(sisph_t* s, double dt, sisph_step_report* rep);

/* Adaptive time step for the next step, from the step that last
 * completed (sisph_step or sisph_correct):
 *   dt_cfl   = 0.25 h / max_i |u_i|      (fluid velocities after that step)
 *   dt_force = 0.25 sqrt(h / max_i |f_i|), f = f_p + f_visc + f_body + f_avisc + f_astress
 *              of that step (the GTVF shift is not a force on u, eq:int:vnp1)
 *   dt_next  = min(dt_cfl, dt_force)
 * +INFINITY for an unrestricted criterion (zero maximum).  The maxima are
 * reduced on the device inside the step (no extra pass); slab ranks allreduce
 * them (collective call).  Output pointers may be NULL.  Errors: SISPH_EINVAL
 * before the first completed step. */
int sisph_next_dt(sisph_t* s, double* dt_next, double* dt_cfl, double* dt_force);

/* Copy a field out / in, creation-id order.  count must equal n (scalars) or
 * n * dim (vectors), else SISPH_EINVAL.  TAG is read only. */
int sisph_get_field(sisph_t* s, sisph_field f, double* out, int64_t count);
int sisph_set_field(sisph_t* s, sisph_field f, const double* in, int64_t count);

/* The same with fp32 host buffers (half the host<->device bytes: the I/O of an
 * fp32 handle's state at its own precision).  An fp64 handle widens on set and
 * rounds on get.  Buffers may be pageable or pinned host memory, or device
 * memory (cudaMemcpyDefault); the call is stream-ordered and returns after the
 * copy (get) / the device-side scatter is enqueued (set).  Errors as above. */
int sisph_get_field_f32(sisph_t* s, sisph_field f, float* out, int64_t count);
int sisph_set_field_f32(sisph_t* s, sisph_field f, const float* in, int64_t count);

/* Pipelined input (the state a caller feeds for the NEXT step, uploaded while
 * the current one computes): sisph_stage_field / _f32 enqueue the host->device
 * copy of `in` (same fields, counts and layout as sisph_set_field) on the
 * handle's upload stream and return at once; the handle's state is unchanged
 * until sisph_commit_staged, which makes the handle's stream wait for the
 * staged copies and scatters them in staging order (stream-ordered, like
 * sisph_set_field; staging POSITION checks the wall geometry as set_field
 * does).  A field can be staged once per commit.  Ownership: `in` must stay
 * valid and unmodified until sisph_commit_staged returns; pinned host memory
 * makes the copy overlap the handle's kernels (pageable memory is copied
 * synchronously by the driver).  The next staging of a field waits on the
 * device for the previous commit's scatters.  Errors: SISPH_EINVAL (field,
 * count, NULL, or a field staged twice), SISPH_ECUDA. */
int sisph_stage_field(sisph_t* s, sisph_field f, const double* in, int64_t count);
int sisph_stage_field_f32(sisph_t* s, sisph_field f, const float* in, int64_t count);
int sisph_commit_staged(sisph_t* s);

/* Pipelined output: sisph_fetch_field / _f32 enqueue, on the handle's stream,
 * the gather of field f into creation-id order (as sisph_get_field) and its
 * device->host copy on a download stream, and return at once; the handle's
 * stream goes on (e.g. with the next step) while the copy runs.
 * sisph_fetch_wait blocks until the copy is in `out` (returns at once if no
 * fetch is pending).  One fetch at a time: a second fetch before the wait is
 * SISPH_EINVAL.  Ownership: `out` (pinned host memory for an overlapped copy)
 * must stay valid until sisph_fetch_wait returns.  The value is the field as
 * of the point in the handle's stream where the fetch was enqueued.  Errors:
 * SISPH_EINVAL (field, TAG, count, NULL, pending fetch), SISPH_ECUDA. */
int sisph_fetch_field(sisph_t* s, sisph_field f, double* out, int64_t count);
int sisph_fetch_field_f32(sisph_t* s, sisph_field f, float* out, int64_t count);
int sisph_fetch_wait(sisph_t* s);

/* Creation ids in internal order: ids[0 .. n_fluid) are the fluid particles
 * in cell-sorted order, ids[n_fluid .. n) the walls.  n must equal the
 * particle count. */
int sisph_get_order(sisph_t* s, int64_t* ids, int64_t n);

/* The current neighbour sets as CSR in creation-id order, each row sorted by
 * id: offsets[n + 1], ids[*total].  If cap < total only offsets and *total
 * are written and SISPH_EINVAL is returned. */
int sisph_get_neighbors(sisph_t* s, int64_t* offsets, int64_t* ids, int64_t cap, int64_t* total);

/* The neighbour sets of the m particles with creation ids which[0 .. m) only
 * (for large problems): CSR offsets[m + 1], ids[*total], rows in the order of
 * which, each sorted by id.  Errors as sisph_get_neighbors; an id outside
 * [0, n) is SISPH_EINVAL. */
int sisph_get_neighbors_of(sisph_t* s, const int64_t* which, int64_t m, int64_t* offsets, int64_t* ids,
                           int64_t cap, int64_t* total);

/* ---------------------------------------------------------------------------
 * Slab decomposition over several GPUs.  The domain is cut
 * into nranks slabs of equal width along slab_axis; rank r owns the particles
 * whose slab_axis coordinate lies in its slab (sisph_slab_bounds) and keeps
 * read-only halo copies of the neighbour slabs' particles within 1.3 x 3h of
 * its faces.  Per step: fluid particles that left the slab migrate to the
 * neighbour rank; halos are refreshed before every pass that reads them (the
 * PPE sweep: wall pressure and p^{k+1} every sweep); Lambda, the two sums of
 * eq:convergence and the skin are allreduced, so every rank runs the same
 * number of sweeps.  One process (or, for tests, one thread) per rank; every
 * rank calls every entry point collectively, in the same order.
 * ------------------------------------------------------------------------- */
typedef struct sisph_local_group sisph_local_group_t;

typedef struct {
    int nranks;              /* >= 1 (1: same as sisph_create) */
    int rank;                /* 0 .. nranks - 1 */
    int slab_axis;           /* 0 .. dim - 1; slabs must be at least 1.3 x 3h wide */
    uint8_t nccl_id[128];    /* NCCL unique id from sisph_nccl_unique_id on one rank,
                                broadcast to all ranks by the caller (e.g. torch.distributed) */
    const char* nccl_lib;    /* NCCL library to dlopen (NULL: "libnccl.so.2") */
    sisph_local_group_t* local_group;  /* non-NULL: ranks are threads of THIS process sharing
                                          one GPU, exchanging through device copies at host
                                          barriers (tests; no NCCL) */
    int always_slab;         /* 1: the slab path even for nranks == 1 (a periodic slab axis then
                                takes its halo from the rank itself, through the transport) */
} sisph_dist;

/* A fresh NCCL unique id (ncclGetUniqueId of the library nccl_lib, NULL for
 * "libnccl.so.2").  Errors: SISPH_EINVAL (NULL id), SISPH_ENCCL. */
int sisph_nccl_unique_id(const char* nccl_lib, uint8_t id[128]);

/* An in-process group of nranks ranks (see sisph_dist.local_group).  Destroy
 * after every handle of the group. */
int sisph_local_group_create(int nranks, sisph_local_group_t** out);
void sisph_local_group_destroy(sisph_local_group_t* group);

/* [lo, hi) of rank's slab: lo + L r / nranks .. lo + L (r + 1) / nranks along axis. */
int sisph_slab_bounds(const sisph_domain* domain, int axis, int nranks, int rank, double* lo, double* hi);

/* The rank owning slab-axis coordinate y: the slab whose [lo, hi) holds it;
 * below / above a bounded box: the first / last slab.  -1 on bad arguments. */
int sisph_slab_owner(const sisph_domain* domain, int axis, int nranks, double y);

/* Collective create of one rank of a slab-decomposed simulation.  Every rank
 * passes the same GLOBAL arrays (as sisph_create) and keeps its slab and
 * halos.  Field getters of a rank fill the entries of the particles it owns
 * (others are left 0: summing the ranks' arrays gives the whole field);
 * setters take those entries.  The wall geometry is fixed at create.
 * Errors: as sisph_create; SISPH_EINVAL for bad rank / axis or slabs thinner
 * than the halo; SISPH_ENCCL; a step whose skin 2 dt max|u~| exceeds 0.3 x 3h
 * returns SISPH_EINVAL (reduce dt). */
int sisph_create_dist(const double* positions, const double* velocities, const double* masses,
                      const double* densities, const int32_t* tags, int64_t n, double h,
                      const sisph_domain* domain, const sisph_params* params, const sisph_dist* dist,
                      sisph_t** out);

/* Particles owned by this handle (= sisph_get_counts' fluid / wall counts on one GPU). */
int sisph_get_owned_counts(sisph_t* s, int64_t* n_fluid, int64_t* n_wall);

/* Counts: particles, fluid particles, wall particles. */
int sisph_get_counts(const sisph_t* s, int64_t* n, int64_t* n_fluid, int64_t* n_wall);

/* Enable (1) / disable (0) per-phase CUDA-event timing in sisph_step. */
int sisph_set_timing(sisph_t* s, int enable);

/* Device milliseconds of the sweep-kernel launches of the last solve that
 * were bracketed by CUDA events (timing enabled; the first sweep is fused into
 * A11 and not counted), and their number.  Outputs may be NULL. */
int sisph_sweep_timing(sisph_t* s, double* ms, int* n);

/* Wait for all work queued on the handle's stream. */
int sisph_sync(sisph_t* s);

/* Message of the last error of s (or of the calling thread if s is NULL). */
const char* sisph_last_error(const sisph_t* s);

#ifdef __cplusplus
}
#endif
#endif /* SISPH_H */
