/*
 * sisph_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what SISPH (Muta, Ramachandran &
 * Negi, arXiv 1908.01762) computes, written from PAPER.md.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code, header, table or constant generator with
 * the CUDA path (paper_1908_01762_b200/csrc, include/sisph.h).
 *
 * Particles are kept in creation-id order throughout; every sum runs over a
 * neighbour list sorted by ascending id.  Citations "P:a-b" are PAPER.md
 * lines; readings "Rn" are the DESIGN.md / SURVEY.md §8(c) readings.
 */
#ifndef SISPH_ORACLE_H
#define SISPH_ORACLE_H
#include <stdint.h>

typedef struct {
    int dim;                 /* 2 or 3 */
    double lo[3], hi[3];
    int periodic[3];
    double h;                /* uniform smoothing length */
    /* scheme parameters */
    double rho0, nu, g[3], alpha, c_ref, omega, eta, fs_ratio;
    double h_tilde_factor, p_ref;
    int pgrad;               /* 0 symm (eq:mom:sph:press:symm), 1 asymm (eq:mom:sph:press:pij) */
    int pref_external;       /* 0 internal p0 = p_ref, 1 external p0 = min(10|p|, p_ref) */
    int ustar_noslip;        /* 0 slip, 1 no-slip wall u* (R16) */
    int clamp_wall_p;        /* p_w < 0 -> 0 */
    int K;                   /* GTVF sub-steps (R22) */
    int min_iter, max_iter;
    double tol;              /* epsilon of eq:convergence */
    int wall_rho_summation;  /* R4: 1 walls get summation density, 0 walls keep rho0 */
    int ppe_mean_free;       /* R32: 1 = remove the mean of the live rows (not free surface, D_ii != 0)
                                from every Jacobi iterate (null space of a PPE with no Dirichlet row) */
    int conv_mean;           /* R12b: 1 = eq:convergence on means over the fluid, mean|dp| / max(Lambda,
                                mean|p|) ("Lambda ... as a measure of the mean pressure");
                                0 = the sums as printed */
    /* NEXT-4b open boundaries along x (§3.5, reading R34): tags 2 inlet, 3 outlet,
     * 4 dormant (the id pool new inlet particles are drawn from).  After each step, in id
     * order: outlet with x >= x_end -> dormant; fluid with x >= x_outlet -> outlet (u, p
     * frozen); inlet with x >= x_inlet -> fluid, and the lowest dormant id becomes a new
     * inlet particle at x - inlet_length with the same velocity. */
    int open_x;
    double x_inlet, x_outlet, x_end, inlet_length;
    int pref_auto;           /* R33: 1 = internal-flow p_ref := 2 max_i p_i over fluid, taken once from
                                the pressure of the first solve, then constant */
} or_cfg;

typedef struct or_sim or_sim;

typedef struct {
    int iters;
    double residual;
    double lambda;
} or_report;

/* kernel (R1: M6 quintic spline, support 3h) */
double or_W(int dim, double r, double h);
double or_dWdr(int dim, double r, double h);

/* cell geometry + stable counting sort by cell key (A1-A4) */
int or_cell_geometry(const or_cfg* c, int* ncell, double* cell);
int64_t or_cell_key(const or_cfg* c, const double* x3);
void or_cell_order(const or_cfg* c, int64_t n, const double* x3, int64_t* order, int64_t* keys);

/* neighbour sets N(i) = { j != i : |r_ij|^2 < (3h)^2 } (R2), CSR sorted by id.
 * dests == NULL means all particles.  Returns the number of pairs, or -1 if
 * cap is too small (offsets are still filled). */
int64_t or_neighbors_cell(const or_cfg* c, int64_t n, const double* x3, int64_t nd,
                          const int64_t* dests, int64_t* off, int64_t* nbr, int64_t cap);
int64_t or_neighbors_brute(const or_cfg* c, int64_t n, const double* x3, int64_t nd,
                           const int64_t* dests, int64_t* off, int64_t* nbr, int64_t cap);

/* simulation state (id order) */
or_sim* or_create(const or_cfg* c, int64_t n, const double* x3, const double* u3,
                  const double* m, const double* rho, const double* p, const int32_t* tag);
void or_destroy(or_sim* s);
int or_get(or_sim* s, const char* field, double* out);
void or_get_tags(or_sim* s, int32_t* out);
int or_error(or_sim* s);   /* 1: the dormant pool ran out during an inlet spawn */
int or_set(or_sim* s, const char* field, const double* in);

/* Algorithm 1 split as the C ABI splits it */
void or_predict(or_sim* s, double dt);                       /* lines 2-5 + A10/A11 */
void or_predict_stage2(or_sim* s, double dt);                /* A9-A11 from the current xs, us */
void or_solve(or_sim* s, double tol, int max_iter, or_report* rep);  /* lines 6-9 */
void or_correct(or_sim* s, double dt);                       /* lines 10-19 */
void or_step(or_sim* s, double dt, or_report* rep);

/* single passes, for per-stage parity checks; they read the fields the
 * step would have produced (set with or_set) and write theirs */
void or_pass_density(or_sim* s);          /* at x  */
void or_pass_ghost_velocity(or_sim* s);   /* at x  */
void or_pass_wall_pressure(or_sim* s, const double* pk, double* pw_out);   /* at xs */
/* one Jacobi/SOR sweep for the listed fluid dests (all fluid if nd == 0),
 * from pressures pk (all particles, id order); wall entries of pk are used
 * as given.  Writes p^{k+1} for those dests into out[j] (j = position in the
 * dest list). */
void or_pass_sweep(or_sim* s, const double* pk, int64_t nd, const int64_t* dests, double* out);
int64_t or_num_pairs(or_sim* s, int which);  /* 0: build at x, 1: build at xs */

/* adaptive time step of the next step from the last completed
 * step: min(0.25 h / max|u|, 0.25 sqrt(h / max|f|)) over fluid, f = f_p +
 * f_visc + f_body + f_avisc + f_astress; +inf for an unrestricted criterion;
 * -1 if no step has completed */
int or_next_dt(or_sim* s, double* dt_next, double* dt_cfl, double* dt_force);

#endif
