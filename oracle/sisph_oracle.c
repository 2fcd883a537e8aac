/*
 * sisph_oracle.c — TEST INFRASTRUCTURE ONLY (see sisph_oracle.h).
 *
 * Plain fp64 CPU oracle of the SISPH per-step hot path, written from PAPER.md
 * (arXiv 1908.01762).  Compiled with -O2 -ffp-contract=off so that every
 * product and sum is rounded exactly as written.  OpenMP only splits the
 * outer loop over destination particles; each particle's sum runs serially
 * over its neighbour list in ascending id order, and every global reduction
 * runs serially in id order, so results do not depend on the thread count.
 *
 * No code here is shared with the CUDA path.
 */
#include "sisph_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define FLUID 0
#define WALL 1
#define INLET 2     /* open boundaries (R34): prescribed velocity, PPE unknowns */
#define OUTLET 3    /* u, p frozen, advected with the Shepard-extrapolated fluid u_x */
#define DORMANT 4   /* not in the flow: parked far outside the domain */
#define LIQ(t) ((t) == FLUID || (t) == INLET || (t) == OUTLET)
#define UNKNOWN(t) ((t) == FLUID || (t) == INLET)   /* PPE rows */

/* ------------------------------------------------------------------------ */
/* Kernel: reading R1 (the paper only says "quintic spline"). */
/* W(q) = sigma_d / h^d [(3-q)^5 - 6(2-q)^5 + 15(1-q)^5], terms only where    */
/* positive; sigma_2 = 7/(478 pi), sigma_3 = 1/(120 pi).                     */
/* ------------------------------------------------------------------------ */
static double sigma_d(int dim, double h)
{
    if (dim == 2) return 7.0 / (478.0 * M_PI * h * h);
    return 1.0 / (120.0 * M_PI * h * h * h);
}

double or_W(int dim, double r, double h)
{
    double q = r / h;
    double w = 0.0;
    if (q < 3.0) { double t = 3.0 - q; w += t * t * t * t * t; }
    if (q < 2.0) { double t = 2.0 - q; w -= 6.0 * t * t * t * t * t; }
    if (q < 1.0) { double t = 1.0 - q; w += 15.0 * t * t * t * t * t; }
    return sigma_d(dim, h) * w;
}

/* dW/dr = -5 sigma_d / h^(d+1) [(3-q)^4 - 6(2-q)^4 + 15(1-q)^4] */
double or_dWdr(int dim, double r, double h)
{
    double q = r / h;
    double w = 0.0;
    if (q < 3.0) { double t = 3.0 - q; w += t * t * t * t; }
    if (q < 2.0) { double t = 2.0 - q; w -= 6.0 * t * t * t * t; }
    if (q < 1.0) { double t = 1.0 - q; w += 15.0 * t * t * t * t; }
    return -5.0 * sigma_d(dim, h) / h * w;
}

/* grad_i W_ij = dW/dr * r_ij / |r_ij|, and 0 at r = 0 */
static void gradW(int dim, const double d[3], double r, double h, double gw[3])
{
    gw[0] = gw[1] = gw[2] = 0.0;
    if (r > 0.0) {
        double f = or_dWdr(dim, r, h) / r;
        for (int a = 0; a < dim; a++) gw[a] = f * d[a];
    }
}

/* ------------------------------------------------------------------------ */
/* Geometry: minimum image on periodic axes (R26); r^2 summed left to right   */
/* with no contraction (R2).                                                  */
/* ------------------------------------------------------------------------ */
static double rij(const or_cfg* c, const double* xi, const double* xj, double d[3])
{
    d[0] = d[1] = d[2] = 0.0;
    for (int a = 0; a < c->dim; a++) {
        double v = xi[a] - xj[a];
        if (c->periodic[a]) {
            double L = c->hi[a] - c->lo[a];
            if (v > 0.5 * L) v -= L;
            else if (v < -0.5 * L) v += L;
        }
        d[a] = v;
    }
    double r2 = d[0] * d[0] + d[1] * d[1];
    if (c->dim == 3) r2 = r2 + d[2] * d[2];
    return r2;
}

static double support_R(const or_cfg* c) { return 3.0 * c->h; }

static void wrap_pos(const or_cfg* c, double* x)
{
    for (int a = 0; a < c->dim; a++) {
        if (!c->periodic[a]) continue;
        double L = c->hi[a] - c->lo[a];
        if (x[a] >= c->hi[a]) x[a] -= L;
        else if (x[a] < c->lo[a]) x[a] += L;
    }
}

/* R26/R27: n_a = floor(L_a / R) (at least 1), cell_a = L_a / n_a >= R;
 * a periodic axis needs n_a >= 3.  Returns 0 on success, -1 otherwise. */
int or_cell_geometry(const or_cfg* c, int* ncell, double* cell)
{
    double R = support_R(c);
    for (int a = 0; a < 3; a++) { ncell[a] = 1; cell[a] = 1.0; }
    for (int a = 0; a < c->dim; a++) {
        double L = c->hi[a] - c->lo[a];
        int n = (int)floor(L / R);
        if (n < 1) n = 1;
        if (c->periodic[a] && n < 3) return -1;
        ncell[a] = n;
        cell[a] = L / n;
    }
    return 0;
}

static void cell_coords(const or_cfg* c, const int* nc, const double* cl, const double* x, int* cc)
{
    cc[0] = cc[1] = cc[2] = 0;
    for (int a = 0; a < c->dim; a++) {
        double f = floor((x[a] - c->lo[a]) / cl[a]);
        int v;
        if (f < 0.0) v = 0;
        else if (f > (double)(nc[a] - 1)) v = nc[a] - 1;
        else v = (int)f;
        cc[a] = v;
    }
}

int64_t or_cell_key(const or_cfg* c, const double* x3)
{
    int nc[3]; double cl[3]; int cc[3];
    or_cell_geometry(c, nc, cl);
    cell_coords(c, nc, cl, x3, cc);
    return (int64_t)cc[0] + (int64_t)nc[0] * ((int64_t)cc[1] + (int64_t)nc[1] * (int64_t)cc[2]);
}

/* Stable counting sort of the elements 0..n-1 (in their current order) by
 * cell key: order[r] = the element placed at rank r.  Textbook counting sort
 * (count, exclusive prefix sum, in-order placement), hence stable. */
void or_cell_order(const or_cfg* c, int64_t n, const double* x3, int64_t* order, int64_t* keys)
{
    int nc[3]; double cl[3];
    or_cell_geometry(c, nc, cl);
    int64_t ncells = (int64_t)nc[0] * nc[1] * nc[2];
    int64_t* cnt = (int64_t*)calloc((size_t)ncells + 1, sizeof(int64_t));
    int64_t* k = keys ? keys : (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
        int cc[3];
        cell_coords(c, nc, cl, x3 + 3 * i, cc);
        k[i] = (int64_t)cc[0] + (int64_t)nc[0] * ((int64_t)cc[1] + (int64_t)nc[1] * (int64_t)cc[2]);
        cnt[k[i] + 1]++;
    }
    for (int64_t b = 0; b < ncells; b++) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; i++) order[cnt[k[i]]++] = i;
    if (!keys) free(k);
    free(cnt);
}

/* ------------------------------------------------------------------------ */
/* Neighbour sets (R2): N(i) = { j != i : r_ij^2 < R^2 }, R = 3h, sorted by id */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t nd;        /* number of rows (= n: one row per particle) */
    int64_t* off;      /* n + 1 */
    int64_t* nbr;
    int built;
} csr_t;

static int cmp_i64(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

typedef struct {
    int nc[3];
    double cl[3];
    int64_t* start;  /* ncells + 1 */
    int64_t* items;  /* n */
} cellist_t;

static void cellist_build(const or_cfg* c, int64_t n, const double* x3, cellist_t* L)
{
    or_cell_geometry(c, L->nc, L->cl);
    int64_t ncells = (int64_t)L->nc[0] * L->nc[1] * L->nc[2];
    L->start = (int64_t*)calloc((size_t)ncells + 1, sizeof(int64_t));
    L->items = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* keys = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    or_cell_order(c, n, x3, L->items, keys);
    for (int64_t i = 0; i < n; i++) L->start[keys[i] + 1]++;
    for (int64_t b = 0; b < ncells; b++) L->start[b + 1] += L->start[b];
    free(keys);
}

static void cellist_free(cellist_t* L)
{
    free(L->start);
    free(L->items);
}

/* candidates of particle i from its 3^d stencil, filtered by r^2 < R^2 */
static int64_t cell_query(const or_cfg* c, const cellist_t* L, const double* x3, int64_t i,
                          int64_t* out, int64_t cap)
{
    double R = support_R(c), R2 = R * R;
    int cc[3];
    cell_coords(c, L->nc, L->cl, x3 + 3 * i, cc);
    int lo3[3] = {0, 0, 0}, hi3[3] = {0, 0, 0};
    for (int a = 0; a < c->dim; a++) { lo3[a] = -1; hi3[a] = 1; }
    int64_t cnt = 0;
    for (int dz = lo3[2]; dz <= hi3[2]; dz++)
        for (int dy = lo3[1]; dy <= hi3[1]; dy++)
            for (int dx = lo3[0]; dx <= hi3[0]; dx++) {
                int dd[3] = {dx, dy, dz};
                int q[3];
                int skip = 0;
                for (int a = 0; a < 3; a++) {
                    int v = cc[a] + dd[a];
                    if (a < c->dim) {
                        if (c->periodic[a]) v = (v + L->nc[a]) % L->nc[a];
                        else if (v < 0 || v >= L->nc[a]) skip = 1;
                    }
                    q[a] = v;
                }
                if (skip) continue;
                int64_t key = (int64_t)q[0] + (int64_t)L->nc[0] * ((int64_t)q[1] + (int64_t)L->nc[1] * (int64_t)q[2]);
                for (int64_t t = L->start[key]; t < L->start[key + 1]; t++) {
                    int64_t j = L->items[t];
                    if (j == i) continue;
                    double d[3];
                    if (rij(c, x3 + 3 * i, x3 + 3 * j, d) < R2) {
                        if (out && cnt < cap) out[cnt] = j;
                        cnt++;
                    }
                }
            }
    if (out && cnt <= cap) qsort(out, (size_t)cnt, sizeof(int64_t), cmp_i64);
    return cnt;
}

static int64_t brute_query(const or_cfg* c, int64_t n, const double* x3, int64_t i,
                           int64_t* out, int64_t cap)
{
    double R = support_R(c), R2 = R * R;
    int64_t cnt = 0;
    for (int64_t j = 0; j < n; j++) {
        if (j == i) continue;
        double d[3];
        if (rij(c, x3 + 3 * i, x3 + 3 * j, d) < R2) {
            if (out && cnt < cap) out[cnt] = j;
            cnt++;
        }
    }
    return cnt;
}

int64_t or_neighbors_cell(const or_cfg* c, int64_t n, const double* x3, int64_t nd,
                          const int64_t* dests, int64_t* off, int64_t* nbr, int64_t cap)
{
    cellist_t L;
    cellist_build(c, n, x3, &L);
    int64_t m = dests ? nd : n;
    off[0] = 0;
    for (int64_t t = 0; t < m; t++) {
        int64_t i = dests ? dests[t] : t;
        off[t + 1] = off[t] + cell_query(c, &L, x3, i, NULL, 0);
    }
    int64_t total = off[m];
    if (total > cap) { cellist_free(&L); return -1; }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < m; t++) {
        int64_t i = dests ? dests[t] : t;
        cell_query(c, &L, x3, i, nbr + off[t], off[t + 1] - off[t]);
    }
    cellist_free(&L);
    return total;
}

int64_t or_neighbors_brute(const or_cfg* c, int64_t n, const double* x3, int64_t nd,
                           const int64_t* dests, int64_t* off, int64_t* nbr, int64_t cap)
{
    int64_t m = dests ? nd : n;
    off[0] = 0;
    for (int64_t t = 0; t < m; t++) {
        int64_t i = dests ? dests[t] : t;
        off[t + 1] = off[t] + brute_query(c, n, x3, i, NULL, 0);
    }
    int64_t total = off[m];
    if (total > cap) return -1;
    for (int64_t t = 0; t < m; t++) {
        int64_t i = dests ? dests[t] : t;
        brute_query(c, n, x3, i, nbr + off[t], off[t + 1] - off[t]);
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* Simulation state                                                          */
/* ------------------------------------------------------------------------ */
struct or_sim {
    or_cfg c;
    int64_t n;
    int32_t* tag;
    double *x, *u, *ut, *m, *rho, *p;   /* state; u of a wall = its ghost velocity */
    double* uw;                         /* prescribed wall velocity u_i of eq:vg-adami (walls; 0 fluid) */
    int pref_set;                       /* R33: p_ref already taken */
    int error;                          /* R34: dormant pool exhausted */
    double *xs, *us;                    /* r*, u* (walls: xs = x, us = wall u*) */
    double *rhs, *diag, *fs;            /* PPE scratch */
    double* nrm;                        /* wall unit normals */
    double* xk;                         /* GTVF sub-step positions r^K */
    double* anp;                        /* f_visc + f_avisc + f_astress + f_body of the last predict */
    double* ftot;                       /* f^n = anp + f_p of the last correct */
    int stepped;                        /* a correct has completed (ftot valid) */
    double lambda;
    csr_t nb[2];                        /* 0: built at x (r^n), 1: built at xs (r*) */
};

static double* dalloc(int64_t n)
{
    return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
}

static void csr_free(csr_t* b)
{
    free(b->off);
    free(b->nbr);
    b->off = NULL;
    b->nbr = NULL;
    b->built = 0;
}

/* build the neighbour rows of the listed dests (all if nd == 0) */
static void csr_build(or_sim* s, int which, const double* x3, int64_t nd, const int64_t* dests)
{
    csr_t* b = &s->nb[which];
    csr_free(b);
    int64_t n = s->n;
    cellist_t L;
    cellist_build(&s->c, n, x3, &L);
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t m = nd > 0 ? nd : n;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < m; t++) {
        int64_t i = nd > 0 ? dests[t] : t;
        cnt[i] = cell_query(&s->c, &L, x3, i, NULL, 0);
    }
    b->off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) b->off[i + 1] = b->off[i] + cnt[i];
    b->nbr = (int64_t*)malloc((size_t)(b->off[n] > 0 ? b->off[n] : 1) * sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < m; t++) {
        int64_t i = nd > 0 ? dests[t] : t;
        cell_query(&s->c, &L, x3, i, b->nbr + b->off[i], cnt[i]);
    }
    b->nd = n;
    b->built = 1;
    free(cnt);
    cellist_free(&L);
}

int64_t or_num_pairs(or_sim* s, int which)
{
    return s->nb[which].built ? s->nb[which].off[s->n] : -1;
}

static double dot(int dim, const double* a, const double* b)
{
    double r = a[0] * b[0] + a[1] * b[1];
    if (dim == 3) r = r + a[2] * b[2];
    return r;
}

/* eq:vg-no-normal: remove the into-solid normal component only */
static void clip_normal(int dim, double* uw, const double* n)
{
    double un = dot(dim, uw, n);
    if (un < 0.0)
        for (int a = 0; a < dim; a++) uw[a] -= un * n[a];
}

/* Wall normals, §3.4.1 eq:normal-approx / eq:normal, reading R17:
 * sources are wall particles; |n*| < 1/(4h) -> 0 else normalised; then the
 * SPH-smoothed sum (self included) is normalised, and a smoothed vector
 * shorter than 0.01 is set to zero. */
static void compute_normals(or_sim* s)
{
    const or_cfg* c = &s->c;
    int dim = c->dim;
    double h = c->h;
    double* ns = dalloc(3 * s->n);
    csr_t* b = &s->nb[0];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] != WALL) continue;
        double acc[3] = {0, 0, 0};
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            if (s->tag[j] != WALL) continue;
            double d[3], gw[3];
            double r = sqrt(rij(c, s->x + 3 * i, s->x + 3 * j, d));
            gradW(dim, d, r, h, gw);
            double vj = s->m[j] / s->rho[j];
            for (int a = 0; a < dim; a++) acc[a] -= vj * gw[a];
        }
        double mag = sqrt(dot(dim, acc, acc));
        if (mag < 1.0 / (4.0 * h)) acc[0] = acc[1] = acc[2] = 0.0;
        else for (int a = 0; a < dim; a++) acc[a] /= mag;
        for (int a = 0; a < 3; a++) ns[3 * i + a] = acc[a];
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] != WALL) continue;
        double w0 = or_W(dim, 0.0, h) * s->m[i] / s->rho[i];
        double acc[3];
        for (int a = 0; a < 3; a++) acc[a] = w0 * ns[3 * i + a];
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            if (s->tag[j] != WALL) continue;
            double d[3];
            double r = sqrt(rij(c, s->x + 3 * i, s->x + 3 * j, d));
            double wv = or_W(dim, r, h) * s->m[j] / s->rho[j];
            for (int a = 0; a < dim; a++) acc[a] += wv * ns[3 * j + a];
        }
        /* R17: a smoothed normal this short (e.g. the middle of three wall
         * layers, where the layers above and below cancel) has no direction;
         * it stays zero instead of normalising rounding noise */
        double mag = sqrt(dot(dim, acc, acc));
        for (int a = 0; a < 3; a++) s->nrm[3 * i + a] = mag >= 0.01 ? acc[a] / mag : 0.0;
    }
    free(ns);
}

/* R34: a dormant particle sits far below the domain in x (bounded axis), where
 * no distance test can accept it; its fields are zeroed */
static void park(or_sim* s, int64_t i)
{
    const or_cfg* c = &s->c;
    s->x[3 * i] = c->lo[0] - 1.0e3 * (c->hi[0] - c->lo[0] + 1.0);
    for (int a = 0; a < 3; a++) {
        s->u[3 * i + a] = s->ut[3 * i + a] = s->us[3 * i + a] = 0.0;
        s->xs[3 * i + a] = s->x[3 * i + a];
    }
    s->p[i] = 0.0;
}

or_sim* or_create(const or_cfg* c, int64_t n, const double* x3, const double* u3,
                  const double* m, const double* rho, const double* p, const int32_t* tag)
{
    or_sim* s = (or_sim*)calloc(1, sizeof(or_sim));
    s->c = *c;
    s->n = n;
    s->tag = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    memcpy(s->tag, tag, (size_t)n * sizeof(int32_t));
    s->x = dalloc(3 * n); s->u = dalloc(3 * n); s->ut = dalloc(3 * n);
    s->xs = dalloc(3 * n); s->us = dalloc(3 * n); s->nrm = dalloc(3 * n); s->xk = dalloc(3 * n);
    s->m = dalloc(n); s->rho = dalloc(n); s->p = dalloc(n);
    s->rhs = dalloc(n); s->diag = dalloc(n); s->fs = dalloc(n);
    s->anp = dalloc(3 * n); s->ftot = dalloc(3 * n); s->uw = dalloc(3 * n);
    memcpy(s->x, x3, (size_t)(3 * n) * sizeof(double));
    memcpy(s->xs, x3, (size_t)(3 * n) * sizeof(double));
    memcpy(s->u, u3, (size_t)(3 * n) * sizeof(double));
    memcpy(s->ut, u3, (size_t)(3 * n) * sizeof(double));  /* R23: u~0 = u0 */
    memcpy(s->m, m, (size_t)n * sizeof(double));
    memcpy(s->rho, rho, (size_t)n * sizeof(double));
    if (p) memcpy(s->p, p, (size_t)n * sizeof(double));
    /* a wall's creation velocity is its physical velocity (eq:vg-adami);
     * walls never move (R24): a moving lid slides along itself */
    for (int64_t i = 0; i < n; i++)
        if (tag[i] == WALL)
            for (int a = 0; a < 3; a++) {
                s->uw[3 * i + a] = u3[3 * i + a];
                s->ut[3 * i + a] = 0.0;
            }
    for (int64_t i = 0; i < n; i++)
        if (tag[i] == DORMANT) park(s, i);
    csr_build(s, 0, s->x, 0, NULL);
    compute_normals(s);
    return s;
}

void or_destroy(or_sim* s)
{
    if (!s) return;
    csr_free(&s->nb[0]);
    csr_free(&s->nb[1]);
    free(s->tag); free(s->x); free(s->u); free(s->ut); free(s->xs); free(s->us);
    free(s->nrm); free(s->xk); free(s->m); free(s->rho); free(s->p);
    free(s->rhs); free(s->diag); free(s->fs);
    free(s->anp); free(s->ftot); free(s->uw);
    free(s);
}

static double* field_ptr(or_sim* s, const char* f, int* ncomp)
{
    *ncomp = 1;
    if (!strcmp(f, "x")) { *ncomp = 3; return s->x; }
    if (!strcmp(f, "u")) { *ncomp = 3; return s->u; }
    if (!strcmp(f, "ut")) { *ncomp = 3; return s->ut; }
    if (!strcmp(f, "xs")) { *ncomp = 3; return s->xs; }
    if (!strcmp(f, "us")) { *ncomp = 3; return s->us; }
    if (!strcmp(f, "normal")) { *ncomp = 3; return s->nrm; }
    if (!strcmp(f, "xk")) { *ncomp = 3; return s->xk; }
    if (!strcmp(f, "m")) return s->m;
    if (!strcmp(f, "rho")) return s->rho;
    if (!strcmp(f, "p")) return s->p;
    if (!strcmp(f, "rhs")) return s->rhs;
    if (!strcmp(f, "diag")) return s->diag;
    if (!strcmp(f, "fs")) return s->fs;
    if (!strcmp(f, "ftot")) { *ncomp = 3; return s->ftot; }
    if (!strcmp(f, "uwall")) { *ncomp = 3; return s->uw; }
    if (!strcmp(f, "lambda")) return &s->lambda;
    return NULL;
}

int or_get(or_sim* s, const char* field, double* out)
{
    int nc;
    double* src = field_ptr(s, field, &nc);
    if (!src) return -1;
    int64_t cnt = !strcmp(field, "lambda") ? 1 : nc * s->n;
    memcpy(out, src, (size_t)cnt * sizeof(double));
    return 0;
}

int or_set(or_sim* s, const char* field, const double* in)
{
    int nc;
    double* dst = field_ptr(s, field, &nc);
    if (!dst) return -1;
    int64_t cnt = !strcmp(field, "lambda") ? 1 : nc * s->n;
    memcpy(dst, in, (size_t)cnt * sizeof(double));
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Passes of Algorithm 1                                         */
/* ------------------------------------------------------------------------ */

/* eq:summation_density, Alg. 1 line 2; reading R4: fluid (and,
 * if wall_rho_summation, wall) particles, fluid + wall sources, self
 * included; otherwise walls keep the rest density rho0.  Free-surface flag
 * rho_i / rho0 < 0.8 for fluid (R11). */
void or_pass_density(or_sim* s)
{
    const or_cfg* c = &s->c;
    csr_t* b = &s->nb[0];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        double rho = s->m[i] * or_W(c->dim, 0.0, c->h);
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            double d[3];
            double r = sqrt(rij(c, s->x + 3 * i, s->x + 3 * j, d));
            rho += s->m[j] * or_W(c->dim, r, c->h);
        }
        if (s->tag[i] == DORMANT) continue;
        if (s->tag[i] == WALL && !c->wall_rho_summation) rho = c->rho0;
        s->rho[i] = rho;
        s->fs[i] = (s->tag[i] == FLUID && rho / c->rho0 < c->fs_ratio) ? 1.0 : 0.0;
    }
}

/* Shepard average of a fluid vector field with W(r, h/2) (eq:vf);
 * no fluid within the support: the wall's own velocity (reading R15a) */
static void shepard_half(or_sim* s, const csr_t* b, const double* xpos, const double* f,
                         int64_t i, double* out)
{
    const or_cfg* c = &s->c;
    double sw = 0.0, acc[3] = {0, 0, 0};
    for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
        int64_t j = b->nbr[t];
        if (!LIQ(s->tag[j])) continue;
        double d[3];
        double r = sqrt(rij(c, xpos + 3 * i, xpos + 3 * j, d));
        double w = or_W(c->dim, r, 0.5 * c->h);
        for (int a = 0; a < c->dim; a++) acc[a] += f[3 * j + a] * w;
        sw += w;
    }
    for (int a = 0; a < 3; a++) out[a] = sw > 0.0 ? acc[a] / sw : s->uw[3 * i + a];
}

/* Ghost velocity (eq:vf, eq:vg-adami, eq:vg-no-normal, R15):
 * u_w = 2 u_wall - Shepard_{h/2}(u_f) with u_wall the wall's prescribed
 * velocity (s->uw), then clip. */
void or_pass_ghost_velocity(or_sim* s)
{
    const or_cfg* c = &s->c;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] != WALL) continue;
        double ut[3];
        shepard_half(s, &s->nb[0], s->x, s->u, i, ut);
        const double* uwall = s->uw + 3 * i;
        double uw[3] = {2.0 * uwall[0] - ut[0], 2.0 * uwall[1] - ut[1], 2.0 * uwall[2] - ut[2]};
        clip_normal(c->dim, uw, s->nrm + 3 * i);
        for (int a = 0; a < 3; a++) s->u[3 * i + a] = a < c->dim ? uw[a] : 0.0;
    }
}

/* Non-pressure forces and predictors (Alg. 1 lines 3-5):
 *   f_visc  eq:mom:sph:visc, sources fluid + wall (R19)
 *   f_avisc eq:mom:sph:av, reading R20: phi = u_ij.r_ij/(r^2 + eta h^2),
 *           c = c_ref, rhobar = (rho_i + rho_j)/2, f = -sum m_j Pi_ij gradW,
 *           sources fluid + wall (ghost velocities)
 *   f_astress eq:mom:sph:gtvf:stress, reading R21, fluid sources
 *   f_body  = g
 *   u* = u^n + dt (sum f)  (eq:int:vint)
 *   r* = r^n + dt u~^n     (eq:int:rnp1)                                 */
static void pass_forces_predict(or_sim* s, double dt)
{
    const or_cfg* c = &s->c;
    int dim = c->dim;
    double h = c->h;
    csr_t* b = &s->nb[0];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] == INLET || s->tag[i] == OUTLET) {
            /* R34: prescribed / frozen velocity (no momentum update), moved like fluid to r* */
            for (int a = 0; a < 3; a++) {
                s->us[3 * i + a] = s->u[3 * i + a];
                s->xs[3 * i + a] = a < dim ? s->x[3 * i + a] + dt * s->ut[3 * i + a] : 0.0;
                s->anp[3 * i + a] = 0.0;
            }
            wrap_pos(c, s->xs + 3 * i);
            continue;
        }
        if (s->tag[i] != FLUID) {
            for (int a = 0; a < 3; a++) s->xs[3 * i + a] = s->x[3 * i + a];
            continue;
        }
        const double* ui = s->u + 3 * i;
        const double* uti = s->ut + 3 * i;
        double rhoi = s->rho[i];
        double acc[3] = {0, 0, 0};
        for (int a = 0; a < dim; a++) acc[a] = c->g[a];
        double dui[3] = {uti[0] - ui[0], uti[1] - ui[1], uti[2] - ui[2]};
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            double d[3], gw[3];
            double r2 = rij(c, s->x + 3 * i, s->x + 3 * j, d);
            double r = sqrt(r2);
            double dwdr = or_dWdr(dim, r, h);
            gradW(dim, d, r, h, gw);
            const double* uj = s->u + 3 * j;
            double rhoj = s->rho[j], mj = s->m[j];
            double uij[3] = {ui[0] - uj[0], ui[1] - uj[1], ui[2] - uj[2]};
            if (c->nu > 0.0) {
                double f = mj * 4.0 * c->nu / (rhoi + rhoj) * (r * dwdr) / (r2 + c->eta * h * h);
                for (int a = 0; a < dim; a++) acc[a] += f * uij[a];
            }
            if (c->alpha > 0.0) {
                double vr = dot(dim, uij, d);
                if (vr < 0.0) {
                    double phi = vr / (r2 + c->eta * h * h);
                    double rhobar = 0.5 * (rhoi + rhoj);
                    double Pi = -c->alpha * h * c->c_ref * phi / rhobar;
                    for (int a = 0; a < dim; a++) acc[a] -= mj * Pi * gw[a];
                }
            }
            if (LIQ(s->tag[j])) {
                const double* utj = s->ut + 3 * j;
                double duj[3] = {utj[0] - uj[0], utj[1] - uj[1], utj[2] - uj[2]};
                double ai = dot(dim, dui, gw) / rhoi;
                double aj = dot(dim, duj, gw) / rhoj;
                for (int a = 0; a < dim; a++) acc[a] += mj * (ui[a] * ai + uj[a] * aj);
            }
        }
        for (int a = 0; a < 3; a++) {
            s->us[3 * i + a] = a < dim ? ui[a] + dt * acc[a] : 0.0;
            s->xs[3 * i + a] = a < dim ? s->x[3 * i + a] + dt * uti[a] : 0.0;
            s->anp[3 * i + a] = a < dim ? acc[a] : 0.0;
        }
        wrap_pos(c, s->xs + 3 * i);
    }
}

/* Wall u* (reading R16): slip u*_w = Shepard_{h/2}(u*_f),
 * no-slip u*_w = 2 u_wall - Shepard_{h/2}(u*_f); then the normal clip. */
static void pass_wall_ustar(or_sim* s)
{
    const or_cfg* c = &s->c;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] != WALL) continue;
        double ut[3];
        shepard_half(s, &s->nb[1], s->xs, s->us, i, ut);
        double uw[3];
        for (int a = 0; a < 3; a++) uw[a] = c->ustar_noslip ? 2.0 * s->uw[3 * i + a] - ut[a] : ut[a];
        clip_normal(c->dim, uw, s->nrm + 3 * i);
        for (int a = 0; a < 3; a++) s->us[3 * i + a] = a < c->dim ? uw[a] : 0.0;
    }
}

/* fac_ij = 4 m_j / (rho_i (rho_i + rho_j)) * r_ij.gradW_ij / (r^2 + eta h^2)
 * (eq:coeff / eq:coeff1, regulariser per reading R6) */
static double pair_fac(const or_cfg* c, double mj, double rhoi, double rhoj, double r2)
{
    double r = sqrt(r2);
    double dwdr = or_dWdr(c->dim, r, c->h);
    return 4.0 * mj / (rhoi * (rhoi + rhoj)) * (r * dwdr) / (r2 + c->eta * c->h * c->h);
}

/* RHS_i (right side of eq:sph-ppe, R8), D_ii (eq:coeff, R7) and
 * Lambda = max |RHS_i / D_ii| (eq:convergence, R12). */
static void pass_rhs_diag(or_sim* s, double dt)
{
    const or_cfg* c = &s->c;
    int dim = c->dim;
    csr_t* b = &s->nb[1];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++) {
        if (!UNKNOWN(s->tag[i])) { s->rhs[i] = 0.0; s->diag[i] = 0.0; continue; }
        double rhs = 0.0, diag = 0.0, rhoi = s->rho[i];
        const double* usi = s->us + 3 * i;
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            double d[3], gw[3];
            double r2 = rij(c, s->xs + 3 * i, s->xs + 3 * j, d);
            double r = sqrt(r2);
            gradW(dim, d, r, c->h, gw);
            const double* usj = s->us + 3 * j;
            double usij[3] = {usi[0] - usj[0], usi[1] - usj[1], usi[2] - usj[2]};
            rhs += -(s->m[j] / (s->rho[j] * dt)) * dot(dim, usij, gw);
            diag += pair_fac(c, s->m[j], rhoi, s->rho[j], r2);
        }
        s->rhs[i] = rhs;
        s->diag[i] = diag;
    }
    double lam = 0.0;
    for (int64_t i = 0; i < s->n; i++) {
        if (!UNKNOWN(s->tag[i]) || s->fs[i] != 0.0 || s->diag[i] == 0.0) continue;
        double v = fabs(s->rhs[i] / s->diag[i]);
        if (v > lam) lam = v;
    }
    s->lambda = lam;
}

/* Wall pressure eq:p-shepard, reading R14: fluid sources,
 * W(r, h), a_w = 0, sum W = 0 -> 0, clamp p_w < 0 -> 0 if configured. */
static double wall_pressure_one(or_sim* s, const double* pk, int64_t i)
{
    const or_cfg* c = &s->c;
    csr_t* b = &s->nb[1];
    double sw = 0.0, sp = 0.0, sr[3] = {0, 0, 0};
    for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
        int64_t j = b->nbr[t];
        if (!LIQ(s->tag[j])) continue;
        double d[3];
        double r = sqrt(rij(c, s->xs + 3 * i, s->xs + 3 * j, d));
        double w = or_W(c->dim, r, c->h);
        sp += pk[j] * w;
        for (int a = 0; a < c->dim; a++) sr[a] += s->rho[j] * d[a] * w;
        sw += w;
    }
    double pw = 0.0;
    if (sw > 0.0) pw = (sp + dot(c->dim, c->g, sr)) / sw;
    if (c->clamp_wall_p && pw < 0.0) pw = 0.0;
    return pw;
}

void or_pass_wall_pressure(or_sim* s, const double* pk, double* pw_out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; i++)
        if (s->tag[i] == WALL) pw_out[i] = wall_pressure_one(s, pk, i);
}

/* One damped-Jacobi (SOR) update, eq:p-sor, with the special
 * cases of P:530-534 (R11): D_ii == 0 or free surface -> 0. */
static double sweep_one(or_sim* s, const double* pk, int64_t i)
{
    const or_cfg* c = &s->c;
    if (s->fs[i] != 0.0 || s->diag[i] == 0.0) return 0.0;
    csr_t* b = &s->nb[1];
    double S = 0.0, rhoi = s->rho[i];
    for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
        int64_t j = b->nbr[t];
        double d[3];
        double r2 = rij(c, s->xs + 3 * i, s->xs + 3 * j, d);
        S += pair_fac(c, s->m[j], rhoi, s->rho[j], r2) * pk[j];   /* = -OD_ij p_j */
    }
    return c->omega * (s->rhs[i] + S) / s->diag[i] + (1.0 - c->omega) * pk[i];
}

void or_pass_sweep(or_sim* s, const double* pk, int64_t nd, const int64_t* dests, double* out)
{
    if (nd > 0) {
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < nd; t++) out[t] = sweep_one(s, pk, dests[t]);
    } else {
        int64_t t = 0;
        for (int64_t i = 0; i < s->n; i++)
            if (UNKNOWN(s->tag[i])) out[t++] = sweep_one(s, pk, i);
    }
}

/* the r*-stage of or_predict (A9-A11) from the current xs / us: neighbours at r*,
 * wall u*, RHS, D_ii, Lambda.  Tests call it after replacing xs by the r* a
 * working-precision (fp32) handle holds, so that both sides evaluate the pressure
 * solve on the same positions (reading R36); or_predict runs it itself. */
void or_predict_stage2(or_sim* s, double dt)
{
    csr_build(s, 1, s->xs, 0, NULL);                /* neighbours at r* (R3) */
    pass_wall_ustar(s);                             /* A10 */
    pass_rhs_diag(s, dt);                           /* line 6 + Lambda */
}

void or_predict(or_sim* s, double dt)
{
    csr_build(s, 0, s->x, 0, NULL);                 /* neighbours at r^n (R3) */
    or_pass_density(s);                             /* line 2 */
    or_pass_ghost_velocity(s);                      /* A7 */
    pass_forces_predict(s, dt);                     /* lines 3-5 */
    or_predict_stage2(s, dt);                       /* A9-A11 at r* */
}

/* Lines 7-10: iterate eq:p-sor from p^0 = p(t) (R10) until eq:convergence
 * holds (iterate UNTIL, R12), at least min(2, max_iter) sweeps (R13). Walls
 * are refreshed from p^k at the start of every sweep (R14). */
void or_solve(or_sim* s, double tol, int max_iter, or_report* rep)
{
    int64_t n = s->n;
    double* pk = dalloc(n);
    double* pn = dalloc(n);
    memcpy(pk, s->p, (size_t)n * sizeof(double));
    int min_it = s->c.min_iter < max_iter ? s->c.min_iter : max_iter;
    int k = 0;
    double res = 0.0;
    for (;;) {
        or_pass_wall_pressure(s, pk, pk);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++)
            pn[i] = UNKNOWN(s->tag[i]) ? sweep_one(s, pk, i) : pk[i];
        if (s->c.ppe_mean_free) {
            /* reading R32: without a Dirichlet row (no free surface) the PPE operator has the
             * constant null space (its rows sum to zero, eq:coeff / eq:coeff1) and the Jacobi
             * iterate drifts along it; remove the mean of the live rows, in id order */
            double sum = 0.0;
            int64_t cnt = 0;
            for (int64_t i = 0; i < n; i++)
                if (UNKNOWN(s->tag[i]) && s->fs[i] == 0.0 && s->diag[i] != 0.0) {
                    sum += pn[i];
                    cnt++;
                }
            if (cnt > 0) {
                double m = sum / (double)cnt;
                for (int64_t i = 0; i < n; i++)
                    if (UNKNOWN(s->tag[i]) && s->fs[i] == 0.0 && s->diag[i] != 0.0) pn[i] -= m;
            }
        }
        double num = 0.0, den = 0.0;
        int64_t nfl = 0;
        for (int64_t i = 0; i < n; i++) {
            if (!UNKNOWN(s->tag[i])) continue;
            num += fabs(pn[i] - pk[i]);
            den += fabs(pn[i]);
            nfl++;
        }
        if (s->c.conv_mean && nfl > 0) {
            /* reading R12b: the text calls the denominator "the mean pressure" and Lambda "a
             * measure of the mean pressure": compare means, not sums */
            num /= (double)nfl;
            den /= (double)nfl;
        }
        double dd = den > s->lambda ? den : s->lambda;
        if (num == 0.0) res = 0.0;
        else res = dd > 0.0 ? num / dd : INFINITY;
        memcpy(pk, pn, (size_t)n * sizeof(double));
        k++;
        if ((k >= min_it && res < tol) || k >= max_iter) break;
    }
    memcpy(s->p, pk, (size_t)n * sizeof(double));
    if (rep) { rep->iters = k; rep->residual = res; rep->lambda = s->lambda; }
    free(pk);
    free(pn);
}

/* Lines 11-19: final wall pressure, f_p and corrector (eq:int:vnp1), modified
 * GTVF sub-steps (eq:int:gtvf:pos, eq:int:gtvf:vel:tmp) with the pair set
 * frozen at r* (P:454-456), transport velocity (eq:int:vhatnp2) and position
 * update (eq:int:rnp2) from r^n (R24). */
/* R34 conversions after the position update, each in id order:
 *   outlet with x >= x_end     -> dormant (its id returns to the pool)
 *   fluid with x >= x_outlet   -> outlet (u, p frozen from now on)
 *   inlet with x >= x_inlet    -> fluid; the lowest dormant id becomes a new inlet
 *                                 particle at x - inlet_length (same y, z, u, m, rho, p) */
static void open_boundaries(or_sim* s)
{
    const or_cfg* c = &s->c;
    int64_t n = s->n;
    for (int64_t i = 0; i < n; i++)
        if (s->tag[i] == OUTLET && s->x[3 * i] >= c->x_end) {
            s->tag[i] = DORMANT;
            park(s, i);
        }
    for (int64_t i = 0; i < n; i++)
        if (s->tag[i] == FLUID && s->x[3 * i] >= c->x_outlet) s->tag[i] = OUTLET;
    int64_t pool = 0;   /* next candidate dormant id (ids only increase within a step) */
    for (int64_t i = 0; i < n; i++) {
        if (s->tag[i] != INLET || s->x[3 * i] < c->x_inlet) continue;
        s->tag[i] = FLUID;
        while (pool < n && s->tag[pool] != DORMANT) pool++;
        if (pool == n) { s->error = 1; continue; }
        int64_t k = pool++;
        s->tag[k] = INLET;
        for (int a = 0; a < 3; a++) {
            s->x[3 * k + a] = s->x[3 * i + a];
            s->u[3 * k + a] = s->ut[3 * k + a] = s->u[3 * i + a];
            s->xs[3 * k + a] = s->us[3 * k + a] = 0.0;
        }
        s->x[3 * k] -= c->inlet_length;
        s->m[k] = s->m[i];
        s->rho[k] = s->rho[i];
        s->p[k] = s->p[i];
    }
}

int or_error(or_sim* s) { return s->error; }

void or_get_tags(or_sim* s, int32_t* out) { memcpy(out, s->tag, (size_t)s->n * sizeof(int32_t)); }

void or_correct(or_sim* s, double dt)
{
    const or_cfg* c = &s->c;
    int dim = c->dim;
    int64_t n = s->n;
    csr_t* b = &s->nb[1];
    or_pass_wall_pressure(s, s->p, s->p);
    double* unew = dalloc(3 * n);
    /* pressure gradient: eq:mom:sph:press:symm / eq:mom:sph:press:pij (R18) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (s->tag[i] != FLUID) continue;
        double acc[3] = {0, 0, 0};
        double rhoi = s->rho[i], pi = s->p[i];
        for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
            int64_t j = b->nbr[t];
            double d[3], gw[3];
            double r = sqrt(rij(c, s->xs + 3 * i, s->xs + 3 * j, d));
            gradW(dim, d, r, c->h, gw);
            double rhoj = s->rho[j], pj = s->p[j], mj = s->m[j];
            double f;
            if (c->pgrad == 0) f = mj * (pi / (rhoi * rhoi) + pj / (rhoj * rhoj));
            else f = mj / (rhoi * rhoj) * (pj - pi);
            for (int a = 0; a < dim; a++) acc[a] -= f * gw[a];
        }
        for (int a = 0; a < dim; a++) {
            unew[3 * i + a] = s->us[3 * i + a] + dt * acc[a];
            s->ftot[3 * i + a] = s->anp[3 * i + a] + acc[a];   /* f^n = f_np + f_p */
        }
    }
    s->stepped = 1;
    if (c->pref_auto && !s->pref_set) {
        /* reading R33: internal flows take p_ref = 2 max(p_i) "after the first iteration"
         * -- here: over the fluid, from this first solve */
        double mx = -INFINITY;
        for (int64_t i = 0; i < n; i++)
            if (s->tag[i] == FLUID && s->p[i] > mx) mx = s->p[i];
        s->c.p_ref = n > 0 && mx > -INFINITY ? 2.0 * mx : 0.0;
        s->pref_set = 1;
    }
    /* GTVF background pressure p0 (R22) and K sub-steps */
    double* p0 = dalloc(n);
    for (int64_t i = 0; i < n; i++) {
        if (c->pref_external) {
            double v = 10.0 * fabs(s->p[i]);
            p0[i] = v < c->p_ref ? v : c->p_ref;
        } else {
            p0[i] = c->p_ref;
        }
    }
    double* rk = s->xk;
    double* rn = dalloc(3 * n);
    double* vk = dalloc(3 * n);
    double* fk = dalloc(3 * n);
    memcpy(rk, s->xs, (size_t)(3 * n) * sizeof(double));
    double ht = c->h_tilde_factor * c->h;
    double dtau = dt / c->K;
    for (int k = 0; k < c->K; k++) {
        /* f_GTVF(r^k) = -p0_i sum_j m_j / rho_j^2 gradW(r_ij, h~) (eq:mom:sph:gtvf) */
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            if (s->tag[i] != FLUID) continue;
            double acc[3] = {0, 0, 0};
            for (int64_t t = b->off[i]; t < b->off[i + 1]; t++) {
                int64_t j = b->nbr[t];
                double d[3], gw[3];
                double r = sqrt(rij(c, rk + 3 * i, rk + 3 * j, d));
                gradW(dim, d, r, ht, gw);
                double f = s->m[j] / (s->rho[j] * s->rho[j]);
                for (int a = 0; a < dim; a++) acc[a] += f * gw[a];
            }
            for (int a = 0; a < dim; a++) fk[3 * i + a] = -p0[i] * acc[a];
        }
        memcpy(rn, rk, (size_t)(3 * n) * sizeof(double));
        for (int64_t i = 0; i < n; i++) {
            if (s->tag[i] != FLUID) continue;
            for (int a = 0; a < dim; a++) {
                rn[3 * i + a] = rk[3 * i + a] + dtau * vk[3 * i + a] + 0.5 * dtau * dtau * fk[3 * i + a];
                vk[3 * i + a] = vk[3 * i + a] + dtau * fk[3 * i + a];
            }
        }
        memcpy(rk, rn, (size_t)(3 * n) * sizeof(double));
    }
    /* R34: the outlet's advection velocity, Shepard_h of the fluid's u_x^{n+1} at r*, the
     * positions of the pressure solve (fluid sources of the r* list; none in the
     * support: the frozen u_x) */
    double* uout = dalloc(n);
    if (c->open_x) {
        const csr_t* b0 = &s->nb[1];
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            if (s->tag[i] != OUTLET) continue;
            double sw = 0.0, su = 0.0;
            for (int64_t t = b0->off[i]; t < b0->off[i + 1]; t++) {
                int64_t j = b0->nbr[t];
                if (s->tag[j] != FLUID) continue;
                double d[3];
                double w = or_W(dim, sqrt(rij(c, s->xs + 3 * i, s->xs + 3 * j, d)), c->h);
                su += unew[3 * j] * w;
                sw += w;
            }
            uout[i] = sw > 0.0 ? su / sw : s->u[3 * i];
        }
    }
    /* transport velocity and positions */
    for (int64_t i = 0; i < n; i++) {
        if (s->tag[i] == INLET) {
            /* prescribed velocity: r^{n+1} = r^n + dt u, u~ = u */
            for (int a = 0; a < dim; a++) {
                s->x[3 * i + a] += dt * s->u[3 * i + a];
                s->ut[3 * i + a] = s->u[3 * i + a];
            }
            wrap_pos(c, s->x + 3 * i);
            continue;
        }
        if (s->tag[i] == OUTLET) {
            /* u, p frozen; moved along x with the extrapolated fluid u_x */
            s->x[3 * i] += dt * uout[i];
            s->ut[3 * i] = uout[i];
            for (int a = 1; a < 3; a++) s->ut[3 * i + a] = 0.0;
            continue;
        }
        if (s->tag[i] != FLUID) continue;
        for (int a = 0; a < dim; a++) {
            double utn = unew[3 * i + a] + (rk[3 * i + a] - s->xs[3 * i + a]) / dt;
            s->x[3 * i + a] = s->x[3 * i + a] + 0.5 * dt * (utn + s->ut[3 * i + a]);
            s->ut[3 * i + a] = utn;
            s->u[3 * i + a] = unew[3 * i + a];
        }
        wrap_pos(c, s->x + 3 * i);
    }
    if (c->open_x) open_boundaries(s);
    free(unew); free(p0); free(rn); free(vk); free(fk); free(uout);
}

/* Adaptive time step:
 *   dt_cfl   = 0.25 h / max_i |u_i^n|          (max over fluid, velocities after the step)
 *   dt_force = 0.25 sqrt(h / max_i |f_i^n|),  f^n = f_p + f_visc + f_body + f_avisc + f_astress
 *   dt^{n+1} = min(dt_cfl, dt_force)
 * An unrestricted criterion (zero maximum) is +infinity.  Returns -1 if no
 * step has completed. */
int or_next_dt(or_sim* s, double* dt_next, double* dt_cfl, double* dt_force)
{
    if (!s->stepped) return -1;
    int dim = s->c.dim;
    double um = 0.0, fm = 0.0;
    for (int64_t i = 0; i < s->n; i++) {
        if (s->tag[i] != FLUID) continue;
        double u2 = 0.0, f2 = 0.0;
        for (int a = 0; a < dim; a++) {
            u2 += s->u[3 * i + a] * s->u[3 * i + a];
            f2 += s->ftot[3 * i + a] * s->ftot[3 * i + a];
        }
        if (u2 > um) um = u2;
        if (f2 > fm) fm = f2;
    }
    double h = s->c.h;
    double a = um > 0.0 ? 0.25 * h / sqrt(um) : INFINITY;
    double b = fm > 0.0 ? 0.25 * sqrt(h / sqrt(fm)) : INFINITY;
    if (dt_cfl) *dt_cfl = a;
    if (dt_force) *dt_force = b;
    if (dt_next) *dt_next = a < b ? a : b;
    return 0;
}

void or_step(or_sim* s, double dt, or_report* rep)
{
    or_predict(s, dt);
    or_solve(s, s->c.tol, s->c.max_iter, rep);
    or_correct(s, dt);
}
