/*
 * mgard_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never shipped).
 *
 * A plain-C, scalar restatement of the reference HPDR MGARD path
 * (/root/reference/pkg/src/hpdr/mgard/ and hpdr/huffman.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product (paper_2503_06322_b200) never links it.
 *
 * Parity is pinned against golden vectors produced by running the reference
 * itself (tests/golden/gen_golden.py): bit-exact coefficients, keys, Huffman
 * streams and whole blobs.
 *
 * Numerics: IEEE double, no FMA (compile with -ffp-contract=off), and the
 * reference's operation order.  Loops over independent
 * lines / units are OpenMP-parallel; results do not depend on thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "mgard_oracle.h"

#define MAXL 64
#define BLOCK_SYMBOLS 4096        /* huffman.py:29 */
#define MAX_CODE_LEN 32           /* huffman.py:30 */
#define MAX_DICT 65535            /* huffman.py:31 */

static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------------ */
/* hierarchy.py:63-97 build_hierarchy                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
    int rank, L;
    uint64_t dims[4];
    uint64_t cnt[4][MAXL];
    int64_t *map[4][MAXL];  /* finest indices of nodes surviving k coarsenings */
} hier_t;

static void hier_free(hier_t *h) {
    for (int d = 0; d < h->rank; d++)
        for (int k = 0; k < h->L; k++) free(h->map[d][k]);
}

static int hier_build(hier_t *h, int rank, const uint64_t *dims) {
    memset(h, 0, sizeof(*h));
    if (rank < 1 || rank > 4) return ORC_VALIDATION;
    h->rank = rank;
    int nco = 0;
    for (int d = 0; d < rank; d++) {
        if (dims[d] < 1) return ORC_VALIDATION;
        h->dims[d] = dims[d];
        uint64_t n = dims[d];
        int steps = 0;
        while (n > 2) { n = n / 2 + 1; steps++; }      /* coarsen, hierarchy.py:16 */
        if (steps > nco) nco = steps;
    }
    h->L = nco + 1;
    for (int d = 0; d < rank; d++) {
        uint64_t D = dims[d];
        h->cnt[d][0] = D;
        h->map[d][0] = malloc(sizeof(int64_t) * D);
        for (uint64_t i = 0; i < D; i++) h->map[d][0][i] = (int64_t)i;
        for (int k = 1; k <= nco; k++) {
            uint64_t n = h->cnt[d][k - 1];
            if ((n <= 2 && D >= 2) || D == 1) {   /* finished / degenerate dims repeat (:83-90) */
                h->cnt[d][k] = n;
                h->map[d][k] = malloc(sizeof(int64_t) * n);
                memcpy(h->map[d][k], h->map[d][k - 1], sizeof(int64_t) * n);
                continue;
            }
            uint64_t nc = n / 2 + 1;
            h->cnt[d][k] = nc;
            h->map[d][k] = malloc(sizeof(int64_t) * nc);
            for (uint64_t i = 0; i < nc; i++) {
                uint64_t s = 2 * i < n - 1 ? 2 * i : n - 1;   /* :92 clamp */
                h->map[d][k][i] = h->map[d][k - 1][s];
            }
        }
    }
    return ORC_OK;
}

int orc_hierarchy(int rank, const uint64_t *dims, int *L, uint64_t *counts /* rank*L, may be NULL */) {
    hier_t h;
    int rc = hier_build(&h, rank, dims);
    if (rc) return rc;
    *L = h.L;
    if (counts)
        for (int d = 0; d < rank; d++)
            for (int k = 0; k < h.L; k++) counts[d * h.L + k] = h.cnt[d][k];
    hier_free(&h);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* transform.py:45-128 per-(transition, axis) operator tables                */
/* ------------------------------------------------------------------------ */
typedef struct {
    int active;
    uint64_t n, nc, nfo;
    uint64_t *sel;          /* nc */
    uint64_t *fo, *ai, *bi; /* nfo */
    double *t;              /* nfo */
    double *ml, *md, *mu;   /* fine mass bands, n */
    double *tw, *tb, *tu;   /* coarse Thomas factors (w, b', upper), nc */
} axop_t;

static void mass_bands(const int64_t *coords, uint64_t n, double *lo, double *di, double *up) {
    /* transform.py:67-78 _mass_tridiag: diag accumulates h/3 twice, in this order */
    for (uint64_t i = 0; i < n; i++) { lo[i] = 0.0; di[i] = 0.0; up[i] = 0.0; }
    for (uint64_t i = 0; i + 1 < n; i++) {
        double h = (double)(coords[i + 1] - coords[i]);
        di[i] += h / 3.0;
    }
    for (uint64_t i = 0; i + 1 < n; i++) {
        double h = (double)(coords[i + 1] - coords[i]);
        di[i + 1] += h / 3.0;
        lo[i + 1] = h / 6.0;
        up[i] = h / 6.0;
    }
}

static void axop_free(axop_t *o) {
    if (!o->active) return;
    free(o->sel); free(o->fo); free(o->ai); free(o->bi); free(o->t);
    free(o->ml); free(o->md); free(o->mu); free(o->tw); free(o->tb); free(o->tu);
}

static void axop_build(axop_t *o, const int64_t *fine, uint64_t n, const int64_t *coarse, uint64_t nc) {
    memset(o, 0, sizeof(*o));
    if (n == nc) return;                                /* :92-94 inactive */
    o->active = 1; o->n = n; o->nc = nc;
    o->sel = malloc(sizeof(uint64_t) * nc);
    char *mask = calloc(n, 1);
    for (uint64_t c = 0; c < nc; c++) {
        o->sel[c] = 2 * c < n - 1 ? 2 * c : n - 1;
        mask[o->sel[c]] = 1;
    }
    o->nfo = n - nc;
    o->fo = malloc(sizeof(uint64_t) * o->nfo);
    o->ai = malloc(sizeof(uint64_t) * o->nfo);
    o->bi = malloc(sizeof(uint64_t) * o->nfo);
    o->t = malloc(sizeof(double) * o->nfo);
    uint64_t k = 0;
    for (uint64_t j = 0; j < n; j++) if (!mask[j]) o->fo[k++] = j;
    free(mask);
    for (k = 0; k < o->nfo; k++) {
        uint64_t f = o->fo[k];
        o->ai[k] = (f - 1) / 2;
        o->bi[k] = (f + 1 == n - 1) ? nc - 1 : (f + 1) / 2;
        double xa = (double)coarse[o->ai[k]], xb = (double)coarse[o->bi[k]], xj = (double)fine[f];
        o->t[k] = (xj - xa) / (xb - xa);
    }
    o->ml = malloc(sizeof(double) * n); o->md = malloc(sizeof(double) * n); o->mu = malloc(sizeof(double) * n);
    mass_bands(fine, n, o->ml, o->md, o->mu);
    double *cl = malloc(sizeof(double) * nc), *cd = malloc(sizeof(double) * nc);
    o->tu = malloc(sizeof(double) * nc);
    mass_bands(coarse, nc, cl, cd, o->tu);
    /* transform.py:81-89 _thomas_factors */
    o->tw = malloc(sizeof(double) * nc); o->tb = malloc(sizeof(double) * nc);
    o->tw[0] = 0.0; o->tb[0] = cd[0];
    for (uint64_t i = 1; i < nc; i++) {
        o->tw[i] = cl[i] / o->tb[i - 1];
        o->tb[i] = cd[i] - o->tw[i] * o->tu[i - 1];
    }
    free(cl); free(cd);
}

/* Export the tables for one transition so host-planner tests can compare. */
int orc_axis_tables(int rank, const uint64_t *dims, int step, int axis,
                    uint64_t *n_out, uint64_t *nc_out, double *t_out,
                    double *ml, double *md, double *mu, double *tw, double *tb, double *tu) {
    hier_t h;
    int rc = hier_build(&h, rank, dims);
    if (rc) return rc;
    if (step < 0 || step >= h.L - 1 || axis < 0 || axis >= rank) { hier_free(&h); return ORC_VALIDATION; }
    axop_t o;
    axop_build(&o, h.map[axis][step], h.cnt[axis][step], h.map[axis][step + 1], h.cnt[axis][step + 1]);
    *n_out = h.cnt[axis][step]; *nc_out = h.cnt[axis][step + 1];
    if (o.active) {
        if (t_out) memcpy(t_out, o.t, sizeof(double) * o.nfo);
        if (ml) { memcpy(ml, o.ml, 8 * o.n); memcpy(md, o.md, 8 * o.n); memcpy(mu, o.mu, 8 * o.n); }
        if (tw) { memcpy(tw, o.tw, 8 * o.nc); memcpy(tb, o.tb, 8 * o.nc); memcpy(tu, o.tu, 8 * o.nc); }
    }
    axop_free(&o);
    hier_free(&h);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Dense-array helpers: an axis view is (outer, n, inner).                    */
/* ------------------------------------------------------------------------ */
static void view(int rank, const uint64_t *sh, int a, uint64_t *outer, uint64_t *inner) {
    uint64_t o = 1, i = 1;
    for (int d = 0; d < a; d++) o *= sh[d];
    for (int d = a + 1; d < rank; d++) i *= sh[d];
    *outer = o; *inner = i;
}

static uint64_t prod(int rank, const uint64_t *sh) {
    uint64_t p = 1;
    for (int d = 0; d < rank; d++) p *= sh[d];
    return p;
}

/* Gather a sub-grid (per-dim index lists) of a dense array with shape sh. */
static void gather(int rank, const uint64_t *sh, const double *src,
                   const uint64_t *subsh, const int64_t *const *idx, double *dst) {
    uint64_t n = prod(rank, subsh);
    #pragma omp parallel for num_threads(g_threads) schedule(static)
    for (uint64_t f = 0; f < n; f++) {
        uint64_t r = f, off = 0, stride = 1;
        for (int d = rank - 1; d >= 0; d--) {
            uint64_t i = r % subsh[d]; r /= subsh[d];
            off += (uint64_t)idx[d][i] * stride;
            stride *= sh[d];
        }
        dst[f] = src[off];
    }
}

static void scatter(int rank, const uint64_t *sh, double *dst,
                    const uint64_t *subsh, const int64_t *const *idx, const double *src) {
    uint64_t n = prod(rank, subsh);
    #pragma omp parallel for num_threads(g_threads) schedule(static)
    for (uint64_t f = 0; f < n; f++) {
        uint64_t r = f, off = 0, stride = 1;
        for (int d = rank - 1; d >= 0; d--) {
            uint64_t i = r % subsh[d]; r /= subsh[d];
            off += (uint64_t)idx[d][i] * stride;
            stride *= sh[d];
        }
        dst[off] = src[f];
    }
}

/* transform.py:158-178 _prolong_axis: dst[sel]=src; dst[fo]=va+t*(vb-va) */
static void prolong_axis(int rank, const uint64_t *csh, int a, const axop_t *o, const double *src, double *dst) {
    uint64_t outer, inner;
    view(rank, csh, a, &outer, &inner);
    uint64_t nc = o->nc, n = o->n;
    #pragma omp parallel for num_threads(g_threads) schedule(static) collapse(2)
    for (uint64_t p = 0; p < outer; p++)
        for (uint64_t q = 0; q < inner; q++) {
            const double *s = src + p * nc * inner + q;
            double *d = dst + p * n * inner + q;
            for (uint64_t c = 0; c < nc; c++) d[o->sel[c] * inner] = s[c * inner];
            for (uint64_t k = 0; k < o->nfo; k++) {
                double va = s[o->ai[k] * inner], vb = s[o->bi[k] * inner];
                double diff = vb - va;
                double w = o->t[k] * diff;
                d[o->fo[k] * inner] = va + w;
            }
        }
}

/* transform.py:206-226 (_mass_mult_axis) then :181-203 (_restrict_axis) */
static void mass_restrict_axis(int rank, const uint64_t *fsh, int a, const axop_t *o, const double *src, double *dst) {
    uint64_t outer, inner;
    view(rank, fsh, a, &outer, &inner);
    uint64_t nc = o->nc, n = o->n;
    #pragma omp parallel num_threads(g_threads)
    {
        double *y = malloc(sizeof(double) * n);
        #pragma omp for schedule(static) collapse(2)
        for (uint64_t p = 0; p < outer; p++)
            for (uint64_t q = 0; q < inner; q++) {
                const double *x = src + p * n * inner + q;
                double *d = dst + p * nc * inner + q;
                for (uint64_t j = 0; j < n; j++) {
                    double v = o->md[j] * x[j * inner];
                    if (j >= 1) { double w = o->ml[j] * x[(j - 1) * inner]; v = v + w; }
                    if (j + 1 < n) { double w = o->mu[j] * x[(j + 1) * inner]; v = v + w; }
                    y[j] = v;
                }
                for (uint64_t c = 0; c < nc; c++) d[c * inner] = y[o->sel[c]];
                for (uint64_t k = 0; k < o->nfo; k++) {
                    double w = 1.0 - o->t[k];
                    double v = w * y[o->fo[k]];
                    d[o->ai[k] * inner] += v;
                }
                for (uint64_t k = 0; k < o->nfo; k++) {
                    double v = o->t[k] * y[o->fo[k]];
                    d[o->bi[k] * inner] += v;
                }
            }
        free(y);
    }
}

/* transform.py:229-245 _thomas_solve_axis */
static void thomas_axis(int rank, const uint64_t *csh, int a, const axop_t *o, double *arr) {
    uint64_t outer, inner;
    view(rank, csh, a, &outer, &inner);
    uint64_t n = o->nc;
    #pragma omp parallel for num_threads(g_threads) schedule(static) collapse(2)
    for (uint64_t p = 0; p < outer; p++)
        for (uint64_t q = 0; q < inner; q++) {
            double *x = arr + p * n * inner + q;
            for (uint64_t i = 1; i < n; i++) { double w = o->tw[i] * x[(i - 1) * inner]; x[i * inner] = x[i * inner] - w; }
            x[(n - 1) * inner] = x[(n - 1) * inner] / o->tb[n - 1];
            for (uint64_t i = n - 1; i-- > 0;) {
                double w = o->tu[i] * x[(i + 1) * inner];
                x[i * inner] = x[i * inner] - w;
                x[i * inner] = x[i * inner] / o->tb[i];
            }
        }
}

typedef struct {
    hier_t h;
    axop_t ops[MAXL][4];
} plan_t;

static int plan_build(plan_t *P, int rank, const uint64_t *dims) {
    int rc = hier_build(&P->h, rank, dims);
    if (rc) return rc;
    for (int s = 0; s + 1 < P->h.L; s++)
        for (int d = 0; d < rank; d++)
            axop_build(&P->ops[s][d], P->h.map[d][s], P->h.cnt[d][s], P->h.map[d][s + 1], P->h.cnt[d][s + 1]);
    return ORC_OK;
}

static void plan_free(plan_t *P) {
    for (int s = 0; s + 1 < P->h.L; s++)
        for (int d = 0; d < P->h.rank; d++) axop_free(&P->ops[s][d]);
    hier_free(&P->h);
}

/* transform.py:251-260 _correction: mass+restrict per active axis, then Thomas per active axis.
 * mc has shape fsh; the result (shape csh) is written to out. */
static void correction(plan_t *P, int s, const uint64_t *fsh, const double *mc, double *out) {
    int r = P->h.rank;
    uint64_t sh[4];
    memcpy(sh, fsh, sizeof(sh));
    double *cur = NULL;
    const double *in = mc;
    for (int a = 0; a < r; a++) {
        axop_t *o = &P->ops[s][a];
        if (!o->active) continue;
        uint64_t nsh[4];
        memcpy(nsh, sh, sizeof(nsh));
        nsh[a] = o->nc;
        double *nxt = malloc(sizeof(double) * prod(r, nsh));
        mass_restrict_axis(r, sh, a, o, in, nxt);
        free(cur);
        cur = nxt; in = nxt;
        memcpy(sh, nsh, sizeof(sh));
    }
    uint64_t n = prod(r, sh);
    if (!cur) { cur = malloc(8 * n); memcpy(cur, mc, 8 * n); }
    for (int a = 0; a < r; a++) {
        axop_t *o = &P->ops[s][a];
        if (o->active) thomas_axis(r, sh, a, o, cur);
    }
    memcpy(out, cur, 8 * n);
    free(cur);
}

/* transform.py:261-268 _interpolate; coarse has shape csh, result shape fsh */
static void interpolate(plan_t *P, int s, const uint64_t *csh, const double *coarse, double *pred) {
    int r = P->h.rank;
    uint64_t sh[4];
    memcpy(sh, csh, sizeof(sh));
    double *cur = NULL;
    const double *in = coarse;
    for (int a = 0; a < r; a++) {
        axop_t *o = &P->ops[s][a];
        if (!o->active) continue;
        uint64_t nsh[4];
        memcpy(nsh, sh, sizeof(nsh));
        nsh[a] = o->n;
        double *nxt = malloc(sizeof(double) * prod(r, nsh));
        prolong_axis(r, sh, a, o, in, nxt);
        free(cur);
        cur = nxt; in = nxt;
        memcpy(sh, nsh, sizeof(sh));
    }
    uint64_t n = prod(r, sh);
    if (!cur) memcpy(pred, coarse, 8 * n);
    else { memcpy(pred, cur, 8 * n); free(cur); }
}

static void level_shapes(plan_t *P, int s, uint64_t *fsh, uint64_t *csh,
                         const int64_t **fmap, const int64_t **cmap, const int64_t **csel, int64_t **tmp) {
    for (int d = 0; d < P->h.rank; d++) {
        fsh[d] = P->h.cnt[d][s];
        csh[d] = P->h.cnt[d][s + 1];
        fmap[d] = P->h.map[d][s];
        cmap[d] = P->h.map[d][s + 1];
        axop_t *o = &P->ops[s][d];
        tmp[d] = malloc(sizeof(int64_t) * csh[d]);
        for (uint64_t c = 0; c < csh[d]; c++) tmp[d][c] = o->active ? (int64_t)o->sel[c] : (int64_t)c;
        csel[d] = tmp[d];
    }
}

/* transform.py:287-323 decompose (work array in finest layout, like the reference) */
static int decompose_plan(plan_t *P, const void *in, int dtype, double *work, double *vmin, double *vmax) {
    int r = P->h.rank;
    uint64_t N = prod(r, P->h.dims);
    double mn = INFINITY, mx = -INFINITY;
    int has_nan = 0;
    if (dtype == ORC_F32) {
        const float *u = in;
        for (uint64_t i = 0; i < N; i++) {
            double v = (double)u[i];
            work[i] = v;
        }
    } else if (dtype == ORC_F64) {
        memcpy(work, in, 8 * N);
    } else return ORC_VALIDATION;
    /* numpy min/max propagate NaN */
    for (uint64_t i = 0; i < N; i++) {
        double v = work[i];
        if (v != v) has_nan = 1;
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    if (has_nan) { mn = NAN; mx = NAN; }
    *vmin = mn; *vmax = mx;
    for (int s = 0; s + 1 < P->h.L; s++) {
        uint64_t fsh[4], csh[4];
        const int64_t *fmap[4], *cmap[4], *csel[4];
        int64_t *tmp[4];
        level_shapes(P, s, fsh, csh, fmap, cmap, csel, tmp);
        uint64_t nf = prod(r, fsh), nc = prod(r, csh);
        double *sub = malloc(8 * nf), *coarse = malloc(8 * nc), *pred = malloc(8 * nf), *corr = malloc(8 * nc);
        gather(r, P->h.dims, work, fsh, fmap, sub);
        gather(r, fsh, sub, csh, csel, coarse);
        interpolate(P, s, csh, coarse, pred);
        #pragma omp parallel for num_threads(g_threads) schedule(static)
        for (uint64_t i = 0; i < nf; i++) sub[i] = sub[i] - pred[i];   /* mc */
        correction(P, s, fsh, sub, corr);
        scatter(r, P->h.dims, work, fsh, fmap, sub);
        #pragma omp parallel for num_threads(g_threads) schedule(static)
        for (uint64_t i = 0; i < nc; i++) coarse[i] = coarse[i] + corr[i];
        scatter(r, P->h.dims, work, csh, cmap, coarse);
        free(sub); free(coarse); free(pred); free(corr);
        for (int d = 0; d < r; d++) free(tmp[d]);
    }
    return ORC_OK;
}

int orc_decompose(const void *in, int dtype, int rank, const uint64_t *dims, double *coef, double *vmin, double *vmax) {
    plan_t *P = calloc(1, sizeof(plan_t));
    int rc = plan_build(P, rank, dims);
    if (!rc) rc = decompose_plan(P, in, dtype, coef, vmin, vmax);
    plan_free(P); free(P);
    return rc;
}

/* transform.py:326-348 recompose */
static void recompose_plan(plan_t *P, const double *coef, double *work) {
    int r = P->h.rank;
    uint64_t N = prod(r, P->h.dims);
    memcpy(work, coef, 8 * N);
    for (int s = P->h.L - 2; s >= 0; s--) {
        uint64_t fsh[4], csh[4];
        const int64_t *fmap[4], *cmap[4], *csel[4];
        int64_t *tmp[4];
        level_shapes(P, s, fsh, csh, fmap, cmap, csel, tmp);
        uint64_t nf = prod(r, fsh), nc = prod(r, csh);
        double *mc = malloc(8 * nf), *cv = malloc(8 * nc), *corr = malloc(8 * nc), *pred = malloc(8 * nf);
        double *zeros = calloc(nc, 8);
        gather(r, P->h.dims, work, fsh, fmap, mc);
        scatter(r, fsh, mc, csh, csel, zeros);                    /* mc[coarse_sel] = 0.0 */
        correction(P, s, fsh, mc, corr);
        gather(r, P->h.dims, work, csh, cmap, cv);
        #pragma omp parallel for num_threads(g_threads) schedule(static)
        for (uint64_t i = 0; i < nc; i++) cv[i] = cv[i] - corr[i];
        interpolate(P, s, csh, cv, pred);
        #pragma omp parallel for num_threads(g_threads) schedule(static)
        for (uint64_t i = 0; i < nf; i++) pred[i] = pred[i] + mc[i];
        scatter(r, P->h.dims, work, fsh, fmap, pred);
        free(mc); free(cv); free(corr); free(pred); free(zeros);
        for (int d = 0; d < r; d++) free(tmp[d]);
    }
}

int orc_recompose(const double *coef, int rank, const uint64_t *dims, double *out) {
    plan_t *P = calloc(1, sizeof(plan_t));
    int rc = plan_build(P, rank, dims);
    if (!rc) recompose_plan(P, coef, out);
    plan_free(P); free(P);
    return rc;
}

/* hierarchy.py:44-48 coarsest_flat_indices (row-major meshgrid order) */
static uint64_t coarsest_indices(const hier_t *h, uint64_t *out) {
    int r = h->rank, k = h->L - 1;
    uint64_t sub[4];
    for (int d = 0; d < r; d++) sub[d] = h->cnt[d][k];
    uint64_t n = prod(r, sub);
    if (out)
        for (uint64_t f = 0; f < n; f++) {
            uint64_t rr = f, off = 0, stride = 1;
            for (int d = r - 1; d >= 0; d--) {
                uint64_t i = rr % sub[d]; rr /= sub[d];
                off += (uint64_t)h->map[d][k][i] * stride;
                stride *= h->dims[d];
            }
            out[f] = off;
        }
    return n;
}

int orc_coarsest_indices(int rank, const uint64_t *dims, uint64_t *out, uint64_t *n) {
    hier_t h;
    int rc = hier_build(&h, rank, dims);
    if (rc) return rc;
    *n = coarsest_indices(&h, out);
    hier_free(&h);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* quantize.py:50-98 / :101-125                                              */
/* ------------------------------------------------------------------------ */
int orc_quantize(const double *coef, int rank, const uint64_t *dims, double u_min, double u_max,
                 double eb_rel, uint32_t dict_size, int has_range, double r0, double r1,
                 uint32_t *keys, uint64_t *outlier_idx, int64_t *outlier_bins, uint64_t *n_out,
                 double *coarse_vals, uint64_t *n_coarse, double *eb_abs_out, double *bin_out, int *levels) {
    if (!(0.0 < eb_rel && eb_rel < 1.0)) return ORC_VALIDATION;
    if (dict_size < 2 || dict_size > 65535) return ORC_VALIDATION;
    hier_t h;
    int rc = hier_build(&h, rank, dims);
    if (rc) return rc;
    uint64_t N = prod(rank, dims);
    for (uint64_t i = 0; i < N; i++)
        if (!isfinite(coef[i])) { hier_free(&h); return ORC_VALIDATION; }
    double vmin = has_range ? r0 : u_min, vmax = has_range ? r1 : u_max;
    double eb_abs = eb_rel * (vmax - vmin);
    double bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)h.L : 1.0;
    uint64_t nco = coarsest_indices(&h, NULL);
    uint64_t *cidx = malloc(8 * nco);
    coarsest_indices(&h, cidx);
    for (uint64_t i = 0; i < nco; i++) coarse_vals[i] = coef[cidx[i]];
    int64_t *bins = malloc(8 * N);
    double amax = 0.0;
    for (uint64_t i = 0; i < N; i++) {
        double sc = coef[i] / bin;
        double a = fabs(sc);
        if (a > amax) amax = a;
        bins[i] = (int64_t)rint(sc);
    }
    if (amax >= 4611686018427387904.0) { free(bins); free(cidx); hier_free(&h); return ORC_VALIDATION; }
    for (uint64_t i = 0; i < nco; i++) bins[cidx[i]] = 0;
    int64_t half = dict_size / 2;
    uint64_t no = 0;
    for (uint64_t i = 0; i < N; i++) {
        int64_t b = bins[i];
        if ((b < 0 ? -b : b) >= half) {
            outlier_idx[no] = i; outlier_bins[no] = b; no++;
            b = 0;
        }
        keys[i] = (uint32_t)(((uint64_t)b << 1) ^ (uint64_t)(b >> 63));
    }
    *n_out = no; *n_coarse = nco; *eb_abs_out = eb_abs; *bin_out = bin; *levels = h.L;
    free(bins); free(cidx); hier_free(&h);
    return ORC_OK;
}

int orc_dequantize(const uint32_t *keys, uint64_t nkeys, int rank, const uint64_t *dims, uint32_t dict_size,
                   double bin, const uint64_t *oidx, const int64_t *obins, uint64_t n_out,
                   const double *coarse_vals, uint64_t n_coarse, double *coef) {
    hier_t h;
    int rc = hier_build(&h, rank, dims);
    if (rc) return rc;
    uint64_t N = prod(rank, dims);
    if (nkeys != N) { hier_free(&h); return ORC_VALIDATION; }
    for (uint64_t i = 0; i < N; i++)
        if (keys[i] >= dict_size) { hier_free(&h); return ORC_VALIDATION; }
    for (uint64_t i = 0; i < N; i++) {
        uint64_t k = keys[i];
        int64_t b = (int64_t)(k >> 1) ^ -(int64_t)(k & 1);
        coef[i] = (double)b * bin;
    }
    for (uint64_t i = 0; i < n_out; i++) {
        int64_t ix = (int64_t)oidx[i];
        if (ix < 0) ix += (int64_t)N;                 /* numpy negative-index semantics */
        if (ix < 0 || (uint64_t)ix >= N) { hier_free(&h); return ORC_INDEX; }
        coef[ix] = (double)obins[i] * bin;
    }
    uint64_t nco = coarsest_indices(&h, NULL);
    uint64_t *cidx = malloc(8 * nco);
    coarsest_indices(&h, cidx);
    if (n_coarse != nco) { free(cidx); hier_free(&h); return ORC_VALIDATION; }
    for (uint64_t i = 0; i < nco; i++) coef[cidx[i]] = coarse_vals[i];
    free(cidx); hier_free(&h);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* huffman.py                                                                */
/* ------------------------------------------------------------------------ */
int orc_histogram(const uint32_t *keys, uint64_t n, uint32_t dict_size, int64_t *counts) {
    if (dict_size < 1 || dict_size > MAX_DICT) return ORC_VALIDATION;
    for (uint32_t k = 0; k < dict_size; k++) counts[k] = 0;
    for (uint64_t i = 0; i < n; i++) {
        if (keys[i] >= dict_size) return ORC_VALIDATION;
        counts[keys[i]]++;
    }
    return ORC_OK;
}

/* huffman.py:107-157, literal restatement of the in-place length computation */
static void lengths_in_place(int64_t *a, int64_t n) {
    if (n == 1) { a[0] = 1; return; }
    int64_t s = 0, r = 0;
    for (int64_t t = 0; t < n - 1; t++) {
        if (s >= n || (r < t && a[r] < a[s])) { a[t] = a[r]; a[r] = t; r++; }
        else { a[t] = a[s]; s++; }
        if (s >= n || (r < t && a[r] < a[s])) { a[t] += a[r]; a[r] = t; r++; }
        else { a[t] += a[s]; s++; }
    }
    a[n - 2] = 0;
    for (int64_t t = n - 3; t >= 0; t--) a[t] = a[a[t]] + 1;
    int64_t avail = 1, used = 0, depth = 0, t = n - 2, x = n - 1;
    while (avail > 0) {
        while (t >= 0 && a[t] == depth) { used++; t--; }
        while (avail > used) { a[x] = depth; x--; avail--; }
        avail = 2 * used; used = 0; depth++;
    }
}

static const int64_t *g_sort_counts;
static int cmp_count_key(const void *pa, const void *pb) {
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    int64_t ca = g_sort_counts[a], cb = g_sort_counts[b];
    if (ca != cb) return ca < cb ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static const uint8_t *g_sort_lens;
static int cmp_len_key(const void *pa, const void *pb) {
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    if (g_sort_lens[a] != g_sort_lens[b]) return g_sort_lens[a] < g_sort_lens[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* huffman.py:188-204; returns ORC_OVERFLOW when a code value leaves uint32 */
int orc_canonical_codes(const uint8_t *lengths, uint32_t dict_size, uint32_t *codes) {
    uint32_t *order = malloc(4 * (dict_size ? dict_size : 1));
    uint32_t np_ = 0;
    for (uint32_t k = 0; k < dict_size; k++) { codes[k] = 0; if (lengths[k]) order[np_++] = k; }
    if (np_ == 0) { free(order); return ORC_OK; }
    g_sort_lens = lengths;
    qsort(order, np_, 4, cmp_len_key);
    uint64_t code = 0;
    int prev = lengths[order[0]];
    for (uint32_t i = 0; i < np_; i++) {
        int ln = lengths[order[i]];
        int sh = ln - prev;
        if (code != 0) {
            if (sh >= 32) { free(order); return ORC_OVERFLOW; }   /* code >= 1 -> code << 32 leaves uint32 */
            code <<= sh;                                          /* code <= 2^32, sh < 32: no 64-bit wrap */
        }
        if (code >> 32) { free(order); return ORC_OVERFLOW; }     /* numpy: int out of bounds for uint32 */
        codes[order[i]] = (uint32_t)code;
        code++;
        prev = ln;
    }
    free(order);
    return ORC_OK;
}

/* huffman.py:160-185 */
int orc_build_codebook(const int64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes) {
    uint32_t *present = malloc(4 * dict_size);
    uint32_t np_ = 0;
    for (uint32_t k = 0; k < dict_size; k++) { lengths[k] = 0; codes[k] = 0; if (counts[k] > 0) present[np_++] = k; }
    if (np_ == 0) { free(present); return ORC_VALIDATION; }
    if (np_ == 1) { lengths[present[0]] = 1; free(present); return ORC_OK; }
    g_sort_counts = counts;
    qsort(present, np_, 4, cmp_count_key);     /* (count, key): stable argsort over ascending keys */
    int64_t *a = malloc(8 * np_);
    for (uint32_t i = 0; i < np_; i++) a[i] = counts[present[i]];
    lengths_in_place(a, np_);
    int64_t mx = 0;
    for (uint32_t i = 0; i < np_; i++) if (a[i] > mx) mx = a[i];
    if (mx > MAX_CODE_LEN) { free(a); free(present); return ORC_VALIDATION; }
    for (uint32_t i = 0; i < np_; i++) lengths[present[i]] = (uint8_t)a[i];
    free(a); free(present);
    return orc_canonical_codes(lengths, dict_size, codes);
}

static void put_u16(uint8_t *p, uint16_t v) { memcpy(p, &v, 2); }
static void put_u32(uint8_t *p, uint32_t v) { memcpy(p, &v, 4); }
static void put_u64(uint8_t *p, uint64_t v) { memcpy(p, &v, 8); }

/* Upper bound of the Huffman stream size for n symbols. */
uint64_t orc_huffman_bound(uint64_t n, uint32_t dict_size) {
    uint64_t units = (n + BLOCK_SYMBOLS - 1) / BLOCK_SYMBOLS;
    return 2 + 8 + dict_size + 4 + 8 * units + 8 + 4 * n + 8;
}

/* huffman.py:366-396 */
int orc_huffman_compress(const uint32_t *keys, uint64_t n, uint32_t dict_size, uint8_t *out, uint64_t cap, uint64_t *len) {
    if (dict_size < 1 || dict_size > MAX_DICT) return ORC_VALIDATION;
    int64_t *counts = malloc(8 * dict_size);
    int rc = orc_histogram(keys, n, dict_size, counts);
    if (rc) { free(counts); return rc; }
    if (cap < orc_huffman_bound(n, dict_size)) { free(counts); return ORC_VALIDATION; }
    uint64_t pos = 0;
    put_u16(out, (uint16_t)dict_size); put_u64(out + 2, n); pos = 10;
    if (n == 0) {
        memset(out + pos, 0, dict_size); pos += dict_size;
        put_u32(out + pos, 0); pos += 4; put_u64(out + pos, 0); pos += 8;
        *len = pos; free(counts); return ORC_OK;
    }
    uint8_t *lens = malloc(dict_size);
    uint32_t *codes = malloc(4 * dict_size);
    rc = orc_build_codebook(counts, dict_size, lens, codes);
    if (rc) { free(counts); free(lens); free(codes); return rc; }
    memcpy(out + pos, lens, dict_size); pos += dict_size;
    uint32_t npresent = 0;
    for (uint32_t k = 0; k < dict_size; k++) npresent += counts[k] > 0;
    if (npresent == 1) {
        put_u32(out + pos, 0); pos += 4; put_u64(out + pos, 0); pos += 8;
        *len = pos; free(counts); free(lens); free(codes); return ORC_OK;
    }
    uint64_t units = (n + BLOCK_SYMBOLS - 1) / BLOCK_SYMBOLS;
    uint64_t *ubits = malloc(8 * units);
    #pragma omp parallel for num_threads(g_threads) schedule(static)
    for (uint64_t u = 0; u < units; u++) {
        uint64_t lo = u * BLOCK_SYMBOLS, hi = lo + BLOCK_SYMBOLS < n ? lo + BLOCK_SYMBOLS : n, b = 0;
        for (uint64_t i = lo; i < hi; i++) b += lens[keys[i]];
        ubits[u] = b;
    }
    put_u32(out + pos, (uint32_t)units); pos += 4;
    uint64_t total = 0;
    for (uint64_t u = 0; u < units; u++) { put_u64(out + pos + 8 * u, total); total += ubits[u]; }
    pos += 8 * units;
    put_u64(out + pos, total); pos += 8;
    uint64_t nbytes = (total + 7) / 8;
    uint8_t *packed = out + pos;
    memset(packed, 0, nbytes);
    /* MSB-first packing (np.packbits); units are written in parallel, boundary bytes with atomics-free
       ownership: each unit writes bits into a private buffer, then merged serially at boundaries. */
    uint64_t *uoff = malloc(8 * units);
    uint64_t acc = 0;
    for (uint64_t u = 0; u < units; u++) { uoff[u] = acc; acc += ubits[u]; }
    #pragma omp parallel for num_threads(g_threads) schedule(static)
    for (uint64_t u = 0; u < units; u++) {
        uint64_t lo = u * BLOCK_SYMBOLS, hi = lo + BLOCK_SYMBOLS < n ? lo + BLOCK_SYMBOLS : n;
        uint64_t bp = uoff[u];
        uint64_t first_byte = bp >> 3, last_byte = (uoff[u] + ubits[u] + 7) >> 3;
        for (uint64_t i = lo; i < hi; i++) {
            uint32_t c = codes[keys[i]];
            int L = lens[keys[i]];
            for (int b = L - 1; b >= 0; b--, bp++) {
                if ((c >> b) & 1u) {
                    uint64_t by = bp >> 3;
                    uint8_t m = (uint8_t)(0x80u >> (bp & 7));
                    if (by == first_byte || by + 1 == last_byte) {
                        #pragma omp atomic
                        packed[by] |= m;
                    } else packed[by] |= m;
                }
            }
        }
    }
    pos += nbytes;
    *len = pos;
    free(uoff); free(ubits); free(counts); free(lens); free(codes);
    return ORC_OK;
}

/* huffman.py:292-313, bit-serial canonical walk with numba int64 (wrapping) arithmetic */
static int64_t decode_unit(const uint8_t *packed, uint64_t limit, uint64_t start, uint64_t nsym,
                           const int64_t *first_code, const int64_t *first_rank, const int64_t *cnt,
                           const uint32_t *sym, int max_len, uint32_t *out) {
    uint64_t pos = start;
    for (uint64_t i = 0; i < nsym; i++) {
        uint64_t cw = pos;
        uint64_t code = 0;
        int length = 0;
        for (;;) {
            if (pos >= limit || length >= max_len) return (int64_t)cw;
            uint64_t bit = (packed[pos >> 3] >> (7 - (pos & 7))) & 1;
            code = (code << 1) | bit;
            pos++; length++;
            int64_t idx = (int64_t)(code - (uint64_t)first_code[length]);
            if (0 <= idx && idx < cnt[length]) { out[i] = sym[first_rank[length] + idx]; break; }
        }
    }
    return -1;
}

/* huffman.py:399-435; returns keys (n written to *n_out).  bit_off gets CorruptStreamError.bit_offset. */
int orc_huffman_decompress(const uint8_t *in, uint64_t len, uint32_t *keys, uint64_t cap, uint64_t *n_out, int64_t *bit_off) {
    *bit_off = -1;
    if (len < 10) return ORC_CORRUPT;
    uint16_t dict; uint64_t n;
    memcpy(&dict, in, 2); memcpy(&n, in + 2, 8);
    uint64_t pos = 10;
    if (len < pos + dict + 4) return ORC_CORRUPT;
    const uint8_t *lens = in + pos; pos += dict;
    uint32_t units; memcpy(&units, in + pos, 4); pos += 4;
    if (len < pos + 8ull * units + 8) return ORC_CORRUPT;
    const uint8_t *offs = in + pos; pos += 8ull * units;
    uint64_t total; memcpy(&total, in + pos, 8); pos += 8;
    *n_out = n;
    if (n == 0) return ORC_OK;
    uint32_t np_ = 0, first = 0;
    int max_len = 0;
    for (uint32_t k = 0; k < dict; k++) if (lens[k]) { if (!np_) first = k; np_++; if (lens[k] > max_len) max_len = lens[k]; }
    if (np_ == 0) return ORC_CORRUPT;
    if (n > cap) return ORC_VALIDATION;
    if (units == 0 && total == 0) {
        if (np_ != 1) return ORC_CORRUPT;
        for (uint64_t i = 0; i < n; i++) keys[i] = first;
        return ORC_OK;
    }
    uint64_t pbytes = total / 8 + (total % 8 != 0);
    if (len - pos < pbytes) { *bit_off = (int64_t)((len - pos) * 8); return ORC_CORRUPT; }
    uint32_t *codes = malloc(4 * (uint64_t)(dict ? dict : 1));
    int rc = orc_canonical_codes(lens, dict, codes);
    free(codes);
    if (rc) return rc;
    uint64_t need = (n + BLOCK_SYMBOLS - 1) / BLOCK_SYMBOLS;
    if (units < need) return ORC_CORRUPT;
    /* _decode_tables huffman.py:207-225 */
    int64_t first_code[258] = {0}, first_rank[258] = {0}, cnt[258] = {0};
    uint32_t *sym = malloc(4 * np_);
    uint32_t m = 0;
    for (uint32_t k = 0; k < dict; k++) if (lens[k]) { sym[m++] = k; cnt[lens[k]]++; }
    g_sort_lens = lens;
    qsort(sym, np_, 4, cmp_len_key);
    uint64_t code = 0; int64_t rank = 0;
    for (int ln = 1; ln <= max_len; ln++) {
        if (ln > 1) code <<= 1;
        first_code[ln] = (int64_t)code; first_rank[ln] = rank;
        code += (uint64_t)cnt[ln]; rank += cnt[ln];
    }
    const uint8_t *packed = in + pos;
    int64_t *errs = malloc(8 * need);
    #pragma omp parallel for num_threads(g_threads) schedule(dynamic, 16)
    for (uint64_t u = 0; u < need; u++) {
        uint64_t lo = u * BLOCK_SYMBOLS, c = n - lo < BLOCK_SYMBOLS ? n - lo : BLOCK_SYMBOLS;
        uint64_t st; memcpy(&st, offs + 8 * u, 8);
        errs[u] = decode_unit(packed, total, st, c, first_code, first_rank, cnt, sym, max_len, keys + lo);
    }
    rc = ORC_OK;
    for (uint64_t u = 0; u < need; u++) if (errs[u] >= 0) { *bit_off = errs[u]; rc = ORC_CORRUPT; break; }
    free(errs); free(sym);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* codec.py:25-56 / :59-113 whole-blob path                                  */
/* ------------------------------------------------------------------------ */
int orc_mgard_compress(const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                       uint32_t dict_size, int has_range, double r0, double r1,
                       uint8_t **blob, uint64_t *blob_len) {
    if (dtype != ORC_F32 && dtype != ORC_F64) return ORC_VALIDATION;
    plan_t *P = calloc(1, sizeof(plan_t));
    int rc = plan_build(P, rank, dims);
    if (rc) { free(P); return rc; }
    uint64_t N = prod(rank, dims);
    double *coef = malloc(8 * N);
    double vmin, vmax;
    decompose_plan(P, in, dtype, coef, &vmin, &vmax);
    uint32_t *keys = malloc(4 * N);
    uint64_t *oidx = malloc(8 * N);
    int64_t *obins = malloc(8 * N);
    uint64_t nco = coarsest_indices(&P->h, NULL);
    double *cv = malloc(8 * nco);
    uint64_t no, nc2; double eb_abs, bin; int L;
    rc = orc_quantize(coef, rank, dims, vmin, vmax, eb_rel, dict_size, has_range, r0, r1,
                      keys, oidx, obins, &no, cv, &nc2, &eb_abs, &bin, &L);
    free(coef);
    if (rc) goto done;
    uint64_t hb = orc_huffman_bound(N, dict_size);
    uint64_t cap = 1 + 8 * rank + 49 + 8 + 16 * no + 8 + 8 * nco + hb;
    uint8_t *out = malloc(cap);
    uint64_t p = 0;
    out[p++] = (uint8_t)rank;
    for (int d = 0; d < rank; d++) { put_u64(out + p, dims[d]); p += 8; }
    out[p++] = (uint8_t)dtype;
    memcpy(out + p, &eb_rel, 8); p += 8;
    put_u32(out + p, dict_size); p += 4;
    double umin = has_range ? r0 : vmin, umax = has_range ? r1 : vmax;
    memcpy(out + p, &umin, 8); p += 8;
    memcpy(out + p, &umax, 8); p += 8;
    memcpy(out + p, &eb_abs, 8); p += 8;
    memcpy(out + p, &bin, 8); p += 8;
    put_u32(out + p, (uint32_t)L); p += 4;
    put_u64(out + p, no); p += 8;
    memcpy(out + p, oidx, 8 * no); p += 8 * no;
    memcpy(out + p, obins, 8 * no); p += 8 * no;
    put_u64(out + p, nco); p += 8;
    memcpy(out + p, cv, 8 * nco); p += 8 * nco;
    uint64_t hl;
    rc = orc_huffman_compress(keys, N, dict_size, out + p, cap - p, &hl);
    if (rc) { free(out); goto done; }
    p += hl;
    *blob = out; *blob_len = p;
done:
    free(keys); free(oidx); free(obins); free(cv);
    plan_free(P); free(P);
    return rc;
}

void orc_free(void *p) { free(p); }

/* Decompress into out (dtype from blob: F32 -> float, F64 -> double). */
int orc_mgard_decompress(const uint8_t *blob, uint64_t len, void *out, uint64_t out_cap,
                         int *dtype_out, int *rank_out, uint64_t *dims_out, int64_t *bit_off) {
    *bit_off = -1;
    uint64_t p = 0;
    if (len < 1) return ORC_CORRUPT;
    int rank = blob[0]; p = 1;
    if (len < p + 8ull * rank + 49) return ORC_CORRUPT;
    uint64_t dims[255];
    for (int d = 0; d < rank; d++) { memcpy(&dims[d], blob + p, 8); p += 8; }
    int dtype = blob[p++];
    double eb_rel, umin, umax, eb_abs, bin; uint32_t dict, L;
    memcpy(&eb_rel, blob + p, 8); p += 8;
    memcpy(&dict, blob + p, 4); p += 4;
    memcpy(&umin, blob + p, 8); p += 8;
    memcpy(&umax, blob + p, 8); p += 8;
    memcpy(&eb_abs, blob + p, 8); p += 8;
    memcpy(&bin, blob + p, 8); p += 8;
    memcpy(&L, blob + p, 4); p += 4;
    if (len < p + 8) return ORC_CORRUPT;
    uint64_t no; memcpy(&no, blob + p, 8); p += 8;
    if ((len - p) / 16 < no) return ORC_CORRUPT;
    const uint8_t *oidx = blob + p; p += 8 * no;
    const uint8_t *obins = blob + p; p += 8 * no;
    if (len < p + 8) return ORC_CORRUPT;
    uint64_t nco; memcpy(&nco, blob + p, 8); p += 8;
    if ((len - p) / 8 < nco) return ORC_CORRUPT;
    const uint8_t *cv = blob + p; p += 8 * nco;
    if (dtype > 6) return ORC_CORRUPT;
    if (rank < 1 || rank > 4) return ORC_VALIDATION;
    if (dtype != ORC_F32 && dtype != ORC_F64) return ORC_VALIDATION;   /* oracle handles float outputs only */
    uint64_t N = prod(rank, dims);
    uint64_t hn = 0;
    /* peek the symbol count to size the key buffer */
    if (len - p >= 10) memcpy(&hn, blob + p + 2, 8);
    uint32_t *keys = malloc(4 * (hn ? hn : 1));
    uint64_t nk;
    int rc = orc_huffman_decompress(blob + p, len - p, keys, hn, &nk, bit_off);
    if (rc) { free(keys); return rc; }
    plan_t *P = calloc(1, sizeof(plan_t));
    rc = plan_build(P, rank, dims);
    if (rc) { free(keys); free(P); return rc; }
    if ((uint32_t)P->h.L != L) { rc = ORC_CORRUPT; goto out; }
    if (out_cap < N * (dtype == ORC_F32 ? 4 : 8)) { rc = ORC_VALIDATION; goto out; }
    double *coef = malloc(8 * N);
    uint64_t *oi = malloc(8 * (no ? no : 1)); int64_t *ob = malloc(8 * (no ? no : 1)); double *cvv = malloc(8 * (nco ? nco : 1));
    memcpy(oi, oidx, 8 * no); memcpy(ob, obins, 8 * no); memcpy(cvv, cv, 8 * nco);
    rc = orc_dequantize(keys, nk, rank, dims, dict, bin, oi, ob, no, cvv, nco, coef);
    free(oi); free(ob); free(cvv);
    if (!rc) {
        double *work = malloc(8 * N);
        recompose_plan(P, coef, work);
        if (dtype == ORC_F32) { float *o = out; for (uint64_t i = 0; i < N; i++) o[i] = (float)work[i]; }
        else memcpy(out, work, 8 * N);
        free(work);
        *dtype_out = dtype; *rank_out = rank;
        for (int d = 0; d < rank; d++) dims_out[d] = dims[d];
    }
    free(coef);
out:
    free(keys);
    plan_free(P); free(P);
    return rc;
}
