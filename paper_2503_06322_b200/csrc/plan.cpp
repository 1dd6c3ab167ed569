// plan.cpp -- compiled with -ffp-contract=off: every + and * rounds like numpy.
#include "plan.hpp"

#include <string>

#include "error.hpp"
#include "hpdr_b200.h"

namespace hpdr {

// transform.py:67-78 _mass_tridiag: diag[:-1] += h/3 first, then diag[1:] += h/3.
static void mass_bands(const std::vector<int32_t> &x, std::vector<double> &lo, std::vector<double> &di,
                       std::vector<double> &up) {
    size_t n = x.size();
    lo.assign(n, 0.0);
    di.assign(n, 0.0);
    up.assign(n, 0.0);
    for (size_t i = 0; i + 1 < n; i++) di[i] += (double)(x[i + 1] - x[i]) / 3.0;
    for (size_t i = 0; i + 1 < n; i++) {
        double h = (double)(x[i + 1] - x[i]);
        di[i + 1] += h / 3.0;
        lo[i + 1] = h / 6.0;
        up[i] = h / 6.0;
    }
}

// transform.py:92-117 _axis_ops, re-laid out per fine node (prolong) and per coarse node (restrict)
static void axis_tables(AxisTables &a, const std::vector<int32_t> &fine, const std::vector<int32_t> &coarse) {
    const int64_t n = (int64_t)fine.size(), nc = (int64_t)coarse.size();
    a.n = n;
    a.nc = nc;
    if (n == nc) { a.active = false; return; }
    a.active = true;
    std::vector<int64_t> sel(nc);
    std::vector<char> is_sel(n, 0);
    for (int64_t c = 0; c < nc; c++) {
        sel[c] = 2 * c < n - 1 ? 2 * c : n - 1;   // hierarchy.py:92 clamp
        is_sel[sel[c]] = 1;
    }
    a.pa.assign(n, 0); a.pb.assign(n, -1); a.pt.assign(n, 0.0);
    a.r0.assign(nc, 0); a.rr.assign(nc, -1); a.rl.assign(nc, -1);
    a.wr.assign(nc, 0.0); a.wl.assign(nc, 0.0);
    for (int64_t c = 0; c < nc; c++) { a.pa[sel[c]] = (int32_t)c; a.r0[c] = (int32_t)sel[c]; }
    for (int64_t f = 0; f < n; f++) {
        if (is_sel[f]) continue;
        int64_t ai = (f - 1) / 2;
        int64_t bi = (f + 1 == n - 1) ? nc - 1 : (f + 1) / 2;
        double xa = (double)coarse[ai], xb = (double)coarse[bi], xj = (double)fine[f];
        double t = (xj - xa) / (xb - xa);
        a.pa[f] = (int32_t)ai;
        a.pb[f] = (int32_t)bi;
        a.pt[f] = t;
        // restrict (transform.py:181-203): dst[ai] += (1-t)*y[f] (first), dst[bi] += t*y[f] (second)
        a.rr[ai] = (int32_t)f;
        a.wr[ai] = 1.0 - t;
        a.rl[bi] = (int32_t)f;
        a.wl[bi] = t;
    }
    a.fa.assign(n, 0);
    a.fb.assign(n, 0);
    for (int64_t f = 0; f < n; f++) {
        a.fa[f] = a.r0[a.pa[f]];
        a.fb[f] = a.pb[f] >= 0 ? a.r0[a.pb[f]] : a.fa[f];
    }
    mass_bands(fine, a.ml, a.md, a.mu);
    std::vector<double> cl, cd;
    mass_bands(coarse, cl, cd, a.tu);
    // transform.py:81-89 _thomas_factors
    a.tw.assign(nc, 0.0);
    a.tb = cd;
    for (int64_t i = 1; i < nc; i++) {
        a.tw[i] = cl[i] / a.tb[i - 1];
        a.tb[i] = cd[i] - a.tw[i] * a.tu[i - 1];
    }
    a.tr.resize(nc);
    for (int64_t i = 0; i < nc; i++) a.tr[i] = 1.0 / a.tb[i];
    a.pinfo.assign(n, PlaneInfo{});
    for (int64_t j = 0; j < n; j++) {
        PlaneInfo &p = a.pinfo[j];
        p.fo = a.pb[j] >= 0;
        p.ca = a.pa[j];
        p.cb = p.fo ? a.pb[j] : a.pa[j];
        p.fa = a.fa[j];
        p.fb = a.fb[j];
        p.t = a.pt[j];
        p.md = a.md[j];
        p.ml = a.ml[j];
        p.mu = a.mu[j];
        p.emit = -1;
    }
    for (int64_t c = 0; c < nc; c++) {
        const int64_t need = a.rr[c] >= 0 ? a.rr[c] : a.r0[c];
        PlaneInfo &p = a.pinfo[need];
        p.emit = (int32_t)c;
        p.e_rr = a.rr[c] >= 0;
        p.e_rl = a.rl[c] >= 0;
        p.ewr = a.wr[c];
        p.ewl = a.wl[c];
    }
}

void build_host_plan(HostPlan &p, int rank, const uint64_t *dims) {
    if (rank < 1 || rank > 4) throw Error{HPDR_ERR_VALIDATION, "rank must be 1..4", -1};
    p.rank = rank;
    for (int d = 0; d < 4; d++) p.dims[d] = 1;
    for (int d = 0; d < rank; d++) {
        if (dims[d] < 1) throw Error{HPDR_ERR_VALIDATION, "extents must be >= 1", -1};
        if (dims[d] > 0x7fffffffULL) throw Error{HPDR_ERR_VALIDATION, "extent exceeds 2^31-1", -1};
        p.dims[4 - rank + d] = (int64_t)dims[d];
    }
    int nco = 0;
    for (int d = 0; d < 4; d++) {
        int64_t n = p.dims[d];
        int steps = 0;
        while (n > 2) { n = n / 2 + 1; steps++; }
        if (steps > nco) nco = steps;
    }
    p.L = nco + 1;
    for (int d = 0; d < 4; d++) {
        const int64_t D = p.dims[d];
        p.cnt[d].assign(1, D);
        p.map[d].assign(1, std::vector<int32_t>(D));
        for (int64_t i = 0; i < D; i++) p.map[d][0][i] = (int32_t)i;
        for (int k = 1; k <= nco; k++) {
            int64_t n = p.cnt[d][k - 1];
            if ((n <= 2 && D >= 2) || D == 1) {   // hierarchy.py:83-90
                p.cnt[d].push_back(n);
                p.map[d].push_back(p.map[d][k - 1]);
                continue;
            }
            int64_t nc = n / 2 + 1;
            std::vector<int32_t> m(nc);
            for (int64_t i = 0; i < nc; i++) m[i] = p.map[d][k - 1][2 * i < n - 1 ? 2 * i : n - 1];
            p.cnt[d].push_back(nc);
            p.map[d].push_back(m);
        }
    }
    p.steps.assign(p.L - 1, StepTables());
    for (int s = 0; s + 1 < p.L; s++) {
        StepTables &st = p.steps[s];
        for (int d = 0; d < 4; d++) {
            st.fsh[d] = p.cnt[d][s];
            st.csh[d] = p.cnt[d][s + 1];
            axis_tables(st.ax[d], p.map[d][s], p.map[d][s + 1]);
        }
    }
    // hierarchy.py:44-48 coarsest_flat_indices, row-major over the coarsest maps
    const int k = p.L - 1;
    p.coarsest.clear();
    for (int64_t a = 0; a < p.cnt[0][k]; a++)
        for (int64_t b = 0; b < p.cnt[1][k]; b++)
            for (int64_t c = 0; c < p.cnt[2][k]; c++)
                for (int64_t e = 0; e < p.cnt[3][k]; e++) {
                    int64_t f = (((int64_t)p.map[0][k][a] * p.dims[1] + p.map[1][k][b]) * p.dims[2] +
                                 p.map[2][k][c]) * p.dims[3] + p.map[3][k][e];
                    p.coarsest.push_back(f);
                }
}

}  // namespace hpdr
