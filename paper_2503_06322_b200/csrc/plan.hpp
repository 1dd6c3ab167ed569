// plan.hpp -- host-side multilevel hierarchy and per-(transition, axis) operator tables.
//
// Restates hpdr/mgard/hierarchy.py:63-97 (build_hierarchy) and
// hpdr/mgard/transform.py:45-128 (AxisOps/_mass_tridiag/_thomas_factors/_axis_ops)
// with the same IEEE operation order (compiled with -ffp-contract=off), and lays the
// tables out for the device kernels.
#pragma once

#include <stdint.h>

#include <vector>

namespace hpdr {

// Everything a march along one axis needs at fine index j, in one 80-byte record (built on the
// host so the device loop does one broadcast load per plane instead of a dependent chain).
struct PlaneInfo {
    int32_t fa, fb, ca, cb;   // fine / coarse indices of the coarse neighbours (= j / c at coarse nodes)
    double t;                 // interpolation weight (0 at coarse nodes)
    double md, ml, mu;        // fine mass bands at j
    int32_t fo;               // 1 when j is a fine-only node
    int32_t emit;             // coarse c whose restriction completes once y(j) is known, else -1
    int32_t e_rr, e_rl;       // c has a right (1 - t_R) / left (t_L) fine-only contribution
    double ewr, ewl;          // those weights
};
static_assert(sizeof(PlaneInfo) == 80, "PlaneInfo layout");

struct AxisTables {
    std::vector<PlaneInfo> pinfo;   // per fine node
    bool active = false;
    int64_t n = 1, nc = 1;
    // prolong (GPK), per fine node j: pa/pb coarse neighbours (pb < 0: copy of coarse pa), t weight
    std::vector<int32_t> pa, pb;
    std::vector<double> pt;
    std::vector<int32_t> fa, fb;   // fine indices of those coarse neighbours (fa = fb = j at coarse nodes)
    // mass-transfer (LPK), per coarse node c: own fine index r0, right/left fine-only
    // neighbours rr/rl (-1 when absent), weights wr = 1 - t_R and wl = t_L
    std::vector<int32_t> r0, rr, rl;
    std::vector<double> wr, wl;
    // fine mass bands, per fine node
    std::vector<double> ml, md, mu;
    // coarse-mass Thomas factors (w, b', upper), per coarse node
    std::vector<double> tw, tb, tu;
    std::vector<double> tr;   // RN(1 / b'): seed of the verified fast division in the Thomas sweeps
};

struct StepTables {
    int64_t fsh[4], csh[4];     // level shapes (padded 4-D) before / after this transition
    AxisTables ax[4];
};

struct HostPlan {
    int rank = 0;               // caller's rank (1..4)
    int L = 1;                  // total_levels
    int64_t dims[4];            // padded 4-D dims
    std::vector<int64_t> cnt[4];               // cnt[d][k]
    std::vector<std::vector<int32_t>> map[4];  // map[d][k][i]: finest index
    std::vector<StepTables> steps;             // steps[s], s = 0 is finest -> next
    std::vector<int64_t> coarsest;             // flat indices of coarsest nodes (<= 16)
    int64_t total() const { return dims[0] * dims[1] * dims[2] * dims[3]; }
};

// Throws hpdr::Error(HPDR_ERR_VALIDATION) for bad dims.
void build_host_plan(HostPlan &p, int rank, const uint64_t *dims);

}  // namespace hpdr
