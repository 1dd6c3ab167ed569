// fused.cuh -- fused level kernels for ranks <= 3 (padded dims (1, n0, n1, n2)).
#pragma once

#include "context.cuh"

namespace hpdr {

// Finest-grid index maps of one level (3-D view) and the finest extents of axes 1, 2.
struct LevelMap {
    const int32_t *m0, *m1, *m2;
    int64_t D1, D2;
};

bool fused_supported(const DevPlan &p);

// Decompose transition st_i: mc -> coef (fine-only nodes), coarse-node gather -> Cg, and the
// axis-0 mass-transfer -> Z0.  F is the dense fine level (float when f32).
void fused_pass1_decompose(const DevPlan &p, int st_i, const void *F, bool f32, double *coef, double *Z0,
                           double *Cg, cudaStream_t s);
// Recompose transition st_i: mc gathered from coef (coarse nodes zero) -> axis-0 mass-transfer -> Z0.
void fused_pass1_recompose(const DevPlan &p, int st_i, const double *coef, double *Z0, cudaStream_t s);
// Axis-1 and axis-2 mass-transfer: Z0 -> B (the coarse-grid right-hand side of the Thomas solves).
void fused_pass2(const DevPlan &p, int st_i, const double *Z0, double *B, cudaStream_t s);
// D = P(cv) + mc on the fine level; out_dtype 0 writes float, otherwise double.
void fused_final(const DevPlan &p, int st_i, const double *cv, const double *coef, void *D, int out_dtype,
                 cudaStream_t s);

}  // namespace hpdr
