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

// Quantize-on-write targets (quantize.py:63-84 applied as each coefficient is finalised).
struct QuantOut {
    double bin;
    const double *bin_dev = nullptr;   // when set, the bin width is read here (graph replays)
    long long half;
    uint32_t dict;
    uint16_t *keys;               // N keys, finest order (16 bits: dict_size <= 65535, quantize.py:61)
    uint32_t *omask;              // N/32 words: outlier flags (zeroed by the caller)
    long long *obins;             // N slots, written only at outliers
    unsigned long long *hist;     // dict counts (zeroed by the caller)
    int *flags;                   // bit0 non-finite, bit1 |c/bin| >= 2^62
};

// quad.cu: pass 1 with one 2 x 2 node quad per thread (regular all-active 3-D transitions).
bool quad_eligible(const DevPlan &p, int st_i);
// quad.cu: the recompose output of a regular all-active transition, one 2 x 2 node quad per thread.
template <typename TOut>
void launch_final_quad(const double *cv, const double *corr, int n0, int n1, int n2, const DevAxis &a0,
                       const DevAxis &a1, const DevAxis &a2, const LevelMap &lm, const double *coef, TOut *D, int j_base,
                       int j_count, cudaStream_t s);
template <int MODE, typename TIn>
void launch_pass1_quad(const TIn *F, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1, const DevAxis &a2,
                       const LevelMap &lm, double *coef, double *Z0, double *Cg, const QuantOut &q, int c_base,
                       int c_count, cudaStream_t s);

// Decompose transition st_i writing keys instead of fp64 coefficients.
void fused_pass1_quantize(const DevPlan &p, int st_i, const void *F, bool f32, const QuantOut &q, double *Z0,
                          double *Cg, cudaStream_t s, int c_lo = 0, int c_hi = -1);
// Fine-only nodes of the finest level quantized from fp64 coefficients (streamed relative mode).
void quantize_fine(const DevPlan &p, const double *coef, const QuantOut &q, cudaStream_t s);
// Coarsest nodes (quantize.py:64-77): bin-limit / finiteness checks, key 0, histogram.
void quantize_coarsest(const DevPlan &p, const double *coarsest_vals, const QuantOut &q, cudaStream_t s);

// Decompose transition st_i: mc -> coef (fine-only nodes), coarse-node gather -> Cg, and the
// axis-0 mass-transfer -> Z0.  F is the dense fine level (float when f32).
void fused_pass1_decompose(const DevPlan &p, int st_i, const void *F, bool f32, double *coef, double *Z0,
                           double *Cg, cudaStream_t s, int c_lo = 0, int c_hi = -1);
// Recompose transition st_i: mc gathered from coef (coarse nodes zero) -> axis-0 mass-transfer -> Z0.
void fused_pass1_recompose(const DevPlan &p, int st_i, const double *coef, double *Z0, cudaStream_t s, int c_lo = 0,
                           int c_hi = -1);
// Axis-1 and axis-2 mass-transfer: Z0 -> B (the coarse-grid right-hand side of the Thomas solves).
void fused_pass2(const DevPlan &p, int st_i, const double *Z0, double *B, cudaStream_t s, int p_lo = 0,
                 int p_hi = -1);
// Output planes of pass 1 along axis 0 (coarse count, or the fine count when axis 0 is inactive).
int fused_out_planes(const DevPlan &p, int st_i);
// D = P(cv) + mc on the fine level; out_dtype 0 writes float, otherwise double.  With corr the coarse
// values are cv - corr (transform.py:345, coarse - correction), formed as they are read.
void fused_final(const DevPlan &p, int st_i, const double *cv, const double *coef, void *D, int out_dtype,
                 cudaStream_t s, int j_lo = 0, int j_hi = -1, const double *corr = nullptr);

// tiny.cu: every transition from the first one whose fine level fits one block (>= st_min; -1 none)
// run in one kernel, levels resident in shared memory.
int tiny_start(const DevPlan &p, int st_min);
// Quantizing decomposition of transitions st_a .. L-2 from the dense level F0; the coarsest level to
// DL, quantized raw (replaces per-level pass 1 / pass 2 / Thomas and quantize_coarsest).
void tiny_decompose_quantize(const DevPlan &p, int st_a, const double *F0, double *DL, const QuantOut &q,
                             cudaStream_t s);
// Recomposition of transitions L-2 .. st_a from the coefficient set; level st_a's dense values to D.
void tiny_recompose(const DevPlan &p, int st_a, const double *coef, double *D, cudaStream_t s);

}  // namespace hpdr
