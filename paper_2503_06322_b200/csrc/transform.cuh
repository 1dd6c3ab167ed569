// transform.cuh -- multilevel decomposition / recomposition on the device.
#pragma once

#include "context.cuh"

namespace hpdr {

// Work buffers used by one decompose / recompose (owned by the context).
struct LevelBuffers {
    double *lvl0;     // finest dense level (N)
    double *arena;    // coarser dense levels
    double *mc;       // residual of the current transition
    double *t0, *t1;  // prolong / restrict intermediates
    double *cg;       // coarse gather / corrected coarse values
};

LevelBuffers level_buffers(hpdr_ctx *ctx, DevPlan &p);

// Global min/max of the input (numpy min/max semantics: NaN propagates).
// Order-key min/max accumulator: mm = {~0, 0, 0} initially (min key, max key, NaN seen).
void minmax_accumulate(const void *d_in, int dtype, int64_t n, unsigned long long *mm, cudaStream_t s);
void minmax_from_keys(const unsigned long long *mm_host, double *vmin, double *vmax);
void minmax_device(hpdr_ctx *ctx, const void *d_in, int dtype, int64_t n, double *vmin, double *vmax,
                   cudaStream_t s);

// transform.py:287-323.  d_in: device array of dtype (0 = f32, 1 = f64).  coef: N doubles in
// finest-grid order.  Returns the coarsest dense level (<= 16 values, device).
const double *decompose_device(hpdr_ctx *ctx, DevPlan &p, const void *d_in, int dtype, double *coef,
                               cudaStream_t s);

// transform.py:326-348.  coef: N doubles.  Returns the finest dense level (device, N doubles).
double *recompose_device(hpdr_ctx *ctx, DevPlan &p, const double *coef, cudaStream_t s);

struct QuantOut;
// Fused decomposition with quantize-on-write (ranks <= 3, use_fused): keys / outlier mask /
// histogram are produced by the level kernels; returns the coarsest dense level (device).
const double *decompose_quantize(hpdr_ctx *ctx, DevPlan &p, const void *d_in, int dtype, const QuantOut &q,
                                 cudaStream_t s);

// Streamed variant for a HOST input (L > 1, use_fused): dim-0 chunks are copied on the context's
// H2D stream while the finest level's pass 1 / pass 2 run on the chunks that have landed.
// Relative mode (has_range false) stores the finest coefficients and quantizes them once the
// global min/max is complete; q.bin is set here.  Returns the coarsest dense level.
const double *decompose_quantize_streamed(hpdr_ctx *ctx, DevPlan &p, const void *host_in, int dtype, bool has_range,
                                          double range_min, double range_max, double eb_rel, QuantOut &q,
                                          double *u_min, double *u_max, cudaStream_t s);

// Recompose straight into out (device) in the blob's dtype (fused final level for ranks <= 3).
// With host_out the result also lands there: the finest level is produced in dim-0 slabs whose
// D2H on the copy stream overlaps the next slab (out is then the device staging buffer).
// T0_pre / ev_pre: the finest transition's correction, already being computed elsewhere (event
// recorded after it); otherwise it is computed here on the side stream.
// T0_pre / ev_pre: the finest transition's correction computed by the caller (streamed decode);
// t0_plane_axis_only: it holds only the plane-axis (dim-0) solve, the in-plane axes are left to the
// slab loop (thomas_plane_split).
// T1_pre / ev1_pre: the same for transition 1 (complete solve).
void recompose_into(hpdr_ctx *ctx, DevPlan &p, const double *coef, void *out, int out_dtype, cudaStream_t s,
                    void *host_out = nullptr, const double *T0_pre = nullptr, cudaEvent_t ev_pre = nullptr,
                    bool t0_plane_axis_only = false, const double *T1_pre = nullptr, cudaEvent_t ev1_pre = nullptr);
// Whether transition st_i's Thomas solves can be split into the plane-axis sweep (over the whole
// grid) and the in-plane sweeps per range of coarse planes (rank <= 3, plane axis active, not a
// one-block grid): the finest level's output slabs then only wait for their own planes.
bool thomas_plane_split(const DevPlan &p, int st_i);
// The plane-axis sweep / the in-plane sweeps of coarse planes [c_lo, c_hi) (thomas_plane_split).
void thomas_plane_axis(const DevPlan &p, int st_i, double *T, cudaStream_t s);
void thomas_in_planes(const DevPlan &p, int st_i, double *T, int c_lo, int c_hi, cudaStream_t s);
// Plane-axis forward elimination that follows the right-hand side as its coarse planes are
// produced (same rank / axis conditions as thomas_plane_split; env HPDR_NO_FWD_STREAM disables):
// thomas_plane_fwd eliminates coarse planes [c_lo, c_hi) given the planes below are done, and
// thomas_finish_fwd completes the solve -- the planes from f_done on, back substitution, then (when
// in_planes) the in-plane axes, `add_base` + x into `add_dst` on the last sweep as thomas_all does.
bool thomas_fwd_stream(const DevPlan &p, int st_i);
void thomas_plane_fwd(const DevPlan &p, int st_i, double *T, int c_lo, int c_hi, cudaStream_t s);
void thomas_finish_fwd(const DevPlan &p, int st_i, double *T, int f_done, bool in_planes, cudaStream_t s,
                       const double *add_base = nullptr, double *add_dst = nullptr);
// Elements of pass 1's output Z0 at transition st_i.
int64_t z0_elems(const DevPlan &p, int st_i);
// Thomas solves of every active axis of transition st_i's coarse grid, in place.
// All IPK solves of transition st_i on T (in place); with add_dst, the last sweep writes
// add_dst = add_base + correction instead (coarse + corr folded into the solve).
void thomas_all(const DevPlan &p, int st_i, double *T, cudaStream_t s, const double *add_base = nullptr,
                double *add_dst = nullptr);

// True when the fused level kernels serve these dims (ranks <= 3) and HPDR_GENERIC != 1.
bool use_fused(const DevPlan &p);

// codec.py:113 values.astype(dtype): cast fp64 to the blob's dtype code.
void cast_output(const double *src, void *dst, int dtype, int64_t n, cudaStream_t s);

}  // namespace hpdr
