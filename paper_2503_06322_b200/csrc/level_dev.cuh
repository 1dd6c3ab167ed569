// level_dev.cuh -- device helpers shared by the fused level kernels (fused.cu, quad.cu):
// separately rounded fp64 arithmetic in the reference's operation order, the quantize-on-write
// node (quantize.py:73-84), per-axis neighbour records and the slab split of a march.
#pragma once

#include "fused.cuh"

namespace hpdr {
namespace lvl {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double lerp(double va, double vb, double t) { return dadd(va, dmul(t, dsub(vb, va))); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Verified fast IEEE division for the back substitution.  q1 = q0 + (a - b q0) r with
// r = RN(1/b) (host table) is accepted only when its exact residual a - b q1 (an FMA) proves
// |a/b - q1| < half the smaller gap next to q1, i.e. q1 == RN(a/b) = __ddiv_rn(a, b); anything
// else (ties, subnormal / huge / non-finite values) raises `bad` and the caller redoes the line
// with __ddiv_rn.  Zeros take a * r, which carries the IEEE sign of a / b.
__device__ __forceinline__ double div_fast(double a, double b, double r, bool &bad) {
    if (a == 0.0) return __dmul_rn(a, r);
    const double q0 = __dmul_rn(a, r);
    const double q1 = __fma_rn(__fma_rn(-q0, b, a), r, q0);
    const double rem = __fma_rn(-q1, b, a);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(q1);
    const int ex = (int)((bits >> 52) & 0x7ff);
    const int mant0 = (bits & 0xfffffffffffffULL) == 0;
    // h = 2^(E - 53) (2^(E - 54) at a power of two), E the unbiased exponent of q1
    const double h = __longlong_as_double((long long)(ex - 53 - mant0) << 52);
    const double bound = fabs(b) * h;   // exact: power-of-two scaling of a normal value
    bad |= !(ex > 120 && ex < 1900) || !(bound > 1e-290) || !(fabs(rem) < bound);
    return q1;
}



// Histogram count of `key` (shared-memory bins flushed once per block).
// (__match_any_sync aggregation measured slower here: 2.67 vs 1.73 ms for the level-0 pass)
__device__ __forceinline__ void hist_add(uint32_t *sh, unsigned long long *g, bool sh_ok, uint32_t key) {
    if (sh_ok) atomicAdd(&sh[key], 1u);
    else atomicAdd(&g[key], 1ULL);
}

// The bin width: a launch parameter, or read from device memory (CUDA-graph replays).
__device__ __forceinline__ double qbin(const QuantOut &q) { return q.bin_dev ? *q.bin_dev : q.bin; }

// One fine node's quantization (quantize.py:73-84), in the double domain.  r = rint(mc / bin)
// (IEEE division, half to even) is computed with one multiply by rb = RN(1/bin): the correctly
// rounded quotient q and qa = RN(mc * rb) differ by < |q| 2^-51, so rint(qa) == rint(q) unless qa
// lies within that distance of a half-integer -- then (and for |qa| >= 2^61) the IEEE division
// decides; |mc / bin| >= 2^62 is the bin overflow.  Outlier iff |r| >= dict/2, key = zigzag(r)
// (exact: non-outlier |r| < 2^15), histogram.
__device__ __forceinline__ uint32_t quant_key(double mc, const QuantOut &q, double rbin, int64_t f, int &fl) {
    // a non-finite mc makes qa, r and dist NaN / inf, so it always takes the checked path
    const double qa = dmul(mc, rbin);
    double r = rint(qa);
    const double dist = 0.5 - fabs(dsub(qa, r));
    if (!(dist > fabs(qa) * 0x1p-49 && fabs(qa) < 0x1p61)) {
        if (!isfinite(mc)) {
            fl |= 1;
            r = 0.0;
        } else {
            const double sc = mc / qbin(q);
            if (fabs(sc) >= 4611686018427387904.0) {
                fl |= 2;
                r = 0.0;
            } else {
                r = rint(sc);
            }
        }
    }
    uint32_t key = 0;
    if (fabs(r) >= (double)q.half) {   // outlier (:80-83)
        q.obins[f] = (long long)r;
        atomicOr(&q.omask[f >> 5], 1u << (f & 31));
    } else {
        const int ri = (int)r;   // exact: |r| < 2^15
        key = ((uint32_t)ri << 1) ^ (uint32_t)(ri >> 31);   // zigzag (quantize.py:24-31)
    }
    q.keys[f] = (uint16_t)key;
    return key;
}

// quant_key plus the histogram count of the key.
__device__ __forceinline__ void quant_node(double mc, const QuantOut &q, double rbin, int64_t f, int &fl,
                                           uint32_t *sh_hist, bool sh_ok) {
    hist_add(sh_hist, q.hist, sh_ok, quant_key(mc, q, rbin, f, fl));
}

// Per-thread description of one axis at a fine index j: coarse neighbours (fine indices fa/fb,
// coarse indices ca/cb), weight t and whether j is a fine-only node along this axis.
struct Nb {
    int fa, fb, ca, cb;
    double t;
    bool fo;
};

template <bool A>
__device__ __forceinline__ Nb neighbours(const DevAxis &ax, int j) {
    Nb r;
    if (!A) {
        r.fa = r.fb = r.ca = r.cb = j;
        r.t = 0.0;
        r.fo = false;
        return r;
    }
    const int b = __ldg(ax.pb + j);
    r.fo = b >= 0;
    r.ca = __ldg(ax.pa + j);
    r.cb = r.fo ? b : r.ca;
    r.fa = __ldg(ax.fa + j);
    r.fb = __ldg(ax.fb + j);
    r.t = r.fo ? __ldg(ax.pt + j) : 0.0;
    return r;
}

__device__ __forceinline__ void slab_range(int nc, int nz, int z, int &lo, int &hi) {
    const int base = nc / nz, rem = nc % nz;
    lo = z * base + min(z, rem);
    hi = lo + base + (z < rem ? 1 : 0);
}

// Fine-plane range a slab of coarse outputs [c_lo, c_hi) marches over / owns.
template <bool A0>
__device__ __forceinline__ void slab_planes(const DevAxis &ax0, int n0, int nc0, int c_lo, int c_hi, int &j_start,
                                            int &j_end, int &own_lo, int &own_hi) {
    if (A0) {
        j_start = max(0, __ldg(ax0.r0 + c_lo) - 2);
        j_end = min(n0 - 1, __ldg(ax0.r0 + c_hi - 1) + 2);
        own_lo = c_lo == 0 ? 0 : __ldg(ax0.r0 + c_lo);
        own_hi = c_hi == nc0 ? n0 : __ldg(ax0.r0 + c_hi);
    } else {
        j_start = own_lo = c_lo;
        j_end = c_hi - 1;
        own_hi = c_hi;
    }
}

}  // namespace lvl
}  // namespace hpdr
