// transform.cu -- per-axis multilevel kernels (GPK prolong, LPK mass-transfer, IPK Thomas)
// and the level drivers for decompose / recompose.
//
// Bit-exactness: every operation uses the reference's association order with explicit
// round-to-nearest intrinsics (no FMA contraction; the library is also built with
// -fmad=false).  See SURVEY Appendix B and transform.py:158-245.
#include "transform.cuh"

#include <stdlib.h>

#include "fused.cuh"
#include "level_dev.cuh"

namespace hpdr {

namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
using lvl::ddiv;

// ---------------------------------------------------------------- input conversion / range
__global__ void k_to_f64(const void *__restrict__ in, int dtype, double *__restrict__ out, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (dtype == 0) {
        const float *f = (const float *)in;
        for (; i < n; i += stride) out[i] = (double)f[i];
    } else {
        const double *f = (const double *)in;
        for (; i < n; i += stride) out[i] = f[i];
    }
}

// Order-preserving integer key of a double (-0 < +0; NaNs are tracked separately).
__device__ __forceinline__ unsigned long long ord_key(double v) {
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}

__global__ void k_minmax(const void *__restrict__ in, int dtype, int64_t n, unsigned long long *res) {
    unsigned long long mn = ~0ULL, mx = 0ULL;
    int nan = 0;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto fold = [&](double v) {
        if (v != v) {
            nan = 1;
            return;
        }
        const unsigned long long k = ord_key(v);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    };
    // fp32, 16-byte aligned: 32-bit order keys (the same total order as the fp64 keys: float ->
    // double is monotone, -0 < +0), the NaN test as a max over |bits|; 4 x 16 B loads in flight
    if (dtype == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
        const uint4 *v4 = reinterpret_cast<const uint4 *>(in);
        const int64_t n4 = n / 4;
        int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        uint32_t kmn = ~0u, kmx = 0u, amax = 0u;
        auto f32 = [&](uint32_t b) {
            const uint32_t k = b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
            kmn = min(kmn, k);
            kmx = max(kmx, k);
            amax = max(amax, b & 0x7fffffffu);
        };
        for (; j + 3 * stride < n4; j += 4 * stride) {
            uint4 w[4];
#pragma unroll
            for (int k = 0; k < 4; k++) w[k] = __ldg(v4 + j + k * stride);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                f32(w[k].x);
                f32(w[k].y);
                f32(w[k].z);
                f32(w[k].w);
            }
        }
        for (; j < n4; j += stride) {
            const uint4 w = __ldg(v4 + j);
            f32(w.x);
            f32(w.y);
            f32(w.z);
            f32(w.w);
        }
        if (amax > 0x7f800000u) nan = 1;
        if (kmn != ~0u) {   // back to the fp64 keys via the float values
            const uint32_t bmn = (kmn >> 31) ? (kmn & 0x7fffffffu) : ~kmn, bmx = (kmx >> 31) ? (kmx & 0x7fffffffu) : ~kmx;
            if (!(amax > 0x7f800000u)) {
                fold((double)__uint_as_float(bmn));
                fold((double)__uint_as_float(bmx));
            }
        }
        i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // scalar tail below
    }
    // 8 independent loads in flight per thread (the streamed chunks are small: latency-bound otherwise)
    constexpr int U = 8;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        double v[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            v[k] = dtype == 0 ? (double)__ldg((const float *)in + i + k * stride) : __ldg((const double *)in + i + k * stride);
#pragma unroll
        for (int k = 0; k < U; k++) fold(v[k]);
    }
    for (; i < n; i += stride) fold(dtype == 0 ? (double)((const float *)in)[i] : ((const double *)in)[i]);
    for (int o = 16; o; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
        nan |= __shfl_xor_sync(0xffffffffu, nan, o);
    }
    __shared__ unsigned long long smn[32], smx[32];
    __shared__ int snan[32];
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { smn[w] = mn; smx[w] = mx; snan[w] = nan; }
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        mn = l < nw ? smn[l] : ~0ULL;
        mx = l < nw ? smx[l] : 0ULL;
        nan = l < nw ? snan[l] : 0;
        for (int o = 16; o; o >>= 1) {
            unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
        }
        if (l == 0) {
            atomicMin(&res[0], mn);
            atomicMax(&res[1], mx);
            if (nan) atomicOr(&res[2], 1ULL);
        }
    }
}

// ---------------------------------------------------------------- level gathers / scatters
// Iterate rows (i0, i1, i2) of a dense 4-D shape; threads cover i3.
#define FOR_ROWS(SH)                                                                       \
    const int64_t rows_ = (SH).n[0] * (SH).n[1] * (SH).n[2];                               \
    for (int64_t r_ = blockIdx.y; r_ < rows_; r_ += gridDim.y)                             \
        for (int64_t i3 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i3 < (SH).n[3];  \
             i3 += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ void row_coords(int64_t r, const Shape4 &s, int64_t &i0, int64_t &i1, int64_t &i2) {
    i2 = r % s.n[2];
    int64_t t = r / s.n[2];
    i1 = t % s.n[1];
    i0 = t / s.n[1];
}

struct Sel4 { const int32_t *s[4]; };   // per-axis index lists (nullptr: identity / all)

// dst(csh)[c] = src(fsh)[sel(c)]  -- the coarse selector of transform.py:265-272
__global__ void k_gather_coarse(const double *__restrict__ src, Shape4 fsh, double *__restrict__ dst, Shape4 csh,
                                Sel4 sel) {
    FOR_ROWS(csh) {
        int64_t c0, c1, c2;
        row_coords(r_, csh, c0, c1, c2);
        int64_t j0 = sel.s[0] ? sel.s[0][c0] : c0, j1 = sel.s[1] ? sel.s[1][c1] : c1;
        int64_t j2 = sel.s[2] ? sel.s[2][c2] : c2, j3 = sel.s[3] ? sel.s[3][i3] : i3;
        dst[r_ * csh.n[3] + i3] = src[((j0 * fsh.n[1] + j1) * fsh.n[2] + j2) * fsh.n[3] + j3];
    }
}

__device__ __forceinline__ bool is_coarse(const Sel4 &pb, int64_t i0, int64_t i1, int64_t i2, int64_t i3) {
    return (!pb.s[0] || pb.s[0][i0] < 0) && (!pb.s[1] || pb.s[1][i1] < 0) && (!pb.s[2] || pb.s[2][i2] < 0) &&
           (!pb.s[3] || pb.s[3][i3] < 0);
}

// coef[map(i)] = src[i] for the level's nodes (fine_only: skip nodes that survive to the
// next level; they are overwritten later exactly as in transform.py:314-315)
__global__ void k_scatter_level(const double *__restrict__ src, Shape4 sh, double *__restrict__ coef, Shape4 dims,
                                Sel4 map, Sel4 pb, int fine_only) {
    FOR_ROWS(sh) {
        int64_t i0, i1, i2;
        row_coords(r_, sh, i0, i1, i2);
        if (fine_only && is_coarse(pb, i0, i1, i2, i3)) continue;
        int64_t f = (((int64_t)map.s[0][i0] * dims.n[1] + map.s[1][i1]) * dims.n[2] + map.s[2][i2]) * dims.n[3] +
                    map.s[3][i3];
        coef[f] = src[r_ * sh.n[3] + i3];
    }
}

// dst[i] = coef[map(i)], zeroed at nodes of the next-coarser level (transform.py:339-343)
__global__ void k_gather_level(const double *__restrict__ coef, Shape4 dims, Sel4 map, Sel4 pb, double *__restrict__ dst,
                               Shape4 sh, int zero_coarse) {
    FOR_ROWS(sh) {
        int64_t i0, i1, i2;
        row_coords(r_, sh, i0, i1, i2);
        double v;
        if (zero_coarse && is_coarse(pb, i0, i1, i2, i3)) {
            v = 0.0;
        } else {
            int64_t f = (((int64_t)map.s[0][i0] * dims.n[1] + map.s[1][i1]) * dims.n[2] + map.s[2][i2]) *
                            dims.n[3] + map.s[3][i3];
            v = coef[f];
        }
        dst[r_ * sh.n[3] + i3] = v;
    }
}

// ---------------------------------------------------------------- GPK: prolongation along one axis
// MODE 0: dst = pred;  MODE 1: dst = aux - pred (decompose residual, transform.py:312);
// MODE 2: dst = pred + aux (recompose, transform.py:347)
template <int MODE, typename IT>
__global__ void k_prolong(const double *__restrict__ src, double *__restrict__ dst, const double *__restrict__ aux,
                          int64_t outer, int32_t nc, int32_t n, int64_t inner, const int32_t *__restrict__ pa,
                          const int32_t *__restrict__ pb, const double *__restrict__ pt) {
    const IT in_ = (IT)inner;
    const IT per = (IT)n * in_;
    for (int64_t p = blockIdx.y; p < outer; p += gridDim.y) {
        const double *s = src + p * (int64_t)nc * inner;
        double *d = dst + p * (int64_t)n * inner;
        const double *x = MODE ? aux + p * (int64_t)n * inner : nullptr;
        for (IT e = blockIdx.x * (IT)blockDim.x + threadIdx.x; e < per; e += (IT)gridDim.x * blockDim.x) {
            IT j = e / in_;
            IT q = e - j * in_;
            int a = pa[j], b = pb[j];
            double va = s[(IT)a * in_ + q];
            double v = va;
            if (b >= 0) {
                double vb = s[(IT)b * in_ + q];
                v = dadd(va, dmul(pt[j], dsub(vb, va)));
            }
            if (MODE == 1) v = dsub(x[e], v);
            if (MODE == 2) v = dadd(v, x[e]);
            d[e] = v;
        }
    }
}

// ---------------------------------------------------------------- LPK: mass multiply + restriction
template <typename IT>
__device__ __forceinline__ double mass_y(const double *__restrict__ x, IT in_, int j, int n,
                                         const double *__restrict__ ml, const double *__restrict__ md,
                                         const double *__restrict__ mu) {
    double v = dmul(md[j], x[(IT)j * in_]);
    if (j >= 1) v = dadd(v, dmul(ml[j], x[(IT)(j - 1) * in_]));
    if (j + 1 < n) v = dadd(v, dmul(mu[j], x[(IT)(j + 1) * in_]));
    return v;
}

template <typename IT>
__global__ void k_mass_restrict(const double *__restrict__ src, double *__restrict__ dst, int64_t outer, int32_t n,
                                int32_t nc, int64_t inner, DevAxis ax) {
    const IT in_ = (IT)inner;
    const IT per = (IT)nc * in_;
    for (int64_t p = blockIdx.y; p < outer; p += gridDim.y) {
        const double *s = src + p * (int64_t)n * inner;
        double *d = dst + p * (int64_t)nc * inner;
        for (IT e = blockIdx.x * (IT)blockDim.x + threadIdx.x; e < per; e += (IT)gridDim.x * blockDim.x) {
            IT c = e / in_;
            IT q = e - c * in_;
            const double *x = s + q;
            double v = mass_y<IT>(x, in_, ax.r0[c], n, ax.ml, ax.md, ax.mu);
            int r = ax.rr[c];
            if (r >= 0) v = dadd(v, dmul(ax.wr[c], mass_y<IT>(x, in_, r, n, ax.ml, ax.md, ax.mu)));
            int l = ax.rl[c];
            if (l >= 0) v = dadd(v, dmul(ax.wl[c], mass_y<IT>(x, in_, l, n, ax.ml, ax.md, ax.mu)));
            d[e] = v;
        }
    }
}

// div_fast: the verified fast IEEE division of the back substitution (level_dev.cuh).
using lvl::div_fast;

// ---------------------------------------------------------------- IPK: batched Thomas solves
// Optional epilogue of the last sweep of a correction solve: instead of the correction x itself, write
// dst = base + x (decompose: coarse + corr, transform.py:317) -- the elementwise k_add folded into
// the solve (the correction buffer then holds intermediate values only).
struct Epi {
    const double *base = nullptr;
    double *dst = nullptr;
};
template <bool EPI>
__device__ __forceinline__ void epi_store(double *arr, int64_t i, double v, const Epi &e) {
    if (EPI) e.dst[i] = dadd(__ldg(e.base + i), v);
    else arr[i] = v;
}

// Strided axis: one thread per line, threads along the contiguous inner index (coalesced).
template <bool EPI>
__global__ void k_thomas_strided(double *__restrict__ arr, int64_t outer, int32_t n, int64_t inner,
                                 const double *__restrict__ tw, const double *__restrict__ tb,
                                 const double *__restrict__ tu, Epi epi) {
    const int64_t lines = outer * inner;
    for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < lines; ln += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = ln / inner, q = ln - p * inner;
        double *x = arr + p * (int64_t)n * inner + q;
        double prev = x[0];
        for (int i = 1; i < n; i++) {
            double v = dsub(x[(int64_t)i * inner], dmul(tw[i], prev));
            x[(int64_t)i * inner] = v;
            prev = v;
        }
        double last = ddiv(prev, tb[n - 1]);
        const int64_t o = x - arr;
        epi_store<EPI>(arr, o + (int64_t)(n - 1) * inner, last, epi);
        for (int i = n - 2; i >= 0; i--) {
            double v = dsub(x[(int64_t)i * inner], dmul(tu[i], last));
            v = ddiv(v, tb[i]);
            epi_store<EPI>(arr, o + (int64_t)i * inner, v, epi);
            last = v;
        }
    }
}

// Contiguous axis: each warp owns 32 lines and walks them in 32x32 shared-memory tiles,
// loading and storing tile rows coalesced and running one line per lane.
constexpr int kThomasWarps = 4;
template <bool EPI>
__global__ void __launch_bounds__(kThomasWarps * 32) k_thomas_contig(double *__restrict__ arr, int64_t lines, int32_t n,
                                                                     const double *__restrict__ tw,
                                                                     const double *__restrict__ tb,
                                                                     const double *__restrict__ tu,
                                                                     const double *__restrict__ tr, Epi epi) {
    __shared__ double tile[kThomasWarps][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double (*T)[33] = tile[w];
    for (int64_t base = ((int64_t)blockIdx.x * kThomasWarps + w) * 32; base < lines;
         base += (int64_t)gridDim.x * kThomasWarps * 32) {
        const int nl = (int)min64(32, lines - base);
        double prev = 0.0;
        for (int t0 = 0; t0 < n; t0 += 32) {
            const int m = min(32, n - t0);
            // tile rows land by cp.async: all 32 row segments in flight at once
            if (lane < m)
                for (int r = 0; r < nl; r++) cp_async<8>(&T[r][lane], arr + (base + r) * n + t0 + lane);
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
            if (lane < nl) {
                for (int k = 0; k < m; k++) {
                    const int i = t0 + k;
                    double v = T[lane][k];
                    if (i > 0) v = dsub(v, dmul(tw[i], prev));
                    if (i == n - 1) v = ddiv(v, tb[n - 1]);
                    T[lane][k] = v;
                    prev = v;
                }
            }
            __syncwarp();
            for (int r = 0; r < nl; r++)
                if (lane < m) arr[(base + r) * n + t0 + lane] = T[r][lane];
            __syncwarp();
        }
        double last = prev;
        for (int t0 = ((n - 1) / 32) * 32; t0 >= 0; t0 -= 32) {
            const int m = min(32, n - t0);
            if (lane < m)
                for (int r = 0; r < nl; r++) cp_async<8>(&T[r][lane], arr + (base + r) * n + t0 + lane);
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
            if (lane < nl) {
                for (int k = m - 1; k >= 0; k--) {
                    const int i = t0 + k;
                    if (i == n - 1) continue;
                    double v = dsub(T[lane][k], dmul(tu[i], last));
                    v = ddiv(v, tb[i]);
                    T[lane][k] = v;
                    last = v;
                }
            }
            __syncwarp();
            if (EPI) {   // coarse + corr: the coarse values of the tile rows in flight together
                for (int r0 = 0; r0 < nl; r0 += 8) {
                    double cv[8];
#pragma unroll
                    for (int k = 0; k < 8; k++)
                        cv[k] = (r0 + k < nl && lane < m) ? __ldg(epi.base + (base + r0 + k) * n + t0 + lane) : 0.0;
#pragma unroll
                    for (int k = 0; k < 8; k++)
                        if (r0 + k < nl && lane < m) epi.dst[(base + r0 + k) * n + t0 + lane] = dadd(cv[k], T[r0 + k][lane]);
                }
            } else {
                for (int r = 0; r < nl; r++)
                    if (lane < m) arr[(base + r) * n + t0 + lane] = T[r][lane];
            }
            __syncwarp();
        }
    }
}

// Register-blocked sweeps: one thread per line, U values of the line loaded ahead of the
// recurrence (double-buffered), so the sequential dependency never waits on DRAM.  Works for
// strided (inner > 1, coalesced across threads) and contiguous (inner == 1) lines alike.
template <int U, bool EPI, int PH = 0>
__global__ void __launch_bounds__(128) k_thomas_reg(double *__restrict__ arr, int64_t outer, int32_t n, int64_t inner,
                                                    const double *__restrict__ tw, const double *__restrict__ tb,
                                                    const double *__restrict__ tu, const double *__restrict__ tr,
                                                    Epi epi, int32_t f_lo = 1, int32_t f_hi = 0) {
    // PH 0: the whole solve.  PH 1: forward elimination of positions [f_lo, f_hi) only (f_lo >= 1; the
    // planes below are already eliminated -- a solve that follows its right-hand side as it is
    // produced).  PH 2: back substitution only.  The split solve does the same operations in the
    // same order as PH 0.
    const int64_t lines = outer * inner;
    if (PH == 0) f_hi = n;
    for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < lines; ln += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = ln / inner, q = ln - p * inner;
        double *x = arr + p * (int64_t)n * inner + q;
        const int64_t o = p * (int64_t)n * inner + q;
        double cur[U], nxt[U];
        auto load = [&](double *buf, int i0, int lim) {
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int i = i0 + k;
                if (i >= 0 && i < lim) buf[k] = x[(int64_t)i * inner];
            }
        };
        double prev;
        if (PH != 2) {
            // forward elimination: x_i -= w_i x_{i-1}
            prev = x[(int64_t)(f_lo - 1) * inner];
            load(cur, f_lo, f_hi);
            for (int i0 = f_lo; i0 < f_hi; i0 += U) {
                if (i0 + U < f_hi) load(nxt, i0 + U, f_hi);
#pragma unroll
                for (int k = 0; k < U; k++) {
                    const int i = i0 + k;
                    if (i < f_hi) {
                        const double v = dsub(cur[k], dmul(__ldg(tw + i), prev));
                        x[(int64_t)i * inner] = v;
                        prev = v;
                    }
                }
#pragma unroll
                for (int k = 0; k < U; k++) cur[k] = nxt[k];
            }
        } else {
            prev = x[(int64_t)(n - 1) * inner];
        }
        if (PH == 1) continue;
        double last = ddiv(prev, __ldg(tb + n - 1));   // (__ddiv_rn beat a checked fast division here)
        epi_store<EPI>(arr, o + (int64_t)(n - 1) * inner, last, epi);
        // back substitution: x_i = (x_i - u_i x_{i+1}) / b'_i, i = n-2 .. 0
        load(cur, n - 1 - U, n);
        for (int i1 = n - 2; i1 >= 0; i1 -= U) {
            if (i1 - U >= 0) load(nxt, i1 - 2 * U + 1, n);
#pragma unroll
            for (int k = U - 1; k >= 0; k--) {
                const int i = i1 - (U - 1 - k);
                if (i >= 0) {
                    double v = dsub(cur[k], dmul(__ldg(tu + i), last));
                    v = ddiv(v, __ldg(tb + i));
                    epi_store<EPI>(arr, o + (int64_t)i * inner, v, epi);
                    last = v;
                }
            }
#pragma unroll
            for (int k = 0; k < U; k++) cur[k] = nxt[k];
        }
    }
}

// Tiled Thomas solve: one warp owns 32 lines, staged whole in shared memory by cp.async
// (strided axes: row i of the tile = 32 consecutive inner columns, one coalesced 256-byte
// segment; contiguous axis: 32 contiguous lines, row stride padded odd so lane-per-line reads are
// bank-conflict free).  Forward elimination and back substitution run in shared memory with the
// reference's rounding (transform.py:236-242; division verified as above, exact redo otherwise),
// then the tile is written back coalesced: 16 bytes of DRAM traffic per node.
constexpr int kThomasTileMaxN = 880;   // 32 lines x 880 x 8 B = 220 KB of shared memory

template <bool CONTIG, bool EPI>
__global__ void __launch_bounds__(32) k_thomas_tile(double *__restrict__ arr, int64_t outer, int32_t n,
                                                    int64_t inner, int32_t ls, const double *__restrict__ tw,
                                                    const double *__restrict__ tb, const double *__restrict__ tu,
                                                    const double *__restrict__ tr, Epi epi) {
    extern __shared__ __align__(16) double tsm[];
    const int lane = threadIdx.x;
    // element (line l, position i) of the tile
    auto at = [&](int l, int i) -> double & { return CONTIG ? tsm[(int64_t)l * ls + i] : tsm[(int64_t)i * 32 + l]; };
    const int64_t tiles_per_outer = CONTIG ? 1 : (inner + 31) / 32;
    const int64_t tiles = CONTIG ? (outer + 31) / 32 : outer * tiles_per_outer;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t p = 0, q0 = 0, l0 = 0;
        int nl;
        if (CONTIG) {
            l0 = t * 32;
            nl = (int)min64(32, outer - l0);
        } else {
            p = t / tiles_per_outer;
            q0 = (t - p * tiles_per_outer) * 32;
            nl = (int)min64(32, inner - q0);
        }
        // stage the tile
        if (CONTIG) {
            for (int l = 0; l < nl; l++) {
                const double *src = arr + (l0 + l) * (int64_t)n;
                for (int i = lane; i < n; i += 32) cp_async<8>(&at(l, i), src + i);
            }
        } else if (lane < nl) {
            const double *src = arr + p * (int64_t)n * inner + q0 + lane;
            for (int i = 0; i < n; i++) cp_async<8>(&at(lane, i), src + (int64_t)i * inner);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane < nl) {
            // forward elimination x_i -= w_i x_{i-1}, 8 values per batch read ahead of the chain
            constexpr int U = 8;
            double prev = at(lane, 0);
            int i0 = 1;
            for (; i0 + U <= n; i0 += U) {
                double v[U], w[U];
#pragma unroll
                for (int k = 0; k < U; k++) {
                    v[k] = at(lane, i0 + k);
                    w[k] = __ldg(tw + i0 + k);
                }
#pragma unroll
                for (int k = 0; k < U; k++) {
                    prev = dsub(v[k], dmul(w[k], prev));
                    v[k] = prev;
                }
#pragma unroll
                for (int k = 0; k < U; k++) at(lane, i0 + k) = v[k];
            }
            for (; i0 < n; i0++) {
                prev = dsub(at(lane, i0), dmul(__ldg(tw + i0), prev));
                at(lane, i0) = prev;
            }
            // back substitution: x_{n-1} /= b'_{n-1}; x_i = (x_i - u_i x_{i+1}) / b'_i with the
            // verified fast division off the dependency chain's check; a failed check redoes the
            // line from the untouched global values with __ddiv_rn
            bool bad = false;
            double last = div_fast(prev, __ldg(tb + n - 1), __ldg(tr + n - 1), bad);
            at(lane, n - 1) = last;
            int i1 = n - 2;
            for (; i1 - U + 1 >= 0; i1 -= U) {
                double v[U], u[U], b[U], r[U];
#pragma unroll
                for (int k = 0; k < U; k++) {
                    v[k] = at(lane, i1 - k);
                    u[k] = __ldg(tu + i1 - k);
                    b[k] = __ldg(tb + i1 - k);
                    r[k] = __ldg(tr + i1 - k);
                }
#pragma unroll
                for (int k = 0; k < U; k++) {
                    last = div_fast(dsub(v[k], dmul(u[k], last)), b[k], r[k], bad);
                    v[k] = last;
                }
#pragma unroll
                for (int k = 0; k < U; k++) at(lane, i1 - k) = v[k];
            }
            for (; i1 >= 0; i1--) {
                last = div_fast(dsub(at(lane, i1), dmul(__ldg(tu + i1), last)), __ldg(tb + i1), __ldg(tr + i1), bad);
                at(lane, i1) = last;
            }
            if (bad) {   // rare: the whole line again, exactly
                const int64_t st_ = CONTIG ? 1 : inner;
                const double *src = CONTIG ? arr + (l0 + lane) * (int64_t)n : arr + p * (int64_t)n * inner + q0 + lane;
                prev = src[0];
                at(lane, 0) = prev;
                for (int i = 1; i < n; i++) {
                    prev = dsub(src[(int64_t)i * st_], dmul(__ldg(tw + i), prev));
                    at(lane, i) = prev;
                }
                last = ddiv(prev, __ldg(tb + n - 1));
                at(lane, n - 1) = last;
                for (int i = n - 2; i >= 0; i--) {
                    last = ddiv(dsub(at(lane, i), dmul(__ldg(tu + i), last)), __ldg(tb + i));
                    at(lane, i) = last;
                }
            }
        }
        __syncwarp();
        // write back (with the coarse + corr epilogue the coarse values of 8 elements are loaded
        // together, ahead of their stores)
        if (CONTIG) {
            const int tot = nl * n;
            const int64_t o = l0 * (int64_t)n;   // the tile's lines are contiguous
            for (int j0 = lane; j0 < tot; j0 += 32 * 8) {
                double cv[8];
                if (EPI) {
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        const int j = j0 + 32 * k;
                        cv[k] = j < tot ? __ldg(epi.base + o + j) : 0.0;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int j = j0 + 32 * k;
                    if (j < tot) {
                        const int l = j / n, i = j - l * n;
                        if (EPI) epi.dst[o + j] = dadd(cv[k], at(l, i));
                        else arr[o + j] = at(l, i);
                    }
                }
            }
        } else if (lane < nl) {
            const int64_t o = p * (int64_t)n * inner + q0 + lane;
            for (int i0 = 0; i0 < n; i0 += 8) {
                double cv[8];
                if (EPI) {
#pragma unroll
                    for (int k = 0; k < 8; k++) cv[k] = i0 + k < n ? __ldg(epi.base + o + (int64_t)(i0 + k) * inner) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 8; k++)
                    if (i0 + k < n) {
                        if (EPI) epi.dst[o + (int64_t)(i0 + k) * inner] = dadd(cv[k], at(lane, i0 + k));
                        else arr[o + (int64_t)(i0 + k) * inner] = at(lane, i0 + k);
                    }
            }
        }
        __syncwarp();
    }
}

// Self-test of div_fast against __ddiv_rn over pseudo-random operands (hpdr_selftest_div).
__global__ void k_selftest_div(uint64_t n, uint64_t seed, unsigned long long *mism, unsigned long long *fallback) {
    unsigned long long m = 0, f = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + i * 0x9E3779B97F4A7C15ULL;
        auto mix = [](uint64_t x) {
            x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
            x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
            return x ^ (x >> 31);
        };
        const uint64_t r1 = mix(z), r2 = mix(z + 1);
        // a: any sign, exponent within +-40 of 1; b: positive, exponent within +-20 (Thomas pivots)
        const double a = __longlong_as_double((long long)((r1 & 0x800fffffffffffffULL) | ((uint64_t)(1023 - 40 + (r1 >> 52) % 81) << 52)));
        const double b = __longlong_as_double((long long)((r2 & 0x000fffffffffffffULL) | ((uint64_t)(1023 - 20 + (r2 >> 52) % 41) << 52)));
        bool bad = false;
        const double q = div_fast(a, b, ddiv(1.0, b), bad);
        if (bad) f++;
        else if (__double_as_longlong(q) != __double_as_longlong(ddiv(a, b))) m++;
    }
    if (m) atomicAdd(mism, m);
    if (f) atomicAdd(fallback, f);
}

// All Thomas solves of one small coarse grid in a single CTA (grid staged in shared memory): the
// axes in order with a barrier between them (transform.py:259-260), each line by one thread with the
// same recurrence and rounding as k_thomas_reg.  Replaces up to 3 latency-bound launches per small
// level (the coarse end of every hierarchy, and every level of a thin pipeline chunk).
constexpr int kThomasSmallMax = 16384;   // doubles (128 KB of shared memory)
constexpr int kThomasSmallTabs = 8192;   // staged table doubles (64 KB)

struct AxesArg {
    DevAxis ax[4];
};

template <bool EPI>
__global__ void __launch_bounds__(512) k_thomas_small(double *__restrict__ arr, Shape4 sh, AxesArg A, Epi epi,
                                                      int stage_tabs) {
    extern __shared__ double g[];
    const int64_t N = sh.size();
    // the axes' (w, b', u) tables ride along in shared memory (loaded together with the grid, so the
    // recurrences never wait on a cold table load)
    double *tabs = g + N;
    const double *tw[4], *tb[4], *tu[4], *tr[4];
    {
        int off = 0;
        for (int a = 0; a < 4; a++) {
            const DevAxis &ax = A.ax[a];
            tw[a] = ax.tw;
            tb[a] = ax.tb;
            tu[a] = ax.tu;
            tr[a] = ax.tr;
            if (!ax.active || !stage_tabs) continue;
            const int n = ax.nc;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                tabs[off + i] = __ldg(ax.tw + i);
                tabs[off + n + i] = __ldg(ax.tb + i);
                tabs[off + 2 * n + i] = __ldg(ax.tu + i);
                tabs[off + 3 * n + i] = __ldg(ax.tr + i);
            }
            tw[a] = tabs + off;
            tb[a] = tabs + off + n;
            tu[a] = tabs + off + 2 * n;
            tr[a] = tabs + off + 3 * n;
            off += 4 * n;
        }
    }
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) g[i] = arr[i];
    __syncthreads();
    for (int a = 0; a < 4; a++) {
        const DevAxis &ax = A.ax[a];
        if (!ax.active) continue;
        int64_t outer = 1, inner = 1;
        for (int d = 0; d < a; d++) outer *= sh.n[d];
        for (int d = a + 1; d < 4; d++) inner *= sh.n[d];
        const int n = ax.nc;
        const double *W = tw[a], *B = tb[a], *U = tu[a], *Rr = tr[a];
        // verified fast division (div_fast), exact __ddiv_rn for the rare operand it cannot certify
        auto div = [](double x, double b, double r) {
            bool bad = false;
            const double q = div_fast(x, b, r, bad);
            return bad ? ddiv(x, b) : q;
        };
        const int64_t lines = outer * inner;
        for (int64_t ln = threadIdx.x; ln < lines; ln += blockDim.x) {
            const int64_t p = ln / inner, q = ln - p * inner;
            double *x = g + p * (int64_t)n * inner + q;
            double prev = x[0];
            for (int i = 1; i < n; i++) {
                prev = dsub(x[(int64_t)i * inner], dmul(W[i], prev));
                x[(int64_t)i * inner] = prev;
            }
            double last = div(prev, B[n - 1], Rr[n - 1]);
            x[(int64_t)(n - 1) * inner] = last;
            for (int i = n - 2; i >= 0; i--) {
                last = div(dsub(x[(int64_t)i * inner], dmul(U[i], last)), B[i], Rr[i]);
                x[(int64_t)i * inner] = last;
            }
        }
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) epi_store<EPI>(arr, i, g[i], epi);
}

// ---------------------------------------------------------------- elementwise
__global__ void k_add(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ o, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = dadd(a[i], b[i]);
}
__global__ void k_sub(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ o, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = dsub(a[i], b[i]);
}

template <typename T>
__global__ void k_cast(const double *__restrict__ src, T *__restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (T)src[i];
}

// ---------------------------------------------------------------- host helpers
void view(const Shape4 &sh, int a, int64_t &outer, int64_t &inner) {
    outer = 1;
    inner = 1;
    for (int d = 0; d < a; d++) outer *= sh.n[d];
    for (int d = a + 1; d < 4; d++) inner *= sh.n[d];
}

dim3 rows_grid(const Shape4 &sh) {
    int64_t rows = sh.n[0] * sh.n[1] * sh.n[2];
    unsigned gx = (unsigned)std::min<int64_t>((sh.n[3] + 255) / 256, 64);
    unsigned gy = (unsigned)std::min<int64_t>(rows, 65535);
    if (gx < 1) gx = 1;
    if (gy < 1) gy = 1;
    return dim3(gx, gy);
}

void prolong(const double *src, double *dst, const double *aux, int mode, const Shape4 &csh, int a,
             const DevAxis &ax, cudaStream_t s) {
    int64_t outer, inner;
    view(csh, a, outer, inner);
    const int64_t per = (int64_t)ax.n * inner;
    dim3 grid(grid_for(per, 256, 4096), (unsigned)std::min<int64_t>(outer, 65535));
    const bool small = per < (1LL << 32);
    KPROF("k_prolong", 8.0 * outer * ((double)ax.nc * inner + (mode ? 2.0 : 1.0) * per), s);
#define PL(M)                                                                                                \
    if (small)                                                                                                  \
        k_prolong<M, uint32_t><<<grid, 256, 0, s>>>(src, dst, aux, outer, ax.nc, ax.n, inner, ax.pa, ax.pb, ax.pt); \
    else                                                                                                        \
        k_prolong<M, uint64_t><<<grid, 256, 0, s>>>(src, dst, aux, outer, ax.nc, ax.n, inner, ax.pa, ax.pb, ax.pt)
    if (mode == 0) PL(0);
    else if (mode == 1) PL(1);
    else PL(2);
#undef PL
    LAUNCH_CHECK();
}

void mass_restrict(const double *src, double *dst, const Shape4 &fsh, int a, const DevAxis &ax, cudaStream_t s) {
    int64_t outer, inner;
    view(fsh, a, outer, inner);
    const int64_t per = (int64_t)ax.nc * inner;
    dim3 grid(grid_for(per, 256, 4096), (unsigned)std::min<int64_t>(outer, 65535));
    KPROF("k_mass_restrict", 8.0 * outer * ((double)ax.n * inner + per), s);
    if (per < (1LL << 32))
        k_mass_restrict<uint32_t><<<grid, 256, 0, s>>>(src, dst, outer, ax.n, ax.nc, inner, ax);
    else
        k_mass_restrict<uint64_t><<<grid, 256, 0, s>>>(src, dst, outer, ax.n, ax.nc, inner, ax);
    LAUNCH_CHECK();
}

void thomas(double *arr, const Shape4 &csh, int a, const DevAxis &ax, cudaStream_t s, Epi epi = Epi{}) {
    int64_t outer, inner;
    view(csh, a, outer, inner);
    KPROF(inner == 1 ? "k_thomas_contig" : "k_thomas_strided", (epi.dst ? 24.0 : 16.0) * outer * inner * ax.nc, s);
    // strided axes: register-blocked lines (coalesced across threads); contiguous axis: the
    // warp-tile transpose kernel measured faster (0.39 vs 0.45 ms at 257^3 coarse grid)
    static const bool legacy = getenv("HPDR_THOMAS_LEGACY") != nullptr;
    static const int tile_mode = [] {   // HPDR_THOMAS_TILE: 0 never, 1 always, unset: few lines only
        const char *e = getenv("HPDR_THOMAS_TILE");
        return e ? atoi(e) : 2;
    }();
    const bool few = outer * inner < (int64_t)148 * 128;
    if (!legacy && (tile_mode == 1 || (tile_mode == 2 && few)) && ax.nc <= kThomasTileMaxN) {
        const int n = ax.nc;
        if (inner == 1) {
            const int ls = n | 1;   // odd row stride: lane-per-line reads hit distinct banks
            const size_t smem = (size_t)32 * ls * 8;
            static int attr_c = 0;
            if (smem > 48 * 1024 && attr_c < (int)smem) {
                for (auto f : {k_thomas_tile<true, false>, k_thomas_tile<true, true>})
                    CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)(32 * (kThomasTileMaxN | 1) * 8)));
                attr_c = 32 * (kThomasTileMaxN | 1) * 8;
            }
            const int64_t tiles = (outer + 31) / 32;
            if (epi.dst)
                k_thomas_tile<true, true><<<(unsigned)std::min<int64_t>(tiles, 148 * 32), 32, smem, s>>>(
                    arr, outer, n, inner, ls, ax.tw, ax.tb, ax.tu, ax.tr, epi);
            else
                k_thomas_tile<true, false><<<(unsigned)std::min<int64_t>(tiles, 148 * 32), 32, smem, s>>>(
                    arr, outer, n, inner, ls, ax.tw, ax.tb, ax.tu, ax.tr, epi);
        } else {
            const size_t smem = (size_t)32 * n * 8;
            static int attr_s = 0;
            if (smem > 48 * 1024 && attr_s < (int)smem) {
                for (auto f : {k_thomas_tile<false, false>, k_thomas_tile<false, true>})
                    CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)(32 * kThomasTileMaxN * 8)));
                attr_s = 32 * kThomasTileMaxN * 8;
            }
            const int64_t tiles = outer * ((inner + 31) / 32);
            if (epi.dst)
                k_thomas_tile<false, true><<<(unsigned)std::min<int64_t>(tiles, 148 * 32), 32, smem, s>>>(
                    arr, outer, n, inner, 0, ax.tw, ax.tb, ax.tu, ax.tr, epi);
            else
                k_thomas_tile<false, false><<<(unsigned)std::min<int64_t>(tiles, 148 * 32), 32, smem, s>>>(
                    arr, outer, n, inner, 0, ax.tw, ax.tb, ax.tu, ax.tr, epi);
        }
    } else if (!legacy && inner > 1) {
        const int64_t lines = outer * inner;
        if (epi.dst)
            k_thomas_reg<8, true><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(arr, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                              ax.tu, ax.tr, epi);
        else
            k_thomas_reg<8, false><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(arr, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                               ax.tu, ax.tr, epi);
    } else if (inner == 1) {
        int64_t lines = outer;
        unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lines + 127) / 128, 148 * 16));
        if (epi.dst) k_thomas_contig<true><<<g, kThomasWarps * 32, 0, s>>>(arr, lines, ax.nc, ax.tw, ax.tb, ax.tu, ax.tr, epi);
        else k_thomas_contig<false><<<g, kThomasWarps * 32, 0, s>>>(arr, lines, ax.nc, ax.tw, ax.tb, ax.tu, ax.tr, epi);
    } else {
        int64_t lines = outer * inner;
        if (epi.dst)
            k_thomas_strided<true><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(arr, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                               ax.tu, epi);
        else
            k_thomas_strided<false><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(arr, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                                ax.tu, epi);
    }
    LAUNCH_CHECK();
}

Sel4 level_map(const DevPlan &p, int k) {
    Sel4 m;
    for (int d = 0; d < 4; d++) m.s[d] = p.map[d][k];
    return m;
}

Sel4 coarse_flags(const DevStep &st) {
    Sel4 f;
    for (int d = 0; d < 4; d++) f.s[d] = st.ax[d].active ? st.ax[d].pb : nullptr;
    return f;
}

double *level_ptr(const LevelBuffers &b, const DevPlan &p, int k) {
    return k == 0 ? b.lvl0 : b.arena + p.level_off[k];
}

// Correction of transform.py:251-260: mass+restrict per active axis, then Thomas per active axis.
const double *correction(const DevStep &st, const double *mc, const LevelBuffers &b, cudaStream_t s) {
    const double *cur = mc;
    Shape4 sh = st.fsh;
    int k = 0;
    for (int a = 0; a < 4; a++) {
        if (!st.ax[a].active) continue;
        double *out = (k++ % 2 == 0) ? b.t0 : b.t1;
        mass_restrict(cur, out, sh, a, st.ax[a], s);
        sh.n[a] = st.csh.n[a];
        cur = out;
    }
    for (int a = 0; a < 4; a++)
        if (st.ax[a].active) thomas(const_cast<double *>(cur), sh, a, st.ax[a], s);
    return cur;
}

// Interpolation of transform.py:261-268, the last axis fused with the residual / add (mode 1 / 2).
void interpolate(const DevStep &st, const double *coarse, double *out, const double *aux, int mode,
                 const LevelBuffers &b, cudaStream_t s) {
    int na = 0;
    for (int a = 0; a < 4; a++) na += st.ax[a].active;
    const double *cur = coarse;
    Shape4 sh = st.csh;
    int k = 0;
    for (int a = 0; a < 4; a++) {
        if (!st.ax[a].active) continue;
        const bool last = (k == na - 1);
        double *dst = last ? out : ((k % 2 == 0) ? b.t0 : b.t1);
        prolong(cur, dst, last ? aux : nullptr, last ? mode : 0, sh, a, st.ax[a], s);
        sh.n[a] = st.fsh.n[a];
        cur = dst;
        k++;
    }
}

}  // namespace

LevelBuffers level_buffers(hpdr_ctx *ctx, DevPlan &p) {
    LevelBuffers b;
    const int64_t N = p.n_total;
    const int64_t C1 = p.host.L > 1 ? p.level_size[1] : 1;
    b.lvl0 = (double *)ctx->dbuf("lvl0", N * 8);
    b.arena = (double *)ctx->dbuf("arena", std::max<int64_t>(p.coarse_arena, 1) * 8);
    b.mc = (double *)ctx->dbuf("mc", N * 8);
    b.t0 = (double *)ctx->dbuf("t0", N * 8);
    b.t1 = (double *)ctx->dbuf("t1", N * 8);
    b.cg = (double *)ctx->dbuf("cg", C1 * 8);
    return b;
}

void minmax_device(hpdr_ctx *ctx, const void *d_in, int dtype, int64_t n, double *vmin, double *vmax, cudaStream_t s) {
    unsigned long long *d = (unsigned long long *)ctx->dbuf("minmax", 32);
    unsigned long long *h = (unsigned long long *)ctx->hbuf("minmax_h", 32);
    store_u64(d, ~0ULL, s);
    store_u64(d + 1, 0ULL, s);
    store_u64(d + 2, 0ULL, s);
    {
        KPROF("k_minmax", (double)n * (dtype == 0 ? 4 : 8), s);
        k_minmax<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(d_in, dtype, n, d);
        LAUNCH_CHECK();
    }
    small_copy(h, d, 24, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (h[2]) {
        *vmin = __builtin_nan("");
        *vmax = __builtin_nan("");
        return;
    }
    auto val = [](unsigned long long k) {
        unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
        double d;
        memcpy(&d, &u, 8);
        return d;
    };
    *vmin = val(h[0]);
    *vmax = val(h[1]);
}

void minmax_accumulate(const void *d_in, int dtype, int64_t n, unsigned long long *mm, cudaStream_t s) {
    KPROF("k_minmax", (double)n * (dtype == 0 ? 4 : 8), s);
    k_minmax<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(d_in, dtype, n, mm);
    LAUNCH_CHECK();
}

void minmax_from_keys(const unsigned long long *h, double *vmin, double *vmax) {
    if (h[2]) {
        *vmin = __builtin_nan("");
        *vmax = __builtin_nan("");
        return;
    }
    auto val = [](unsigned long long k) {
        unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
        double d;
        memcpy(&d, &u, 8);
        return d;
    };
    *vmin = val(h[0]);
    *vmax = val(h[1]);
}

bool use_fused(const DevPlan &p) {
    static const bool generic = getenv("HPDR_GENERIC") != nullptr && getenv("HPDR_GENERIC")[0] == '1';
    return fused_supported(p) && !generic;
}

namespace {

// Work buffers of the fused path: coarse-level arena, pass-1 output Z0, pass-2 / Thomas
// buffer t0 and the coarse gather cg (no full-size fp64 level copies).
LevelBuffers fused_buffers(hpdr_ctx *ctx, DevPlan &p) {
    LevelBuffers b{};
    int64_t zmax = 1, cmax = 1;
    for (const DevStep &st : p.steps) {
        const int64_t m0 = st.ax[1].active ? st.csh.n[1] : st.fsh.n[1];
        zmax = std::max<int64_t>(zmax, m0 * st.fsh.n[2] * st.fsh.n[3]);
        cmax = std::max<int64_t>(cmax, st.csh.size());
    }
    b.arena = (double *)ctx->dbuf("arena", std::max<int64_t>(p.coarse_arena, 1) * 8);
    b.t0 = (double *)ctx->dbuf("t0", cmax * 8);
    b.cg = (double *)ctx->dbuf("cg", cmax * 8);
    b.mc = (double *)ctx->dbuf("z0", zmax * 8);   // Z0 of pass 1
    return b;
}

// Fused decomposition (ranks <= 3): pass 1 (GPK residual + coefficients + axis-0 LPK), pass 2
// (axis-1/2 LPK), IPK Thomas sweeps, coarse + corr.  q != nullptr quantizes on write.
const double *decompose_fused(hpdr_ctx *ctx, DevPlan &p, const void *d_in, int dtype, double *coef,
                              const QuantOut *q, cudaStream_t s, int st_end = -1) {
    LevelBuffers b = fused_buffers(ctx, p);
    const int L = p.host.L;
    double *Z0 = b.mc;
    if (st_end < 0) st_end = L - 1;
    for (int st_i = 0; st_i < st_end; st_i++) {
        const DevStep &st = p.steps[st_i];
        const void *F = st_i == 0 ? d_in : (const void *)level_ptr(b, p, st_i);
        double *Dn = level_ptr(b, p, st_i + 1);
        if (st_i == 1) phase_mark("level0_done", s);
        if (q) fused_pass1_quantize(p, st_i, F, st_i == 0 && dtype == 0, *q, Z0, b.cg, s);
        else fused_pass1_decompose(p, st_i, F, st_i == 0 && dtype == 0, coef, Z0, b.cg, s);
        fused_pass2(p, st_i, Z0, b.t0, s);
        thomas_all(p, st_i, b.t0, s, b.cg, Dn);   // Dn = coarse + corr, fused into the last sweep
    }
    return level_ptr(b, p, L - 1);
}

// Levels 1 .. L-2 of a quantizing decomposition plus the coarsest quantization: small, latency-
// bound launches, replayed from a CUDA graph after the first direct run (the bin width, the only
// per-call scalar, is read from device memory in the graph).
const double *coarse_levels_quantize(hpdr_ctx *ctx, DevPlan &p, const QuantOut &q, cudaStream_t s) {
    LevelBuffers b = fused_buffers(ctx, p);
    const int L = p.host.L;
    double *Z0 = b.mc;
    const int tiny = tiny_start(p, 1);   // the small end of the hierarchy in one block
    auto body = [&](const QuantOut &qq) {
        for (int st_i = 1; st_i + 1 < L; st_i++) {
            if (st_i == tiny) {
                tiny_decompose_quantize(p, st_i, level_ptr(b, p, st_i), level_ptr(b, p, L - 1), qq, s);
                return;
            }
            fused_pass1_quantize(p, st_i, level_ptr(b, p, st_i), false, qq, Z0, b.cg, s);
            fused_pass2(p, st_i, Z0, b.t0, s);
            thomas_all(p, st_i, b.t0, s, b.cg, level_ptr(b, p, st_i + 1));
        }
        quantize_coarsest(p, level_ptr(b, p, L - 1), qq, s);
    };
    static const bool no_graph = getenv("HPDR_NO_GRAPH") != nullptr || getenv("HPDR_DEBUG_SYNC") != nullptr;
    double *bin_dev = (double *)ctx->dbuf("bin_dev", 16);   // allocated on the warm call (CMM: no realloc)
    if (L <= 2 || no_graph || !ctx->graphs_ok || prof_enabled() || !p.graph_warm) {
        p.graph_warm = true;
        body(q);
        return level_ptr(b, p, L - 1);
    }
    const std::vector<uintptr_t> key = {(uintptr_t)b.arena, (uintptr_t)b.mc,  (uintptr_t)b.cg,    (uintptr_t)b.t0,
                                        (uintptr_t)q.keys,  (uintptr_t)q.omask, (uintptr_t)q.obins, (uintptr_t)q.hist,
                                        (uintptr_t)q.flags, (uintptr_t)q.half, (uintptr_t)q.dict,  (uintptr_t)bin_dev};
    DevPlan::Graph *g = nullptr;
    for (auto &e : p.graphs)
        if (e.key == key) g = &e;
    const double binv = q.bin;
    uint64_t binbits;
    memcpy(&binbits, &binv, 8);
    store_u64(bin_dev, binbits, s);
    if (!g) {
        QuantOut qg = q;
        qg.bin_dev = bin_dev;
        cudaGraph_t graph = nullptr;
        CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            body(qg);
        } catch (...) {
            cudaStreamEndCapture(s, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(s, &graph));
        DevPlan::Graph e;
        e.key = key;
        size_t nodes = 0;
        CUDA_CHECK(cudaGraphGetNodes(graph, nullptr, &nodes));
        e.kernels = nodes;
        CUDA_CHECK(cudaGraphInstantiate(&e.exec, graph, 0));
        CUDA_CHECK(cudaGraphDestroy(graph));
        if (p.graphs.size() >= 4) {   // bounded: buffers grow rarely
            cudaGraphExecDestroy(p.graphs.front().exec);
            p.graphs.erase(p.graphs.begin());
        }
        p.graphs.push_back(e);
        g = &p.graphs.back();
    }
    CUDA_CHECK(cudaGraphLaunch(g->exec, s));
    count_launches(g->kernels);
    return level_ptr(b, p, L - 1);
}

}  // namespace

const double *decompose_quantize_streamed(hpdr_ctx *ctx, DevPlan &p, const void *host_in, int dtype, bool has_range,
                                          double range_min, double range_max, double eb_rel, QuantOut &q,
                                          double *u_min, double *u_max, cudaStream_t s) {
    LevelBuffers b = fused_buffers(ctx, p);
    const int L = p.host.L;
    const DevStep &st0 = p.steps[0];
    const int n0 = (int)st0.fsh.n[1];
    const int64_t plane_elems = st0.fsh.n[2] * st0.fsh.n[3];
    const size_t isz = dtype == 0 ? 4 : 8;
    const int64_t N = p.n_total;
    char *d_in = (char *)ctx->dbuf("input", N * isz);
    double *Z0 = b.mc;
    double *coef = has_range ? nullptr : (double *)ctx->dbuf("coef", N * 8);
    // chunks of >= 32 MB (and >= 4 planes) along dim 0
    const int64_t plane_bytes = plane_elems * (int64_t)isz;
    // (a small field still arrives in >= 4 pieces, so its finest pass overlaps the copy)
    const int64_t target = std::min<int64_t>(32LL << 20, std::max<int64_t>(1LL << 20, (int64_t)n0 * plane_bytes / 4));
    int chunk = (int)std::max<int64_t>(4, (target + plane_bytes - 1) / std::max<int64_t>(plane_bytes, 1));
    chunk = std::min(chunk, n0);
    const int K = (n0 + chunk - 1) / chunk;
    unsigned long long *mm = (unsigned long long *)ctx->dbuf("minmax", 32);
    if (has_range) {   // absolute bound: the bin width is known before any data arrives
        const double eb_abs = eb_rel * (range_max - range_min);
        q.bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)L : 1.0;
    } else {
        store_u64(mm, ~0ULL, s);
        store_u64(mm + 1, 0ULL, s);
        store_u64(mm + 2, 0ULL, s);
    }
    // coarse outputs of transition 0 whose 5-plane stencil lies within the first `arrived` planes
    const AxisTables &ax0 = p.host.steps[0].ax[1];
    const int m0 = fused_out_planes(p, 0);
    auto ready = [&](int arrived) -> int {
        if (arrived >= n0) return m0;
        if (!ax0.active) return arrived;
        int c = 0;
        while (c < m0 && ax0.r0[c] + 2 < arrived) c++;
        return c;
    };
    // the event the compute stream waits on before touching chunk k
    CUDA_CHECK(cudaEventRecord(ctx->event(0), s));
    CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(0), 0));   // buffers are free once prior work is done
    const bool pageable_in = classify(host_in) == MemKind::Host;
    auto issue = [&](int k) {   // pageable input: staged while the previous chunk is being reduced
        const int64_t a = (int64_t)k * chunk, e = std::min<int64_t>(n0, a + chunk);
        if (pageable_in)
            stage_h2d(ctx, d_in + a * plane_bytes, (const char *)host_in + a * plane_bytes, (e - a) * plane_bytes,
                      ctx->h2d);
        else
            CUDA_CHECK(cudaMemcpyAsync(d_in + a * plane_bytes, (const char *)host_in + a * plane_bytes,
                                       (e - a) * plane_bytes, cudaMemcpyDefault, ctx->h2d));
        CUDA_CHECK(cudaEventRecord(ctx->event(EvChunkIn, k), ctx->h2d));
    };
    issue(0);
    int c_done = 0;
    const bool fwd = thomas_fwd_stream(p, 0);
    for (int k = 0; k < K; k++) {
        CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(EvChunkIn, k), 0));
        const int64_t a = (int64_t)k * chunk, e = std::min<int64_t>(n0, a + chunk);
        if (!has_range) {
            const int64_t cnt = (e - a) * plane_elems;
            KPROF("k_minmax", (double)cnt * isz, s);
            k_minmax<<<grid_for(cnt, 256, 148 * 8), 256, 0, s>>>(d_in + a * plane_bytes, dtype, cnt, mm);
            LAUNCH_CHECK();
        }
        const int c_ready = ready((int)e);
        if (c_ready > c_done) {
            if (has_range) fused_pass1_quantize(p, 0, d_in, dtype == 0, q, Z0, b.cg, s, c_done, c_ready);
            else fused_pass1_decompose(p, 0, d_in, dtype == 0, coef, Z0, b.cg, s, c_done, c_ready);
            fused_pass2(p, 0, Z0, b.t0, s, c_done, c_ready);
            if (fwd) thomas_plane_fwd(p, 0, b.t0, c_done, c_ready, s);   // the solve follows its right-hand side
            c_done = c_ready;
        }
        if (k + 1 < K) issue(k + 1);
    }
    phase_mark("last_chunk_issued", s);
    bool side = false;
    if (has_range) {
        *u_min = range_min;
        *u_max = range_max;
    } else {
        unsigned long long *h = (unsigned long long *)ctx->hbuf("minmax_h", 32);
        small_copy(h, mm, 24, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
        auto val = [](unsigned long long k) {
            unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
            double d;
            memcpy(&d, &u, 8);
            return d;
        };
        *u_min = h[2] ? __builtin_nan("") : val(h[0]);
        *u_max = h[2] ? __builtin_nan("") : val(h[1]);
        apply_range_hook(ctx, u_min, u_max);   // job-wide range of a block-partitioned field
        const double eb_abs = eb_rel * (*u_max - *u_min);
        q.bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)L : 1.0;
        // the fine coefficients are final: quantize them on the side stream while the level chain
        // (IPK, coarser levels) runs; writes touch disjoint keys and commute (atomic mask / hist)
        CUDA_CHECK(cudaEventRecord(ctx->event(0), s));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->aux, ctx->event(0), 0));
        quantize_fine(p, coef, q, ctx->aux);
        CUDA_CHECK(cudaEventRecord(ctx->event(1), ctx->aux));
        side = true;
    }
    phase_mark("fine_quantized", s);
    // the rest of transition 0 (IPK + coarse update) and the coarser levels
    {
        if (fwd) thomas_finish_fwd(p, 0, b.t0, c_done, true, s, b.cg, level_ptr(b, p, 1));
        else thomas_all(p, 0, b.t0, s, b.cg, level_ptr(b, p, 1));
    }
    phase_mark("thomas_l0", s);
    const double *DL = coarse_levels_quantize(ctx, p, q, s);
    phase_mark("levels_done", s);
    if (side) CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(1), 0));
    return DL;
}

const double *decompose_quantize(hpdr_ctx *ctx, DevPlan &p, const void *d_in, int dtype, const QuantOut &q,
                                 cudaStream_t s) {
    decompose_fused(ctx, p, d_in, dtype, nullptr, &q, s, 1);   // the finest transition
    phase_mark("level0_done", s);
    return coarse_levels_quantize(ctx, p, q, s);
}

const double *decompose_device(hpdr_ctx *ctx, DevPlan &p, const void *d_in, int dtype, double *coef, cudaStream_t s) {
    const int64_t N = p.n_total;
    const int L = p.host.L;
    if (L > 1 && use_fused(p)) {
        const double *DL = decompose_fused(ctx, p, d_in, dtype, coef, nullptr, s);
        Shape4 shL;
        for (int d = 0; d < 4; d++) shL.n[d] = p.host.cnt[d][L - 1];
        Sel4 none{};
        k_scatter_level<<<rows_grid(shL), 256, 0, s>>>(DL, shL, coef, p.dims, level_map(p, L - 1), none, 0);
        LAUNCH_CHECK();
        return DL;
    }
    LevelBuffers b = level_buffers(ctx, p);
    {
        KPROF("k_to_f64", (double)N * (dtype == 0 ? 12 : 16), s);
        k_to_f64<<<grid_for(N, 256, 148 * 16), 256, 0, s>>>(d_in, dtype, b.lvl0, N);
        LAUNCH_CHECK();
    }
    for (int st_i = 0; st_i + 1 < L; st_i++) {
        const DevStep &st = p.steps[st_i];
        double *F = level_ptr(b, p, st_i);
        double *Dn = level_ptr(b, p, st_i + 1);
        Sel4 sel;
        for (int d = 0; d < 4; d++) sel.s[d] = st.ax[d].active ? st.ax[d].r0 : nullptr;
        const int64_t nf = st.fsh.size(), nc = st.csh.size();
        {
            KPROF("k_gather_coarse", 16.0 * nc, s);
            k_gather_coarse<<<rows_grid(st.csh), 256, 0, s>>>(F, st.fsh, b.cg, st.csh, sel);
            LAUNCH_CHECK();
        }
        interpolate(st, b.cg, b.mc, F, 1, b, s);                       // mc = sub - pred
        {
            KPROF("k_scatter_level", 8.0 * nf + 8.0 * (nf - nc), s);
            k_scatter_level<<<rows_grid(st.fsh), 256, 0, s>>>(b.mc, st.fsh, coef, p.dims, level_map(p, st_i),
                                                              coarse_flags(st), 1);
            LAUNCH_CHECK();
        }
        const double *corr = correction(st, b.mc, b, s);
        {
            KPROF("k_add", 24.0 * nc, s);
            k_add<<<grid_for(nc, 256, 148 * 16), 256, 0, s>>>(b.cg, corr, Dn, nc);   // coarse + corr
            LAUNCH_CHECK();
        }
    }
    // coarsest nodal values to their finest positions
    Shape4 shL;
    for (int d = 0; d < 4; d++) shL.n[d] = p.host.cnt[d][L - 1];
    const double *DL = level_ptr(b, p, L - 1);
    if (L == 1) {
        CUDA_CHECK(cudaMemcpyAsync(coef, b.lvl0, N * 8, cudaMemcpyDeviceToDevice, s));
        return b.lvl0;
    }
    Sel4 none{};
    k_scatter_level<<<rows_grid(shL), 256, 0, s>>>(DL, shL, coef, p.dims, level_map(p, L - 1), none, 0);
    LAUNCH_CHECK();
    return DL;
}

double *recompose_device(hpdr_ctx *ctx, DevPlan &p, const double *coef, cudaStream_t s) {
    LevelBuffers b = level_buffers(ctx, p);
    const int L = p.host.L;
    const int64_t N = p.n_total;
    if (L == 1) {
        CUDA_CHECK(cudaMemcpyAsync(b.lvl0, coef, N * 8, cudaMemcpyDeviceToDevice, s));
        return b.lvl0;
    }
    Shape4 shL;
    for (int d = 0; d < 4; d++) shL.n[d] = p.host.cnt[d][L - 1];
    Sel4 none{};
    k_gather_level<<<rows_grid(shL), 256, 0, s>>>(coef, p.dims, level_map(p, L - 1), none, level_ptr(b, p, L - 1),
                                                  shL, 0);
    LAUNCH_CHECK();
    for (int st_i = L - 2; st_i >= 0; st_i--) {
        const DevStep &st = p.steps[st_i];
        double *F = level_ptr(b, p, st_i);
        double *Dc = level_ptr(b, p, st_i + 1);
        const int64_t nf = st.fsh.size(), nc = st.csh.size();
        {
            KPROF("k_gather_level", 8.0 * (nf - nc) + 8.0 * nf, s);
            k_gather_level<<<rows_grid(st.fsh), 256, 0, s>>>(coef, p.dims, level_map(p, st_i), coarse_flags(st), b.mc,
                                                             st.fsh, 1);
            LAUNCH_CHECK();
        }
        const double *corr = correction(st, b.mc, b, s);
        {
            KPROF("k_sub", 24.0 * nc, s);
            k_sub<<<grid_for(nc, 256, 148 * 16), 256, 0, s>>>(Dc, corr, b.cg, nc);   // coarse - corr
            LAUNCH_CHECK();
        }
        interpolate(st, b.cg, F, b.mc, 2, b, s);                                    // pred + mc
    }
    return b.lvl0;
}

int64_t z0_elems(const DevPlan &p, int st_i) {
    const DevStep &st = p.steps[st_i];
    return (int64_t)(st.ax[1].active ? st.csh.n[1] : st.fsh.n[1]) * st.fsh.n[2] * st.fsh.n[3];
}

void thomas_all(const DevPlan &p, int st_i, double *T, cudaStream_t s, const double *add_base, double *add_dst) {
    const DevStep &st = p.steps[st_i];
    Shape4 sh = st.csh;
    Epi epi;
    epi.base = add_base;
    epi.dst = add_dst;
    static const bool no_small = getenv("HPDR_THOMAS_NOSMALL") != nullptr;
    if (!no_small && sh.size() <= kThomasSmallMax) {
        static bool attr = false;
        if (!attr) {
            for (auto f : {k_thomas_small<false>, k_thomas_small<true>})
                CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (kThomasSmallMax + kThomasSmallTabs) * 8));
            attr = true;
        }
        AxesArg A;
        for (int a = 0; a < 4; a++) A.ax[a] = st.ax[a];
        int tab = 0;
        for (int a = 0; a < 4; a++)
            if (st.ax[a].active) tab += 4 * st.ax[a].nc;
        const int stage = tab <= kThomasSmallTabs ? 1 : 0;
        const size_t smem = (size_t)(sh.size() + (stage ? tab : 0)) * 8;
        KPROF("k_thomas_small", (add_dst ? 24.0 : 16.0) * sh.size(), s);
        if (add_dst) k_thomas_small<true><<<1, 512, smem, s>>>(T, sh, A, epi, stage);
        else k_thomas_small<false><<<1, 512, smem, s>>>(T, sh, A, epi, stage);
        LAUNCH_CHECK();
        return;
    }
    int last = -1;
    for (int a = 0; a < 4; a++)
        if (st.ax[a].active) last = a;
    for (int a = 0; a < 4; a++)
        if (st.ax[a].active) thomas(T, sh, a, st.ax[a], s, a == last ? epi : Epi{});
    if (last < 0 && add_dst) {   // no active axis: the correction is the right-hand side itself
        const int64_t nc = sh.size();
        KPROF("k_add", 24.0 * nc, s);
        k_add<<<grid_for(nc, 256, 148 * 16), 256, 0, s>>>(add_base, T, add_dst, nc);
        LAUNCH_CHECK();
    }
}

bool thomas_plane_split(const DevPlan &p, int st_i) {
    static const bool off = getenv("HPDR_NO_PLANE_SPLIT") != nullptr;
    const DevStep &st = p.steps[st_i];
    return !off && p.dims.n[0] == 1 && !st.ax[0].active && st.ax[1].active && st.csh.size() > kThomasSmallMax;
}

void thomas_plane_axis(const DevPlan &p, int st_i, double *T, cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    thomas(T, st.csh, 1, st.ax[1], s);
}

void thomas_in_planes(const DevPlan &p, int st_i, double *T, int c_lo, int c_hi, cudaStream_t s) {
    if (c_hi <= c_lo) return;
    const DevStep &st = p.steps[st_i];
    Shape4 sub = st.csh;
    sub.n[1] = c_hi - c_lo;   // transform.py:259-260: the in-plane axes after the plane axis, per plane
    double *T0 = T + (int64_t)c_lo * st.csh.n[2] * st.csh.n[3];
    for (int a = 2; a < 4; a++)
        if (st.ax[a].active) thomas(T0, sub, a, st.ax[a], s);
}

bool thomas_fwd_stream(const DevPlan &p, int st_i) {
    static const bool off = getenv("HPDR_NO_FWD_STREAM") != nullptr;
    const DevStep &st = p.steps[st_i];
    return !off && p.dims.n[0] == 1 && !st.ax[0].active && st.ax[1].active && st.csh.size() > kThomasSmallMax;
}

void thomas_plane_fwd(const DevPlan &p, int st_i, double *T, int c_lo, int c_hi, cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const DevAxis &ax = st.ax[1];
    const int lo = std::max(c_lo, 1);
    c_hi = std::min(c_hi, (int)ax.nc);
    if (c_hi <= lo) return;
    int64_t outer, inner;
    view(st.csh, 1, outer, inner);
    const int64_t lines = outer * inner;
    KPROF("k_thomas_fwd", 8.0 * lines * (c_hi - lo), s);
    k_thomas_reg<8, false, 1><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(T, outer, ax.nc, inner, ax.tw, ax.tb, ax.tu,
                                                                             ax.tr, Epi{}, lo, c_hi);
    LAUNCH_CHECK();
}

void thomas_finish_fwd(const DevPlan &p, int st_i, double *T, int f_done, bool in_planes, cudaStream_t s,
                       const double *add_base, double *add_dst) {
    const DevStep &st = p.steps[st_i];
    const DevAxis &ax = st.ax[1];
    thomas_plane_fwd(p, st_i, T, f_done, ax.nc, s);
    int last = 1;
    if (in_planes)
        for (int a = 2; a < 4; a++)
            if (st.ax[a].active) last = a;
    Epi epi;
    epi.base = add_base;
    epi.dst = add_dst;
    int64_t outer, inner;
    view(st.csh, 1, outer, inner);
    const int64_t lines = outer * inner;
    KPROF("k_thomas_bwd", (last == 1 && add_dst ? 16.0 : 8.0) * lines * ax.nc, s);
    if (last == 1 && add_dst)
        k_thomas_reg<8, true, 2><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(T, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                                ax.tu, ax.tr, epi);
    else
        k_thomas_reg<8, false, 2><<<grid_for(lines, 128, 148 * 64), 128, 0, s>>>(T, outer, ax.nc, inner, ax.tw, ax.tb,
                                                                                 ax.tu, ax.tr, Epi{});
    LAUNCH_CHECK();
    if (in_planes)
        for (int a = 2; a < 4; a++)
            if (st.ax[a].active) thomas(T, st.csh, a, st.ax[a], s, a == last ? epi : Epi{});
}

void recompose_into(hpdr_ctx *ctx, DevPlan &p, const double *coef, void *out, int out_dtype, cudaStream_t s,
                    void *host_out, const double *T0_pre, cudaEvent_t ev_pre, bool t0_plane_axis_only,
                    const double *T1_pre, cudaEvent_t ev1_pre) {
    const int L = p.host.L;
    if (L == 1 || !use_fused(p)) {
        const double *rec = recompose_device(ctx, p, coef, s);
        cast_output(rec, out, out_dtype, p.n_total, s);
        if (host_out) {
            static const int isz[7] = {4, 8, 4, 8, 4, 8, 1};
            if (classify(host_out) == MemKind::Host) stage_d2h(ctx, host_out, out, p.n_total * isz[out_dtype], s);
            else CUDA_CHECK(cudaMemcpyAsync(host_out, out, p.n_total * isz[out_dtype], cudaMemcpyDeviceToHost, s));
        }
        return;
    }
    const bool direct = out_dtype == 0 || out_dtype == 1;
    LevelBuffers b = fused_buffers(ctx, p);
    if (!direct) b.lvl0 = (double *)ctx->dbuf("lvl0", p.n_total * 8);
    double *Z0 = b.mc;
    Shape4 shL;
    for (int d = 0; d < 4; d++) shL.n[d] = p.host.cnt[d][L - 1];
    Sel4 none{};
    // transitions tiny .. L-2 (the small end) run in one block on the main stream
    const int tiny = tiny_start(p, 1);
    const int top = tiny >= 1 ? tiny : L - 1;   // chain below handles transitions top-1 .. 0
    if (tiny < 1) {
        k_gather_level<<<rows_grid(shL), 256, 0, s>>>(coef, p.dims, level_map(p, L - 1), none,
                                                      level_ptr(b, p, L - 1), shL, 0);
        LAUNCH_CHECK();
    }
    // A level's correction depends only on its own coefficients (transform.py:342-345), so the
    // finest one -- the bulk of the correction work -- runs on the side stream while the coarser
    // levels are recomposed; only coarse - corr of the finest transition waits for it.
    const double *T0f = b.t0;
    const bool side = L > 2;
    cudaEvent_t ev_side = ctx->event(1);
    if (side && T0_pre) {
        T0f = T0_pre;
        ev_side = ev_pre;
    } else if (side) {
        const DevStep &st = p.steps[0];
        double *Z0f = (double *)ctx->dbuf("z0f", z0_elems(p, 0) * 8);
        double *T = (double *)ctx->dbuf("t0f", st.csh.size() * 8);
        T0f = T;
        CUDA_CHECK(cudaEventRecord(ctx->event(0), s));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->aux_hi, ctx->event(0), 0));
        fused_pass1_recompose(p, 0, coef, Z0f, ctx->aux_hi);
        fused_pass2(p, 0, Z0f, T, ctx->aux_hi);
        if (direct && host_out && thomas_plane_split(p, 0)) {   // in-plane sweeps follow the output slabs
            thomas_plane_axis(p, 0, T, ctx->aux_hi);
            t0_plane_axis_only = true;
        } else {
            thomas_all(p, 0, T, ctx->aux_hi);
        }
        CUDA_CHECK(cudaEventRecord(ev_side, ctx->aux_hi));
    }
    // The coarser levels' corrections are independent of each other too: compute them up front,
    // round-robin on the side streams (they are small, latency-bound launches), so the level chain
    // itself is only coarse - corr and pred + mc per level.
    std::vector<const double *> Tl(L, nullptr);
    std::vector<int> ev_l(L, -1);
    if (L > 2) {
        int64_t zc = 0, tc = 0;
        for (int st_i = 1; st_i < top; st_i++) {
            zc += (z0_elems(p, st_i) + 31) & ~int64_t(31);
            tc += (p.steps[st_i].csh.size() + 31) & ~int64_t(31);
        }
        double *zarena = (double *)ctx->dbuf("z0c", std::max<int64_t>(zc, 1) * 8);
        double *tarena = (double *)ctx->dbuf("t0c", std::max<int64_t>(tc, 1) * 8);
        // event ids: 199 / 200 + level (distinct from the streamed decode's and the slab loop's)
        CUDA_CHECK(cudaEventRecord(ctx->event(199), s));   // coef ready
        // side[0] still carries the streamed decode's level-1 solve when T1_pre is set: the coarser
        // levels (the head of the chain) go round-robin on the other three side streams
        const int k0 = T1_pre ? 1 : 0, nk = 4 - k0;
        int k = 0;
        for (int st_i = top - 1; st_i >= 1; st_i--, k++) {
            if (st_i == 1 && T1_pre) continue;   // computed by the caller (streamed decode)
            cudaStream_t x = ctx->side[k0 + k % nk];
            if (k < nk) CUDA_CHECK(cudaStreamWaitEvent(x, ctx->event(199), 0));
            double *Zl = zarena, *T = tarena;
            zarena += (z0_elems(p, st_i) + 31) & ~int64_t(31);
            tarena += (p.steps[st_i].csh.size() + 31) & ~int64_t(31);
            fused_pass1_recompose(p, st_i, coef, Zl, x);
            fused_pass2(p, st_i, Zl, T, x);
            thomas_all(p, st_i, T, x);
            Tl[st_i] = T;
            ev_l[st_i] = st_i;
            CUDA_CHECK(cudaEventRecord(ctx->event(EvLevel, st_i), x));
        }
    }
    if (tiny >= 1) tiny_recompose(p, tiny, coef, level_ptr(b, p, tiny), s);
    phase_mark("tiny", s);
    static const char *kLvlMark[8] = {"final0", "final1", "final2", "final3", "final4", "final5", "final6", "final7"};
    // Host output in slabs: transition 1's final pass (the level-1 grid the finest slabs interpolate
    // from) is cut into plane ranges too, each launched just ahead of the first slab that reads it,
    // so the first D2H does not wait for the whole level-1 grid.
    static const bool no_defer1 = getenv("HPDR_NO_DEFER_L1") != nullptr;
    const bool defer1 = !no_defer1 && direct && host_out && top >= 2 && p.dims.n[0] == 1 &&
                        p.host.steps[0].ax[1].active;
    const double *Dc1 = nullptr, *T1s = nullptr;
    for (int st_i = top - 1; st_i >= 0; st_i--) {
        const DevStep &st = p.steps[st_i];
        double *Dc = level_ptr(b, p, st_i + 1);
        const double *T = b.t0;
        if (st_i == 0 && side) {
            T = T0f;
            CUDA_CHECK(cudaStreamWaitEvent(s, ev_side, 0));
        } else if (st_i == 1 && T1_pre) {
            T = T1_pre;
            CUDA_CHECK(cudaStreamWaitEvent(s, ev1_pre, 0));
            phase_mark("t1_ready", s);
        } else if (Tl[st_i]) {
            T = Tl[st_i];
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(EvLevel, ev_l[st_i]), 0));
        } else {
            fused_pass1_recompose(p, st_i, coef, Z0, s);
            fused_pass2(p, st_i, Z0, b.t0, s);
            thomas_all(p, st_i, b.t0, s);
        }
        // coarse - corr is formed inside the final level kernel as it reads the coarse values
        if (st_i == 1 && defer1) {   // transition 1's output follows the finest slabs (slab loop below)
            Dc1 = Dc;
            T1s = T;
            continue;
        }
        if (st_i == 0) phase_mark("coarse_levels_done", s);
        if (st_i == 0 && direct && host_out) {
            // finest level in dim-0 slabs; each slab's D2H (copy stream) overlaps the next slab
            const int n0 = (int)st.fsh.n[1];
            const int64_t plane_bytes = st.fsh.n[2] * st.fsh.n[3] * (out_dtype == 0 ? 4 : 8);
            const int64_t target = std::min<int64_t>(32LL << 20, std::max<int64_t>(1LL << 20, (int64_t)n0 * plane_bytes / 4));
            int chunk = (int)std::max<int64_t>(4, (target + plane_bytes - 1) / std::max<int64_t>(plane_bytes, 1));
            chunk = std::min(chunk, n0);
            CUDA_CHECK(cudaEventRecord(ctx->event(0), ctx->d2h));
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(0), 0));   // previous call's copies are done
            // every slab is launched first; its D2H follows its event (pageable destinations through the
            // pinned staging ring, host-blocking, while the GPU runs the later slabs)
            const bool pageable_out = classify(host_out) == MemKind::Host;
            int nslab = 0;
            int c_done = 0;   // coarse planes whose in-plane solves are done (t0_plane_axis_only)
            int c1_done = 0;  // level-1 planes written (defer1)
            const int nc0 = (int)st.csh.n[1];
            for (int a = 0, k = 0; a < n0; a += chunk, k++, nslab++) {
                const int e = std::min(n0, a + chunk);
                const AxisTables &h0 = p.host.steps[0].ax[1];
                // the coarse planes this slab's fine planes read
                const int c_need = (e >= n0 || !h0.active) ? nc0 : std::max(h0.pa[e - 1], h0.pb[e - 1]) + 1;
                if (defer1 && c_need > c1_done) {
                    const int c1 = std::min(nc0, (c_need + 1) & ~1);
                    fused_final(p, 1, Dc1, coef, Dc, 1, s, c1_done, c1, T1s);
                    c1_done = c1;
                    if (k == 0) phase_mark("final1_first", s);
                }
                if (t0_plane_axis_only) {
                    thomas_in_planes(p, 0, const_cast<double *>(T), c_done, c_need, s);
                    c_done = std::max(c_done, c_need);
                }
                fused_final(p, 0, Dc, coef, out, out_dtype, s, a, e, T);
                CUDA_CHECK(cudaEventRecord(ctx->event(EvSlabOut, k), s));
            }
            if (pageable_out) {   // one continuous pass of the staging ring, slab events releasing the chunks
                std::vector<StageRange> rs;
                for (int a = 0, k = 0; k < nslab; a += chunk, k++)
                    rs.push_back({(size_t)a * plane_bytes, (size_t)std::min(n0, a + chunk) * plane_bytes,
                                  ctx->event(EvSlabOut, k)});
                stage_d2h_ranges(ctx, (char *)host_out, (const char *)out, rs, ctx->d2h);
            } else {
                for (int a = 0, k = 0; k < nslab; a += chunk, k++) {
                    const int e = std::min(n0, a + chunk);
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(EvSlabOut, k), 0));
                    CUDA_CHECK(cudaMemcpyAsync((char *)host_out + a * plane_bytes, (const char *)out + a * plane_bytes,
                                               (e - a) * plane_bytes, cudaMemcpyDeviceToHost, ctx->d2h));
                }
            }
            CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
        } else if (st_i == 0 && direct) {
            fused_final(p, st_i, Dc, coef, out, out_dtype, s, 0, -1, T);
        } else {
            fused_final(p, st_i, Dc, coef, level_ptr(b, p, st_i), 1, s, 0, -1, T);
            if (st_i < 8) phase_mark(kLvlMark[st_i], s);
        }
    }
    if (!direct) cast_output(b.lvl0, out, out_dtype, p.n_total, s);
    if (host_out && !direct) {
        static const int isz[7] = {4, 8, 4, 8, 4, 8, 1};
        if (classify(host_out) == MemKind::Host) stage_d2h(ctx, host_out, out, p.n_total * isz[out_dtype], s);
        else CUDA_CHECK(cudaMemcpyAsync(host_out, out, p.n_total * isz[out_dtype], cudaMemcpyDeviceToHost, s));
    }
}

void cast_output(const double *src, void *dst, int dtype, int64_t n, cudaStream_t s) {
    unsigned g = grid_for(n, 256, 148 * 16);
    static const int isz[7] = {4, 8, 4, 8, 4, 8, 1};
    KPROF("k_cast", (double)n * (8 + isz[dtype < 0 || dtype > 6 ? 6 : dtype]), s);
    switch (dtype) {
        case 0: k_cast<float><<<g, 256, 0, s>>>(src, (float *)dst, n); break;
        case 1: CUDA_CHECK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, s)); return;
        case 2: k_cast<uint32_t><<<g, 256, 0, s>>>(src, (uint32_t *)dst, n); break;
        case 3: k_cast<uint64_t><<<g, 256, 0, s>>>(src, (uint64_t *)dst, n); break;
        case 4: k_cast<int32_t><<<g, 256, 0, s>>>(src, (int32_t *)dst, n); break;
        case 5: k_cast<int64_t><<<g, 256, 0, s>>>(src, (int64_t *)dst, n); break;
        default: k_cast<uint8_t><<<g, 256, 0, s>>>(src, (uint8_t *)dst, n); break;
    }
    LAUNCH_CHECK();
}

}  // namespace hpdr

extern "C" int hpdr_selftest_div(uint64_t n, uint64_t seed, uint64_t *mismatches, uint64_t *fallbacks) {
    try {
        unsigned long long *d = nullptr;
        CUDA_CHECK(cudaMalloc(&d, 16));
        CUDA_CHECK(cudaMemset(d, 0, 16));
        hpdr::k_selftest_div<<<148 * 8, 256>>>(n, seed, d, d + 1);
        CUDA_CHECK(cudaGetLastError());
        unsigned long long h[2];
        CUDA_CHECK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
        CUDA_CHECK(cudaFree(d));
        *mismatches = h[0];
        *fallbacks = h[1];
        return HPDR_OK;
    } catch (const hpdr::Error &e) {
        hpdr::set_error(e.code, e.msg, e.bit_offset);
        return e.code;
    }
}
