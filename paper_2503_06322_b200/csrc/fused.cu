// fused.cu -- fused level kernels for ranks 1..3 (a 3-D view; rank-4 fields take the
// per-axis path in transform.cu).
//
// One decomposition transition (transform.py:306-315) becomes
//   pass 1   k_level_pass1   residual mc = F - P(F) (GPK, nested lerps in axis order 0,1,2)
//                            -> coefficient write, coarse-node gather, and the axis-0
//                            mass-multiply + restriction (LPK, transform.py:206-203) as a
//                            register march along axis 0
//   pass 2   k_level_pass2   axis-1 LPK march + axis-2 LPK across the block (shared memory)
//   IPK      Thomas sweeps (transform.cu) and coarse + corr
// and recomposition (transform.py:337-347) mirrors it with pass 1 reading mc from the
// coefficients and k_level_final writing pred + mc (or the output dtype at the finest level).
// Every value is produced with the reference's operation order (explicit _rn intrinsics), so
// the result is bit-identical to the per-axis path and to numpy.
#include "fused.cuh"

namespace hpdr {

namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double lerp(double va, double vb, double t) { return dadd(va, dmul(t, dsub(vb, va))); }

template <typename T>
__device__ __forceinline__ double ld(const T *p) { return (double)__ldg(p); }

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
    const int a = ax.pa[j], b = ax.pb[j];
    r.fo = b >= 0;
    r.ca = a;
    r.cb = r.fo ? b : a;
    r.fa = ax.r0[a];
    r.fb = ax.r0[r.cb];
    r.t = r.fo ? ax.pt[j] : 0.0;
    return r;
}

// Sliding mass-multiply + restriction along the march axis (transform.py:206-226 then :181-203):
//   y(j) = (md_j x_j + ml_j x_{j-1}) + mu_j x_{j+1}
//   z(c) = (y(r0_c) + wr_c y(rr_c)) + wl_c y(rl_c)
struct March {
    double m1, m2;        // x(j-1), x(j-2)
    double ya, yb, yc;    // y(k-2), y(k-1), y(k)
    int c;                // next coarse output
};

// Push x(j); emits every z(c) that became computable through emit(c, z).
template <class Emit>
__device__ __forceinline__ void march_push(March &M, const DevAxis &ax, int n, int j, int j_start, double x, int c_hi,
                                           Emit &&emit) {
    auto try_y = [&](int k, double xk, double xkm1, double xkp1, bool has_up) {
        double v = dmul(ax.md[k], xk);
        if (k >= 1) v = dadd(v, dmul(ax.ml[k], xkm1));
        if (has_up) v = dadd(v, dmul(ax.mu[k], xkp1));
        M.ya = M.yb;
        M.yb = M.yc;
        M.yc = v;
        while (M.c < c_hi) {
            const int r0 = ax.r0[M.c], rr = ax.rr[M.c], rl = ax.rl[M.c];
            const int need = rr >= 0 ? rr : r0;
            if (need != k) break;
            double z;
            if (rr >= 0) {
                z = dadd(M.yb, dmul(ax.wr[M.c], M.yc));
                if (rl >= 0) z = dadd(z, dmul(ax.wl[M.c], M.ya));
            } else {
                z = M.yc;
                if (rl >= 0) z = dadd(z, dmul(ax.wl[M.c], M.yb));
            }
            emit(M.c, z);
            M.c++;
        }
    };
    // y(j-1) needs x(j-2) unless j-1 == 0
    if (j >= 1 && (j - 1 == 0 || j - 2 >= j_start)) try_y(j - 1, M.m1, M.m2, x, true);
    if (j == n - 1 && (j == 0 || j - 1 >= j_start)) try_y(j, x, M.m1, 0.0, false);
    M.m2 = M.m1;
    M.m1 = x;
}

// Coarse-plane range of slab z out of nz along an axis with (active) tables.
__device__ __forceinline__ void slab_range(int nc, int nz, int z, int &lo, int &hi) {
    const int base = nc / nz, rem = nc % nz;
    lo = z * base + min(z, rem);
    hi = lo + base + (z < rem ? 1 : 0);
}

// ---------------------------------------------------------------------------------- pass 1
// MODE 0 (decompose):  mc = F - P(F); coef[fine-only] = mc; Cg[coarse] = F; Z0 = R0M0(mc)
// MODE 1 (recompose):  mc = coef at fine-only nodes, 0 at coarse nodes; Z0 = R0M0(mc)
// MODE 2 (decompose with quantize-on-write): as MODE 0 but fine-only nodes are quantized
//   straight into keys / outlier mask / histogram (quantize.py:73-84) instead of coef.
// Z0 = mc along axis 0 when that axis is inactive at this transition.
constexpr int kSmemHist = 4096;

template <int MODE, bool A0, bool A1, bool A2, typename TIn>
__global__ void __launch_bounds__(256) k_level_pass1(const TIn *__restrict__ F, int n0, int n1, int n2, DevAxis ax0,
                                                     DevAxis ax1, DevAxis ax2, LevelMap lm, double *__restrict__ coef,
                                                     const double *__restrict__ coef_in, double *__restrict__ Z0,
                                                     double *__restrict__ Cg, QuantOut q) {
    __shared__ uint32_t sh_hist[MODE == 2 ? kSmemHist : 1];
    const bool sh_ok = MODE == 2 && q.dict <= kSmemHist;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) sh_hist[k] = 0;
    if (MODE == 2) __syncthreads();
    const int j2 = blockIdx.x * 32 + threadIdx.x;
    const int j1 = blockIdx.y * 8 + threadIdx.y;
    const bool act = j1 < n1 && j2 < n2;
    const int nc0 = A0 ? ax0.nc : n0;
    int c_lo, c_hi;
    slab_range(nc0, gridDim.z, blockIdx.z, c_lo, c_hi);
    int fl = 0;
    if (act && c_lo < c_hi) {
        const Nb b1 = neighbours<A1>(ax1, j1), b2 = neighbours<A2>(ax2, j2);
        const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
        int j_start, j_end, own_lo, own_hi;
        if (A0) {
            j_start = max(0, ax0.r0[c_lo] - 2);
            j_end = min(n0 - 1, ax0.r0[c_hi - 1] + 2);
            own_lo = c_lo == 0 ? 0 : ax0.r0[c_lo];
            own_hi = c_hi == nc0 ? n0 : ax0.r0[c_hi];
        } else {
            j_start = c_lo;
            j_end = c_hi - 1;
            own_lo = c_lo;
            own_hi = c_hi;
        }
        const int64_t plane = (int64_t)n1 * n2;
        const int64_t col = (int64_t)j1 * n2 + j2;
        const int64_t fcol = ((int64_t)lm.m1[j1]) * lm.D2 + lm.m2[j2];
        const int64_t fplane = lm.D1 * lm.D2;
        March M;
        M.m1 = M.m2 = M.ya = M.yb = M.yc = 0.0;
        M.c = c_lo;
        auto emit = [&](int c, double z) { Z0[(int64_t)c * plane + col] = z; };
        for (int j = j_start; j <= j_end; j++) {
            const Nb b0 = neighbours<A0>(ax0, j);
            const bool coarse_node = !b0.fo && !b1.fo && !b2.fo;
            const int64_t f = (int64_t)lm.m0[j] * fplane + fcol;
            double mc;
            if (MODE != 1) {
                // GPK: P0 along axis 0 at the corner columns, then P1 along axis 1, then P2 along axis 2
                auto P0 = [&](int y1, int x2) -> double {
                    const double va = ld(F + (int64_t)b0.fa * plane + (int64_t)y1 * n2 + x2);
                    if (!b0.fo) return va;
                    const double vb = ld(F + (int64_t)b0.fb * plane + (int64_t)y1 * n2 + x2);
                    return lerp(va, vb, b0.t);
                };
                auto P1 = [&](int x2) -> double {
                    const double va = P0(b1.fa, x2);
                    if (!b1.fo) return va;
                    return lerp(va, P0(b1.fb, x2), b1.t);
                };
                double pred = P1(b2.fa);
                if (b2.fo) pred = lerp(pred, P1(b2.fb), b2.t);
                const double own = ld(F + (int64_t)j * plane + col);
                mc = dsub(own, pred);
                if (j >= own_lo && j < own_hi) {
                    if (coarse_node) {
                        const int c0 = A0 ? b0.ca : j;
                        Cg[((int64_t)c0 * nc1 + b1.ca) * nc2 + b2.ca] = own;
                    } else if (MODE == 0) {
                        coef[f] = mc;
                    } else {
                        long long b = 0;
                        if (!isfinite(mc)) {
                            fl |= 1;
                        } else {
                            const double sc = mc / q.bin;                 // IEEE division (quantize.py:73)
                            if (fabs(sc) >= 4611686018427387904.0) fl |= 2;
                            else b = (long long)rint(sc);                 // half to even (:76)
                        }
                        if (b >= q.half || -b >= q.half) {                 // outlier (:80-83)
                            q.obins[f] = b;
                            atomicOr(&q.omask[f >> 5], 1u << (f & 31));
                            b = 0;
                        }
                        const uint32_t key = (uint32_t)(((unsigned long long)b << 1) ^ (unsigned long long)(b >> 63));
                        q.keys[f] = key;
                        if (sh_ok) atomicAdd(&sh_hist[key], 1u);
                        else atomicAdd(&q.hist[key], 1ULL);
                    }
                }
            } else {
                mc = coarse_node ? 0.0 : coef_in[f];
            }
            if (A0) march_push(M, ax0, n0, j, j_start, mc, c_hi, emit);
            else Z0[(int64_t)j * plane + col] = mc;
        }
    }
    if (MODE == 2) {
        if (fl) atomicOr(q.flags, fl);
        __syncthreads();
        if (sh_ok)
            for (uint32_t k = tid; k < q.dict; k += 256) {
                const uint32_t c = sh_hist[k];
                if (c) atomicAdd(&q.hist[k], (unsigned long long)c);
            }
    }
}

// Coarsest nodes: raw values are checked (finite, bin limit) like every coefficient, then get key 0.
__global__ void k_quantize_coarsest(const double *__restrict__ vals, const long long *__restrict__ idx, int n,
                                    QuantOut q) {
    const int k = threadIdx.x;
    if (k < n) {
        const double v = vals[k];
        int fl = 0;
        if (!isfinite(v)) fl |= 1;
        else if (fabs(v / q.bin) >= 4611686018427387904.0) fl |= 2;
        if (fl) atomicOr(q.flags, fl);
        q.keys[idx[k]] = 0u;
    }
    if (k == 0) atomicAdd(&q.hist[0], (unsigned long long)n);
}

// ---------------------------------------------------------------------------------- pass 2
// Z0 (m0, n1, n2) -> B (m0, nc1, nc2): axis-1 LPK as a march, axis-2 LPK across the block.
constexpr int kP2Threads = 256;
constexpr int kP2Out = (kP2Threads - 4) / 2;   // coarse outputs along axis 2 per block

template <bool A1, bool A2>
__global__ void __launch_bounds__(kP2Threads) k_level_pass2(const double *__restrict__ Z0, int m0, int n1, int n2,
                                                            DevAxis ax1, DevAxis ax2, double *__restrict__ B,
                                                            int slabs1) {
    __shared__ double sw[kP2Threads];
    __shared__ double sy[kP2Threads];
    const int t = threadIdx.x;
    const int p = blockIdx.y;
    const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
    int c2_lo = 0, c2_cnt = 0, base;
    if (A2) {
        c2_lo = blockIdx.x * kP2Out;
        c2_cnt = min(kP2Out, nc2 - c2_lo);
        base = ax2.r0[c2_lo] - 2;
    } else {
        base = blockIdx.x * kP2Threads;
    }
    const int j2 = base + t;
    const bool in = j2 >= 0 && j2 < n2;
    int c_lo, c_hi;
    slab_range(nc1, slabs1, blockIdx.z, c_lo, c_hi);
    if (c_lo >= c_hi) return;   // uniform across the block
    const double *zp = Z0 + (int64_t)p * n1 * n2;
    double *bp = B + (int64_t)p * nc1 * nc2;
    auto out_row = [&](int c1, double w) {
        if (!A2) {
            if (in) bp[(int64_t)c1 * nc2 + j2] = w;
            return;
        }
        sw[t] = w;
        __syncthreads();
        double y = 0.0;
        if (in) {
            y = dmul(ax2.md[j2], sw[t]);
            if (j2 >= 1 && t >= 1) y = dadd(y, dmul(ax2.ml[j2], sw[t - 1]));
            if (j2 + 1 < n2 && t + 1 < kP2Threads) y = dadd(y, dmul(ax2.mu[j2], sw[t + 1]));
        }
        sy[t] = y;
        __syncthreads();
        if (t < c2_cnt) {
            const int c2 = c2_lo + t;
            const int r0 = ax2.r0[c2] - base, rr = ax2.rr[c2], rl = ax2.rl[c2];
            double z = sy[r0];
            if (rr >= 0) z = dadd(z, dmul(ax2.wr[c2], sy[rr - base]));
            if (rl >= 0) z = dadd(z, dmul(ax2.wl[c2], sy[rl - base]));
            bp[(int64_t)c1 * nc2 + c2] = z;
        }
        __syncthreads();
    };
    if (!A1) {
        for (int j1 = c_lo; j1 < c_hi; j1++) out_row(j1, in ? ld(zp + (int64_t)j1 * n2 + j2) : 0.0);
        return;
    }
    const int j_start = max(0, ax1.r0[c_lo] - 2);
    const int j_end = min(n1 - 1, ax1.r0[c_hi - 1] + 2);
    March M;
    M.m1 = M.m2 = M.ya = M.yb = M.yc = 0.0;
    M.c = c_lo;
    for (int j = j_start; j <= j_end; j++) {
        const double x = in ? ld(zp + (int64_t)j * n2 + j2) : 0.0;
        march_push(M, ax1, n1, j, j_start, x, c_hi, out_row);
    }
}

// ---------------------------------------------------------------------------------- final
// Recompose output of one transition: D(j) = P(cv)(j) + mc(j) (transform.py:346-347), P the
// nested lerps over the corrected coarse values cv (nc0, nc1, nc2), mc from the coefficients.
template <bool A0, bool A1, bool A2, typename TOut>
__global__ void __launch_bounds__(256) k_level_final(const double *__restrict__ cv, int n0, int n1, int n2,
                                                     DevAxis ax0, DevAxis ax1, DevAxis ax2, LevelMap lm,
                                                     const double *__restrict__ coef, TOut *__restrict__ D) {
    const int j2 = blockIdx.x * 32 + threadIdx.x;
    const int j1 = blockIdx.y * 8 + threadIdx.y;
    if (j1 >= n1 || j2 >= n2) return;
    const Nb b1 = neighbours<A1>(ax1, j1), b2 = neighbours<A2>(ax2, j2);
    const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
    int lo, hi;
    slab_range(n0, gridDim.z, blockIdx.z, lo, hi);
    const int64_t col = (int64_t)j1 * n2 + j2;
    const int64_t fcol = ((int64_t)lm.m1[j1]) * lm.D2 + lm.m2[j2];
    const int64_t cplane = (int64_t)nc1 * nc2;
    for (int j = lo; j < hi; j++) {
        const Nb b0 = neighbours<A0>(ax0, j);
        auto P0 = [&](int y1, int x2) -> double {
            const double va = cv[(int64_t)b0.ca * cplane + (int64_t)y1 * nc2 + x2];
            if (!b0.fo) return va;
            return lerp(va, cv[(int64_t)b0.cb * cplane + (int64_t)y1 * nc2 + x2], b0.t);
        };
        auto P1 = [&](int x2) -> double {
            const double va = P0(b1.ca, x2);
            if (!b1.fo) return va;
            return lerp(va, P0(b1.cb, x2), b1.t);
        };
        double pred = P1(b2.ca);
        if (b2.fo) pred = lerp(pred, P1(b2.cb), b2.t);
        const bool coarse_node = !b0.fo && !b1.fo && !b2.fo;
        const double mc = coarse_node ? 0.0 : __ldg(coef + (int64_t)lm.m0[j] * lm.D1 * lm.D2 + fcol);
        D[(int64_t)j * n1 * n2 + col] = (TOut)dadd(pred, mc);
    }
}

int slabs_for(int64_t cols, int planes) {
    const int64_t target = 148LL * 2048 * 2;
    int64_t s = (target + cols - 1) / std::max<int64_t>(cols, 1);
    return (int)std::max<int64_t>(1, std::min<int64_t>(s, std::max(planes, 1)));
}

template <int MODE, typename TIn>
void launch_pass1(int act, const TIn *F, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1,
                  const DevAxis &a2, const LevelMap &lm, double *coef, const double *coef_in, double *Z0, double *Cg,
                  const QuantOut &q, cudaStream_t s) {
    const int planes = (act & 1) ? a0.nc : n0;
    dim3 grid((n2 + 31) / 32, (n1 + 7) / 8, slabs_for((int64_t)n1 * n2, planes));
    dim3 block(32, 8);
#define P1L(M)                                                                                                     \
    case M:                                                                                                        \
        k_level_pass1<MODE, (M & 1) != 0, (M & 2) != 0, (M & 4) != 0, TIn><<<grid, block, 0, s>>>(              \
            F, n0, n1, n2, a0, a1, a2, lm, coef, coef_in, Z0, Cg, q);                                              \
        break;
    switch (act) { P1L(1) P1L(2) P1L(3) P1L(4) P1L(5) P1L(6) P1L(7) default: break; }
#undef P1L
    LAUNCH_CHECK();
}

void launch_pass2(int act, const double *Z0, int m0, int n1, int n2, const DevAxis &a1, const DevAxis &a2, double *B,
                  cudaStream_t s) {
    const bool A1 = act & 2, A2 = act & 4;
    const int nc1 = A1 ? a1.nc : n1, nc2 = A2 ? a2.nc : n2;
    const unsigned gx = A2 ? (unsigned)((nc2 + kP2Out - 1) / kP2Out) : (unsigned)((n2 + kP2Threads - 1) / kP2Threads);
    const int64_t cols = (int64_t)m0 * gx * kP2Threads;
    const int slabs = slabs_for(cols, nc1);
    dim3 grid(gx, (unsigned)m0, (unsigned)slabs);
    if (A1 && A2) k_level_pass2<true, true><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs);
    else if (A1) k_level_pass2<true, false><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs);
    else if (A2) k_level_pass2<false, true><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs);
    else k_level_pass2<false, false><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs);
    LAUNCH_CHECK();
}

template <typename TOut>
void launch_final(int act, const double *cv, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1,
                  const DevAxis &a2, const LevelMap &lm, const double *coef, TOut *D, cudaStream_t s) {
    dim3 grid((n2 + 31) / 32, (n1 + 7) / 8, slabs_for((int64_t)n1 * n2, n0));
    dim3 block(32, 8);
#define FL(M)                                                                                                      \
    case M:                                                                                                        \
        k_level_final<(M & 1) != 0, (M & 2) != 0, (M & 4) != 0, TOut><<<grid, block, 0, s>>>(cv, n0, n1, n2, a0, \
                                                                                              a1, a2, lm, coef, D); \
        break;
    switch (act) { FL(1) FL(2) FL(3) FL(4) FL(5) FL(6) FL(7) default: break; }
#undef FL
    LAUNCH_CHECK();
}

}  // namespace

bool fused_supported(const DevPlan &p) { return p.dims.n[0] == 1; }

void fused_pass1_decompose(const DevPlan &p, int st_i, const void *F, bool f32, double *coef, double *Z0, double *Cg,
                           cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const int n0 = (int)st.fsh.n[1], n1 = (int)st.fsh.n[2], n2 = (int)st.fsh.n[3];
    const int act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    LevelMap lm{p.map[1][st_i], p.map[2][st_i], p.map[3][st_i], p.dims.n[2], p.dims.n[3]};
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    const int64_t zsz = (int64_t)((act & 1) ? st.ax[1].nc : n0) * n1 * n2;
    KPROF("k_level_pass1", (f32 ? 4.0 : 8.0) * nf + 8.0 * (nf - nc) + 8.0 * nc + 8.0 * zsz, s);
    const QuantOut q{};
    if (f32) launch_pass1<0, float>(act, (const float *)F, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, coef,
                                    nullptr, Z0, Cg, q, s);
    else launch_pass1<0, double>(act, (const double *)F, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, coef,
                                 nullptr, Z0, Cg, q, s);
}

void fused_pass1_recompose(const DevPlan &p, int st_i, const double *coef, double *Z0, cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const int n0 = (int)st.fsh.n[1], n1 = (int)st.fsh.n[2], n2 = (int)st.fsh.n[3];
    const int act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    LevelMap lm{p.map[1][st_i], p.map[2][st_i], p.map[3][st_i], p.dims.n[2], p.dims.n[3]};
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    const int64_t zsz = (int64_t)((act & 1) ? st.ax[1].nc : n0) * n1 * n2;
    KPROF("k_level_pass1r", 8.0 * (nf - nc) + 8.0 * zsz, s);
    const QuantOut q{};
    launch_pass1<1, double>(act, nullptr, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, nullptr, coef, Z0, nullptr,
                            q, s);
}

void fused_pass1_quantize(const DevPlan &p, int st_i, const void *F, bool f32, const QuantOut &q, double *Z0,
                          double *Cg, cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const int n0 = (int)st.fsh.n[1], n1 = (int)st.fsh.n[2], n2 = (int)st.fsh.n[3];
    const int act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    LevelMap lm{p.map[1][st_i], p.map[2][st_i], p.map[3][st_i], p.dims.n[2], p.dims.n[3]};
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    const int64_t zsz = (int64_t)((act & 1) ? st.ax[1].nc : n0) * n1 * n2;
    KPROF("k_level_pass1q", (f32 ? 4.0 : 8.0) * nf + 4.0 * (nf - nc) + 8.0 * nc + 8.0 * zsz, s);
    if (f32) launch_pass1<2, float>(act, (const float *)F, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, nullptr,
                                    nullptr, Z0, Cg, q, s);
    else launch_pass1<2, double>(act, (const double *)F, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, nullptr,
                                 nullptr, Z0, Cg, q, s);
}

void quantize_coarsest(const DevPlan &p, const double *coarsest_vals, const QuantOut &q, cudaStream_t s) {
    const int n = (int)p.host.coarsest.size();
    KPROF("k_quantize_coarsest", 16.0 * n, s);
    k_quantize_coarsest<<<1, 32, 0, s>>>(coarsest_vals, p.coarsest, n, q);
    LAUNCH_CHECK();
}

void fused_pass2(const DevPlan &p, int st_i, const double *Z0, double *B, cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const int n0 = (int)st.fsh.n[1], n1 = (int)st.fsh.n[2], n2 = (int)st.fsh.n[3];
    const int act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    const int m0 = (act & 1) ? st.ax[1].nc : n0;
    KPROF("k_level_pass2", 8.0 * m0 * n1 * n2 + 8.0 * st.csh.size(), s);
    launch_pass2(act, Z0, m0, n1, n2, st.ax[2], st.ax[3], B, s);
}

void fused_final(const DevPlan &p, int st_i, const double *cv, const double *coef, void *D, int out_dtype,
                 cudaStream_t s) {
    const DevStep &st = p.steps[st_i];
    const int n0 = (int)st.fsh.n[1], n1 = (int)st.fsh.n[2], n2 = (int)st.fsh.n[3];
    const int act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    LevelMap lm{p.map[1][st_i], p.map[2][st_i], p.map[3][st_i], p.dims.n[2], p.dims.n[3]};
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    KPROF("k_level_final", 8.0 * nc + 8.0 * (nf - nc) + (out_dtype == 0 ? 4.0 : 8.0) * nf, s);
    if (out_dtype == 0)
        launch_final<float>(act, cv, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, coef, (float *)D, s);
    else
        launch_final<double>(act, cv, n0, n1, n2, st.ax[1], st.ax[2], st.ax[3], lm, coef, (double *)D, s);
}

}  // namespace hpdr
