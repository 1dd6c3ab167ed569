// fused.cu -- fused level kernels for ranks 1..3 (a 3-D view; rank-4 fields take the
// per-axis path in transform.cu).
//
// One decomposition transition (transform.py:306-315) becomes
//   pass 1   k_level_pass1   residual mc = F - P(F) (GPK, nested lerps in axis order 0,1,2)
//                            -> coefficient / quantized-key write, coarse-node gather, and the
//                            axis-0 mass-multiply + restriction (LPK, transform.py:206-226 then
//                            :181-203) as a register march along axis 0
//   pass 2   k_level_pass2   axis-1 LPK march + axis-2 LPK across the block (shared memory)
//   IPK      Thomas sweeps (transform.cu) and coarse + corr
// and recomposition (transform.py:337-347) mirrors it with pass 1 reading mc from the
// coefficients and k_level_final writing pred + mc (or the output dtype at the finest level).
//
// The marches are sequential along one axis, so every kernel streams its planes / rows through
// a cp.async shared-memory ring several steps ahead of the arithmetic (the dependency chain of
// the march never waits on DRAM).  Every value is produced with the reference's operation
// order (explicit _rn intrinsics): results are bit-identical to numpy.
#include "level_dev.cuh"

namespace hpdr {

namespace {

using namespace lvl;


// Sliding mass-multiply + restriction along the march axis (transform.py:206-226 then :181-203):
//   y(j) = (md_j x_j + ml_j x_{j-1}) + mu_j x_{j+1}
//   z(c) = (y(r0_c) + wr_c y(rr_c)) + wl_c y(rl_c)
// driven by the host-built PlaneInfo records (which coarse output completes at which y).
struct March {
    double m1, m2;        // x(j-1), x(j-2)
    double ya, yb, yc;    // y(k-2), y(k-1), y(k)
    int c_lo, c_hi;       // coarse outputs this march owns
};

__device__ __forceinline__ void march_init(March &M, int c_lo, int c_hi) {
    M.c_lo = c_lo;
    M.c_hi = c_hi;
    M.m1 = M.m2 = M.ya = M.yb = M.yc = 0.0;
}

template <class Emit>
__device__ __forceinline__ void march_y(March &M, double v, int emit, int rr, int rl, double wr, double wl,
                                        Emit &&out) {
    M.ya = M.yb;
    M.yb = M.yc;
    M.yc = v;
    if (emit >= M.c_lo && emit < M.c_hi) {
        double z;
        if (rr) {
            z = dadd(M.yb, dmul(wr, M.yc));
            if (rl) z = dadd(z, dmul(wl, M.ya));
        } else {
            z = M.yc;
            if (rl) z = dadd(z, dmul(wl, M.yb));
        }
        out(emit, z);
    }
}

// y(k) and its emission for fine index k, reading k's PlaneInfo from the (L1-resident) table.
template <bool NC, typename T>
__device__ __forceinline__ T ldx(const T *p) {   // read-only-path load from global, plain load otherwise
    if (NC) return __ldg(p);
    return *p;
}

template <int MASK = -1, bool NC = MASK == -1, class Emit>
__device__ __forceinline__ void march_emit_y(March &M, const PlaneInfo *__restrict__ P, int k, double xk, double xkm1,
                                             double xkp1, bool has_up, Emit &&out) {
    // NC: records in global memory (read-only path); else shared (MASK != -1: a ring of records)
    const PlaneInfo *p = P + (k & MASK);
    double v = dmul(ldx<NC>(&p->md), xk);
    if (k >= 1) v = dadd(v, dmul(ldx<NC>(&p->ml), xkm1));
    if (has_up) v = dadd(v, dmul(ldx<NC>(&p->mu), xkp1));
    const int4 e = ldx<NC>(reinterpret_cast<const int4 *>(&p->fo));   // fo, emit, e_rr, e_rl
    double wr = 0.0, wl = 0.0;
    if (e.y >= M.c_lo && e.y < M.c_hi) {
        wr = ldx<NC>(&p->ewr);
        wl = ldx<NC>(&p->ewl);
    }
    march_y(M, v, e.y, e.z, e.w, wr, wl, out);
}

// Push x(j) (PlaneInfo table P); emits every restricted value that became computable.
template <int MASK = -1, bool NC = MASK == -1, class Emit>
__device__ __forceinline__ void march_push(March &M, const PlaneInfo *__restrict__ P, int n, int j, int j_start,
                                           double x, Emit &&out) {
    // y(j-1) needs x(j-2) unless j-1 == 0: j >= 1 when the march starts at 0, else j >= j_start + 2
    if (j >= (j_start == 0 ? 1 : j_start + 2)) march_emit_y<MASK, NC>(M, P, j - 1, M.m1, M.m2, x, true, out);
    if (j == n - 1 && (j > j_start || j == 0)) march_emit_y<MASK, NC>(M, P, j, x, M.m1, 0.0, false, out);
    M.m2 = M.m1;
    M.m1 = x;
}

// The interpolation part of a PlaneInfo record (what pass 1 needs per plane).
struct PiHead {
    int fa, fb, ca, fo;
    double t;
};

template <bool NC = true>
__device__ __forceinline__ PiHead load_head(const PlaneInfo *__restrict__ p) {
    const int4 a = ldx<NC>(reinterpret_cast<const int4 *>(p));   // fa, fb, ca, cb
    PiHead h;
    h.fa = a.x;
    h.fb = a.y;
    h.ca = a.z;
    h.fo = ldx<NC>(&p->fo);
    h.t = ldx<NC>(&p->t);
    return h;
}

__device__ __forceinline__ PiHead identity_head(int j) {
    PiHead h;
    h.fa = h.fb = h.ca = j;
    h.fo = 0;
    h.t = 0.0;
    return h;
}


template <typename T>
__device__ __forceinline__ void cp_elem(T *s, const T *g) {
    cp_async<sizeof(T)>(s, g);
}

// ---------------------------------------------------------------------------------- pass 1
// MODE 0 (decompose):  mc = F - P(F); coef[fine-only] = mc; Cg[coarse] = F; Z0 = R0M0(mc)
// MODE 1 (recompose):  mc = coef at fine-only nodes, 0 at coarse nodes; Z0 = R0M0(mc)
// MODE 2 (decompose with quantize-on-write): as MODE 0 but fine-only nodes are quantized
//   straight into keys / outlier mask / histogram (quantize.py:73-84) instead of coef.
// Z0 = mc along axis 0 when that axis is inactive at this transition.
// Block: 32 x 8 columns (j2, j1); each plane of the tile (+1 halo) streams through a cp.async
// ring kRing-2 planes ahead of the march.  Per-thread smem / global offsets are fixed up front;
// per-plane axis-0 data is one PlaneInfo record.
constexpr int kTX = 32, kTY = 8, kHX = kTX + 2, kHY = kTY + 2, kRing = 8;
constexpr int kPlaneElems = kHX * kHY;   // 340
constexpr int kSmemHist = 4096;

template <int MODE, bool A0, bool A1, bool A2, typename TIn>
__global__ void __launch_bounds__(256, 4) k_level_pass1(const TIn *__restrict__ F, int n0, int n1, int n2, DevAxis ax0,
                                                     DevAxis ax1, DevAxis ax2, LevelMap lm, double *__restrict__ coef,
                                                     const double *__restrict__ coef_in, double *__restrict__ Z0,
                                                     double *__restrict__ Cg, QuantOut q, int c_base, int c_count) {
    __shared__ __align__(16) TIn ring[kRing * kPlaneElems];
    __shared__ double sP0[MODE != 1 ? 2 : 1][MODE != 1 ? kPlaneElems : 1];   // axis-0 GPK plane, double-buffered
    __shared__ __align__(16) PlaneInfo piring[kRing];   // axis-0 records of the planes in the ring
    __shared__ uint32_t sh_hist[MODE == 2 ? kSmemHist : 1];
    const bool sh_ok = MODE == 2 && q.dict <= kSmemHist;
    const double rbin = MODE == 2 ? 1.0 / qbin(q) : 0.0;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) sh_hist[k] = 0;
    const int x0 = blockIdx.x * kTX - 1, y0 = blockIdx.y * kTY - 1;   // tile origin incl. halo
    const int j2 = x0 + 1 + tx, j1 = y0 + 1 + ty;
    const bool act = j1 < n1 && j2 < n2;
    const int nc0 = A0 ? ax0.nc : n0;
    int c_lo, c_hi;
    slab_range(c_count, gridDim.z, blockIdx.z, c_lo, c_hi);   // coarse outputs [c_base, c_base + c_count)
    c_lo += c_base;
    c_hi += c_base;
    int fl = 0;
    if (c_lo < c_hi) {   // uniform across the block
        int j_start, j_end, own_lo, own_hi;
        slab_planes<A0>(ax0, n0, nc0, c_lo, c_hi, j_start, j_end, own_lo, own_hi);
        const int64_t plane = (int64_t)n1 * n2;
        const int64_t fplane = lm.D1 * lm.D2;
        const int own_off = (ty + 1) * kHX + tx + 1;
        const int64_t col = (int64_t)j1 * n2 + j2;
        const int64_t fcol = act ? ((int64_t)__ldg(lm.m1 + j1)) * lm.D2 + __ldg(lm.m2 + j2) : 0;
        // this thread's share of each plane load: two tile elements (halo included)
        int soff[2];
        int64_t goff[2];
        bool lv[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int e = tid + k * 256;
            const int yy = e / kHX, xx = e - yy * kHX;
            const int gy = y0 + yy, gx = x0 + xx;
            lv[k] = MODE != 1 && e < kPlaneElems && gy >= 0 && gy < n1 && gx >= 0 && gx < n2;
            soff[k] = e;
            goff[k] = (int64_t)gy * n2 + gx;
        }
        // issue(p) is called for p = j_start, j_start + 1, ... in order: running source pointers and
        // precomputed 32-bit shared addresses keep the per-plane issue cheap
        const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
        const unsigned sa0 = ring_s + soff[0] * (unsigned)sizeof(TIn), sa1 = ring_s + soff[1] * (unsigned)sizeof(TIn);
        const unsigned sown = ring_s + own_off * (unsigned)sizeof(TIn);
        const TIn *gp0 = MODE == 1 ? nullptr : F + goff[0] + (int64_t)j_start * plane;
        const TIn *gp1 = MODE == 1 ? nullptr : F + goff[1] + (int64_t)j_start * plane;
        const unsigned pir_s = (unsigned)__cvta_generic_to_shared(piring) + (unsigned)tid * 16u;
        auto issue = [&](int p) {
            if (p <= j_end) {
                if (A0 && tid < 5)   // the plane's 80-byte PlaneInfo record rides with it
                    cp_async_s<16>(pir_s + (unsigned)(p & (kRing - 1)) * (unsigned)sizeof(PlaneInfo),
                                   reinterpret_cast<const char *>(ax0.pi + p) + tid * 16);
                const unsigned so = (unsigned)(p & (kRing - 1)) * (unsigned)(kPlaneElems * sizeof(TIn));
                if (MODE == 1) {
                    if (act)
                        cp_async_s<sizeof(TIn)>(sown + so,
                                                (const TIn *)(coef_in + (int64_t)__ldg(lm.m0 + p) * fplane + fcol));
                } else {
                    if (lv[0]) cp_async_s<sizeof(TIn)>(sa0 + so, gp0);
                    if (lv[1]) cp_async_s<sizeof(TIn)>(sa1 + so, gp1);
                    gp0 += plane;
                    gp1 += plane;
                }
            }
            cp_async_commit();
        };
        // per-thread axis-1 / axis-2 neighbours as smem offsets within a plane
        Nb b1{}, b2{};
        if (act) {
            b1 = neighbours<A1>(ax1, j1);
            b2 = neighbours<A2>(ax2, j2);
        }
        const int oaa = (b1.fa - y0) * kHX + (b2.fa - x0), oba = (b1.fb - y0) * kHX + (b2.fa - x0);
        const int oab = (b1.fa - y0) * kHX + (b2.fb - x0), obb = (b1.fb - y0) * kHX + (b2.fb - x0);
        const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
        const int64_t cgcol = (int64_t)b1.ca * nc2 + b2.ca;
        const bool col_coarse = !b1.fo && !b2.fo;
        March M;
        march_init(M, c_lo, c_hi);
        auto emit = [&](int c, double z) { Z0[(int64_t)c * plane + col] = z; };
        // GPK stage along axis 0 (P0 = lerp of the fine planes' coarse neighbours), computed once
        // per tile element for plane p into sP0[p & 1]; done one plane ahead of the march so the
        // per-plane barrier also publishes it (transform.py:264-268 order: axis 0, then 1, then 2)
        auto stage_p0 = [&](int p) {
            if (MODE == 1 || p > j_end) return;
            const PiHead ph = A0 ? load_head<false>(piring + (p & (kRing - 1))) : identity_head(p);
            const TIn *ra = ring + (ph.fa & (kRing - 1)) * kPlaneElems;
            const TIn *rb = ring + (ph.fb & (kRing - 1)) * kPlaneElems;
            double *dst = sP0[MODE != 1 ? (p & 1) : 0];
#pragma unroll
            for (int k = 0; k < 2; k++)
                if (lv[k]) {
                    const double va = (double)ra[soff[k]];
                    dst[soff[k]] = ph.fo ? lerp(va, (double)rb[soff[k]], ph.t) : va;
                }
        };
        for (int k = 0; k < kRing - 2; k++) issue(j_start + k);
        if (MODE != 1) {
            cp_async_wait<kRing - 4>();   // planes j_start, j_start + 1 have landed
            __syncthreads();
            stage_p0(j_start);
        }
        for (int j = j_start; j <= j_end; j++) {
            if (MODE != 1) cp_async_wait<kRing - 5>();   // planes <= j + 2 have landed
            else cp_async_wait<kRing - 4>();              // planes <= j + 1 have landed
            __syncthreads();
            issue(j + kRing - 2);          // into the slot of plane j - 2 (no longer read)
            stage_p0(j + 1);               // its neighbours are planes <= j + 2
            if (!act) continue;
            const PiHead pi = A0 ? load_head<false>(piring + (j & (kRing - 1))) : identity_head(j);
            const bool coarse_node = !pi.fo && col_coarse;
            const TIn *rj = ring + (j & (kRing - 1)) * kPlaneElems;
            double mc;
            if (MODE != 1) {
                // GPK: P0 (staged), P1 along axis 1, P2 along axis 2
                const double *P0p = sP0[MODE != 1 ? (j & 1) : 0];
                double p1a = P0p[oaa], p1b = 0.0;
                if (A1 && b1.fo) p1a = lerp(p1a, P0p[oba], b1.t);
                if (A2) {
                    p1b = P0p[oab];
                    if (A1 && b1.fo) p1b = lerp(p1b, P0p[obb], b1.t);
                }
                const double pred = (A2 && b2.fo) ? lerp(p1a, p1b, b2.t) : p1a;
                const double own = (double)rj[own_off];
                mc = dsub(own, pred);
                if (j >= own_lo && j < own_hi) {
                    if (coarse_node) {
                        const int c0 = A0 ? pi.ca : j;
                        Cg[(int64_t)c0 * nc1 * nc2 + cgcol] = own;
                    } else {
                        const int64_t f = (int64_t)__ldg(lm.m0 + j) * fplane + fcol;
                        if (MODE == 0) {
                            coef[f] = mc;
                        } else {
                            quant_node(mc, q, rbin, f, fl, sh_hist, sh_ok);
                        }
                    }
                }
            } else {
                mc = coarse_node ? 0.0 : (double)rj[own_off];
            }
            if (A0) march_push<kRing - 1>(M, piring, n0, j, j_start, mc, emit);
            else Z0[(int64_t)j * plane + col] = mc;
        }
        cp_async_wait<0>();
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

// ---------------------------------------------------------------------------------- pass 1, 2 rows/thread
// k_level_pass1 with a 32 x 16 column tile: each thread owns rows j1 and j1 + 8, so the per-plane
// work that does not depend on the column (barrier, ring issue, PlaneInfo reads, march control) is
// shared by two nodes.  Same arithmetic, same order: bit-identical results.
constexpr int kTY2 = 2 * kTY, kHY2 = kTY2 + 2, kPlane2 = kHX * kHY2;   // 612 elements per plane

template <int MODE, bool A0, bool A1, bool A2, typename TIn>
__global__ void __launch_bounds__(256) k_level_pass1_2r(const TIn *__restrict__ F, int n0, int n1, int n2,
                                                        DevAxis ax0, DevAxis ax1, DevAxis ax2, LevelMap lm,
                                                        double *__restrict__ coef, const double *__restrict__ coef_in,
                                                        double *__restrict__ Z0, double *__restrict__ Cg, QuantOut q,
                                                        int c_base, int c_count) {
    constexpr int PE = MODE == 1 ? kTX * kTY2 : kPlane2;   // ring slot: own elements only in MODE 1
    __shared__ __align__(16) TIn ring[kRing * PE];
    __shared__ double sP0[MODE != 1 ? 2 : 1][MODE != 1 ? kPlane2 : 1];
    __shared__ __align__(16) PlaneInfo piring[kRing];
    __shared__ uint32_t sh_hist[MODE == 2 ? kSmemHist : 1];
    const bool sh_ok = MODE == 2 && q.dict <= kSmemHist;
    const double rbin = MODE == 2 ? 1.0 / qbin(q) : 0.0;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) sh_hist[k] = 0;
    const int x0 = blockIdx.x * kTX - 1, y0 = blockIdx.y * kTY2 - 1;   // tile origin incl. halo
    const int j2 = x0 + 1 + tx;
    const int nc0 = A0 ? ax0.nc : n0;
    int c_lo, c_hi;
    slab_range(c_count, gridDim.z, blockIdx.z, c_lo, c_hi);
    c_lo += c_base;
    c_hi += c_base;
    int fl = 0;
    if (c_lo < c_hi) {   // uniform across the block
        int j_start, j_end, own_lo, own_hi;
        slab_planes<A0>(ax0, n0, nc0, c_lo, c_hi, j_start, j_end, own_lo, own_hi);
        const int64_t plane = (int64_t)n1 * n2;
        const int64_t fplane = lm.D1 * lm.D2;
        const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
        const Nb b2 = j2 < n2 ? neighbours<A2>(ax2, j2) : Nb{};
        const int64_t fcol2 = j2 < n2 ? (int64_t)__ldg(lm.m2 + j2) : 0;
        // per-row state (rows j1 = y0 + 1 + ty + 8 r)
        int j1r[2], own_off[2], oaa[2], oba[2], oab[2], obb[2];
        bool act[2], col_coarse[2];
        int64_t col[2], fcol[2], cgcol[2];
        Nb b1[2];
        March M[2];
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int j1 = y0 + 1 + ty + kTY * r;
            j1r[r] = j1;
            act[r] = j1 < n1 && j2 < n2;
            own_off[r] = MODE == 1 ? (ty + kTY * r) * kTX + tx : (ty + kTY * r + 1) * kHX + tx + 1;
            col[r] = (int64_t)j1 * n2 + j2;
            fcol[r] = act[r] ? ((int64_t)__ldg(lm.m1 + j1)) * lm.D2 + fcol2 : 0;
            b1[r] = act[r] ? neighbours<A1>(ax1, j1) : Nb{};
            oaa[r] = (b1[r].fa - y0) * kHX + (b2.fa - x0);
            oba[r] = (b1[r].fb - y0) * kHX + (b2.fa - x0);
            oab[r] = (b1[r].fa - y0) * kHX + (b2.fb - x0);
            obb[r] = (b1[r].fb - y0) * kHX + (b2.fb - x0);
            cgcol[r] = (int64_t)b1[r].ca * nc2 + b2.ca;
            col_coarse[r] = !b1[r].fo && !b2.fo;
            march_init(M[r], c_lo, c_hi);
        }
        // this thread's share of each plane load: three tile elements (halo included)
        int soff[3];
        int64_t goff[3];
        bool lv[3];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const int e = tid + k * 256;
            const int yy = e / kHX, xx = e - yy * kHX;
            const int gy = y0 + yy, gx = x0 + xx;
            lv[k] = MODE != 1 && e < kPlane2 && gy >= 0 && gy < n1 && gx >= 0 && gx < n2;
            soff[k] = e;
            goff[k] = (int64_t)gy * n2 + gx;
        }
        const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
        const unsigned pir_s = (unsigned)__cvta_generic_to_shared(piring) + (unsigned)tid * 16u;
        const TIn *gp[3];
#pragma unroll
        for (int k = 0; k < 3; k++) gp[k] = MODE == 1 ? nullptr : F + goff[k] + (int64_t)j_start * plane;
        auto issue = [&](int p) {
            if (p <= j_end) {
                if (A0 && tid < 5)
                    cp_async_s<16>(pir_s + (unsigned)(p & (kRing - 1)) * (unsigned)sizeof(PlaneInfo),
                                   reinterpret_cast<const char *>(ax0.pi + p) + tid * 16);
                const unsigned so = ring_s + (unsigned)(p & (kRing - 1)) * (unsigned)(PE * sizeof(TIn));
                if (MODE == 1) {
                    const int64_t fb = (int64_t)__ldg(lm.m0 + p) * fplane;
#pragma unroll
                    for (int r = 0; r < 2; r++)
                        if (act[r])
                            cp_async_s<sizeof(TIn)>(so + own_off[r] * (unsigned)sizeof(TIn),
                                                    (const TIn *)(coef_in + fb + fcol[r]));
                } else {
#pragma unroll
                    for (int k = 0; k < 3; k++) {
                        if (lv[k]) cp_async_s<sizeof(TIn)>(so + soff[k] * (unsigned)sizeof(TIn), gp[k]);
                        gp[k] += plane;
                    }
                }
            }
            cp_async_commit();
        };
        auto stage_p0 = [&](int p) {
            if (MODE == 1 || p > j_end) return;
            const PiHead ph = A0 ? load_head<false>(piring + (p & (kRing - 1))) : identity_head(p);
            const TIn *ra = ring + (ph.fa & (kRing - 1)) * PE;
            const TIn *rb = ring + (ph.fb & (kRing - 1)) * PE;
            double *dst = sP0[MODE != 1 ? (p & 1) : 0];
#pragma unroll
            for (int k = 0; k < 3; k++)
                if (lv[k]) {
                    const double va = (double)ra[soff[k]];
                    dst[soff[k]] = ph.fo ? lerp(va, (double)rb[soff[k]], ph.t) : va;
                }
        };
        for (int k = 0; k < kRing - 2; k++) issue(j_start + k);
        if (MODE != 1) {
            cp_async_wait<kRing - 4>();
            __syncthreads();
            stage_p0(j_start);
        }
        for (int j = j_start; j <= j_end; j++) {
            if (MODE != 1) cp_async_wait<kRing - 5>();   // planes <= j + 2 have landed
            else cp_async_wait<kRing - 4>();              // planes <= j + 1 have landed
            __syncthreads();
            issue(j + kRing - 2);
            stage_p0(j + 1);
            const PiHead pi = A0 ? load_head<false>(piring + (j & (kRing - 1))) : identity_head(j);
            const TIn *rj = ring + (j & (kRing - 1)) * PE;
            const bool own_plane = j >= own_lo && j < own_hi;
            const int64_t fplane_j = own_plane ? (int64_t)__ldg(lm.m0 + j) * fplane : 0;
            const double *P0p = sP0[MODE != 1 ? (j & 1) : 0];
#pragma unroll
            for (int r = 0; r < 2; r++) {
                if (!act[r]) continue;
                const bool coarse_node = !pi.fo && col_coarse[r];
                double mc;
                if (MODE != 1) {
                    double p1a = P0p[oaa[r]], p1b = 0.0;
                    if (A1 && b1[r].fo) p1a = lerp(p1a, P0p[oba[r]], b1[r].t);
                    if (A2) {
                        p1b = P0p[oab[r]];
                        if (A1 && b1[r].fo) p1b = lerp(p1b, P0p[obb[r]], b1[r].t);
                    }
                    const double pred = (A2 && b2.fo) ? lerp(p1a, p1b, b2.t) : p1a;
                    const double own = (double)rj[own_off[r]];
                    mc = dsub(own, pred);
                    if (own_plane) {
                        if (coarse_node) {
                            const int c0 = A0 ? pi.ca : j;
                            Cg[(int64_t)c0 * nc1 * nc2 + cgcol[r]] = own;
                        } else {
                            const int64_t f = fplane_j + fcol[r];
                            if (MODE == 0) coef[f] = mc;
                            else quant_node(mc, q, rbin, f, fl, sh_hist, sh_ok);
                        }
                    }
                } else {
                    mc = coarse_node ? 0.0 : (double)rj[own_off[r]];
                }
                double *zc = Z0 + col[r];
                auto emit = [&](int c, double z) { zc[(int64_t)c * plane] = z; };
                if (A0) march_push<kRing - 1>(M[r], piring, n0, j, j_start, mc, emit);
                else zc[(int64_t)j * plane] = mc;
            }
        }
        cp_async_wait<0>();
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

// ---------------------------------------------------------------------------------- pass 1 (decompose)
// Same contract as k_level_pass1 MODE 0 / 2, with the GPK interpolation evaluated separably
// inside the tile, in the reference's axis order (transform.py:264-268):
//   stage A  P0 = lerp along axis 0 at the tile's coarse rows x coarse columns (from the F ring)
//   stage B  P1 = lerp along axis 1 at the tile rows x coarse columns (from P0)
//   stage C  P2 = lerp along axis 2 per node (from P1); mc = F - P2
// Every P value is computed once per plane instead of once per fine node that uses it.
constexpr int kP1Rows = kTY, kP1Cols = kHX;   // P1 block: tile rows x halo columns

template <int MODE, bool A0, bool A1, bool A2, typename TIn>
__global__ void __launch_bounds__(256) k_level_pass1s(const TIn *__restrict__ F, int n0, int n1, int n2, DevAxis ax0,
                                                      DevAxis ax1, DevAxis ax2, LevelMap lm, double *__restrict__ coef,
                                                      double *__restrict__ Z0, double *__restrict__ Cg, QuantOut q,
                                                      int c_base, int c_count) {
    __shared__ __align__(16) TIn ring[kRing * kPlaneElems];
    __shared__ double sP0[kPlaneElems];
    __shared__ double sP1[kP1Rows * kP1Cols];
    __shared__ uint32_t sh_hist[MODE == 2 ? kSmemHist : 1];
    const bool sh_ok = MODE == 2 && q.dict <= kSmemHist;
    const double rbin = MODE == 2 ? 1.0 / qbin(q) : 0.0;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) sh_hist[k] = 0;
    const int x0 = blockIdx.x * kTX - 1, y0 = blockIdx.y * kTY - 1;   // tile origin incl. halo
    const int j2 = x0 + 1 + tx, j1 = y0 + 1 + ty;
    const bool act = j1 < n1 && j2 < n2;
    const int nc0 = A0 ? ax0.nc : n0;
    int c_lo, c_hi;
    slab_range(c_count, gridDim.z, blockIdx.z, c_lo, c_hi);
    c_lo += c_base;
    c_hi += c_base;
    int fl = 0;
    if (c_lo < c_hi) {   // uniform across the block
        int j_start, j_end, own_lo, own_hi;
        slab_planes<A0>(ax0, n0, nc0, c_lo, c_hi, j_start, j_end, own_lo, own_hi);
        const int64_t plane = (int64_t)n1 * n2;
        const int64_t fplane = lm.D1 * lm.D2;
        // per-thread load slots (two tile elements incl. halo) and stage-A / stage-B work items
        int soff[2];
        int64_t goff[2];
        bool lv[2], needA[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int e = tid + k * 256;
            const int yy = e / kHX, xx = e - yy * kHX;
            const int gy = y0 + yy, gx = x0 + xx;
            const bool in = e < kPlaneElems && gy >= 0 && gy < n1 && gx >= 0 && gx < n2;
            lv[k] = in;
            soff[k] = e;
            goff[k] = (int64_t)gy * n2 + gx;
            // P0 is needed at coarse rows (or every row when axis 1 is inactive) x coarse columns
            needA[k] = in && (!A1 || __ldg(ax1.pb + gy) < 0) && (!A2 || __ldg(ax2.pb + gx) < 0);
        }
        // stage B items: (tile row, halo column) pairs at coarse columns
        int bsoff[2], brow_a[2], brow_b[2];
        double bt[2];
        bool needB[2], bfo[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int e = tid + k * 256;
            const int r = e / kP1Cols, xx = e - r * kP1Cols;
            const int gy = y0 + 1 + r, gx = x0 + xx;
            needB[k] = e < kP1Rows * kP1Cols && gy < n1 && gx >= 0 && gx < n2 && (!A2 || __ldg(ax2.pb + gx) < 0);
            bsoff[k] = e;
            brow_a[k] = brow_b[k] = 0;
            bt[k] = 0.0;
            bfo[k] = false;
            if (needB[k]) {
                const Nb nb = neighbours<A1>(ax1, gy);
                bfo[k] = nb.fo;
                bt[k] = nb.t;
                brow_a[k] = (nb.fa - y0) * kHX + xx;
                brow_b[k] = (nb.fb - y0) * kHX + xx;
            }
        }
        auto issue = [&](int p) {
            if (p <= j_end) {
                TIn *slot = ring + (p & (kRing - 1)) * kPlaneElems;
                const TIn *src = F + (int64_t)p * plane;
                if (lv[0]) cp_async<sizeof(TIn)>(slot + soff[0], src + goff[0]);
                if (lv[1]) cp_async<sizeof(TIn)>(slot + soff[1], src + goff[1]);
            }
            cp_async_commit();
        };
        Nb b1{}, b2{};
        if (act) {
            b1 = neighbours<A1>(ax1, j1);
            b2 = neighbours<A2>(ax2, j2);
        }
        const int own_off = (ty + 1) * kHX + tx + 1;
        const int p1a = ty * kP1Cols + (b2.fa - x0), p1b = ty * kP1Cols + (b2.fb - x0);
        const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
        const int64_t cgcol = (int64_t)b1.ca * nc2 + b2.ca;
        const bool col_coarse = !b1.fo && !b2.fo;
        const int64_t col = (int64_t)j1 * n2 + j2;
        const int64_t fcol = act ? ((int64_t)__ldg(lm.m1 + j1)) * lm.D2 + __ldg(lm.m2 + j2) : 0;
        double *zcol = Z0 + col;
        March M;
        march_init(M, c_lo, c_hi);
        auto emit = [&](int c, double z) { zcol[(int64_t)c * plane] = z; };
        for (int k = 0; k < kRing - 2; k++) issue(j_start + k);
        for (int j = j_start; j <= j_end; j++) {
            cp_async_wait<kRing - 4>();   // planes <= j + 1 have landed
            __syncthreads();
            issue(j + kRing - 2);
            const PiHead pi = A0 ? load_head(ax0.pi + j) : identity_head(j);
            const TIn *ra = ring + (pi.fa & (kRing - 1)) * kPlaneElems;
            const TIn *rb = ring + (pi.fb & (kRing - 1)) * kPlaneElems;
            // stage A: P0 at coarse rows x coarse columns
#pragma unroll
            for (int k = 0; k < 2; k++)
                if (needA[k]) {
                    const double va = (double)ra[soff[k]];
                    sP0[soff[k]] = pi.fo ? lerp(va, (double)rb[soff[k]], pi.t) : va;
                }
            __syncthreads();
            // stage B: P1 at tile rows x coarse columns
#pragma unroll
            for (int k = 0; k < 2; k++)
                if (needB[k]) {
                    const double va = sP0[brow_a[k]];
                    sP1[bsoff[k]] = bfo[k] ? lerp(va, sP0[brow_b[k]], bt[k]) : va;
                }
            __syncthreads();
            if (!act) continue;
            // stage C: P2 per node, residual, outputs
            const double pa = sP1[p1a];
            const double pred = (A2 && b2.fo) ? lerp(pa, sP1[p1b], b2.t) : pa;
            const double own = (double)ring[(j & (kRing - 1)) * kPlaneElems + own_off];
            const double mc = dsub(own, pred);
            if (j >= own_lo && j < own_hi) {
                if (!pi.fo && col_coarse) {
                    const int c0 = A0 ? pi.ca : j;
                    Cg[(int64_t)c0 * nc1 * nc2 + cgcol] = own;
                } else {
                    const int64_t f = (int64_t)__ldg(lm.m0 + j) * fplane + fcol;
                    if (MODE == 0) {
                        coef[f] = mc;
                    } else {
                        quant_node(mc, q, rbin, f, fl, sh_hist, sh_ok);
                    }
                }
            }
            if (A0) march_push(M, ax0.pi, n0, j, j_start, mc, emit);
            else zcol[(int64_t)j * plane] = mc;
        }
        cp_async_wait<0>();
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

// Quantize the fine-only nodes of the finest level from stored fp64 coefficients (the streamed
// relative-mode path, where the bin width is only known after the last input chunk).
template <bool A0, bool A1, bool A2>
__global__ void __launch_bounds__(256) k_quantize_fine(const double *__restrict__ coef, int n0, int n1, int n2,
                                                       DevAxis ax0, DevAxis ax1, DevAxis ax2, QuantOut q) {
    __shared__ uint32_t sh_hist[kSmemHist];
    const bool sh_ok = q.dict <= kSmemHist;
    const double rbin = 1.0 / qbin(q);
    const int tid = threadIdx.y * 32 + threadIdx.x;
    if (sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) sh_hist[k] = 0;
    __syncthreads();
    const int j2 = blockIdx.x * 32 + threadIdx.x, j1 = blockIdx.y * 8 + threadIdx.y;
    int fl = 0;
    if (j1 < n1 && j2 < n2) {
        const bool col_fo = (A1 && __ldg(ax1.pb + j1) >= 0) || (A2 && __ldg(ax2.pb + j2) >= 0);
        int lo, hi;
        slab_range(n0, gridDim.z, blockIdx.z, lo, hi);
        const int64_t plane = (int64_t)n1 * n2, col = (int64_t)j1 * n2 + j2;
        // 8 planes' coefficients in flight per thread before any is quantized (latency-bound otherwise);
        // the histogram is counted in runs of equal keys down the column (smooth data repeats a few
        // keys, so one shared atomic per run instead of per node)
        constexpr int U = 8;
        uint32_t run_key = 0, run_n = 0;
        for (int j0 = lo; j0 < hi; j0 += U) {
            double v[U];
            bool use[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int j = j0 + k;
                use[k] = j < hi && (col_fo || (A0 && __ldg(ax0.pb + j) >= 0));
                v[k] = use[k] ? __ldg(coef + (int64_t)j * plane + col) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < U; k++)
                if (use[k]) {
                    const uint32_t key = quant_key(v[k], q, rbin, (int64_t)(j0 + k) * plane + col, fl);
                    if (key != run_key && run_n) {
                        if (sh_ok) atomicAdd(&sh_hist[run_key], run_n);
                        else atomicAdd(&q.hist[run_key], (unsigned long long)run_n);
                        run_n = 0;
                    }
                    run_key = key;
                    run_n++;
                }
        }
        if (run_n) {
            if (sh_ok) atomicAdd(&sh_hist[run_key], run_n);
            else atomicAdd(&q.hist[run_key], (unsigned long long)run_n);
        }
    }
    if (fl) atomicOr(q.flags, fl);
    __syncthreads();
    if (sh_ok)
        for (uint32_t k = tid; k < q.dict; k += 256) {
            const uint32_t c = sh_hist[k];
            if (c) atomicAdd(&q.hist[k], (unsigned long long)c);
        }
}

// The same quantization streamed in memory order: each warp takes whole rows (plane j, row j1)
// and walks them in 32-node segments, eight in flight, so DRAM sees one sequential sweep (the
// column-walking kernel above reaches 36% of DRAM bandwidth).  Fast path of quant_node
// branch-free, the rest through quant_node.
template <bool A0, bool A1, bool A2>
__global__ void __launch_bounds__(256) k_quantize_fine_rows(const double *__restrict__ coef, int n0, int n1, int n2,
                                                            DevAxis ax0, DevAxis ax1, DevAxis ax2, QuantOut q) {
    __shared__ uint32_t sh_hist[kSmemHist];
    const bool sh_ok = q.dict <= kSmemHist;
    const double rbin = 1.0 / qbin(q);
    const double half = (double)q.half;
    if (sh_ok)
        for (uint32_t k = threadIdx.x; k < q.dict; k += blockDim.x) sh_hist[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int rows = n0 * n1;
    const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    int fl = 0;
    constexpr int U = 8;
    for (int row = wid; row < rows; row += nw) {
        const int j = row / n1, j1 = row - j * n1;
        const bool row_fo = (A0 && __ldg(ax0.pb + j) >= 0) || (A1 && __ldg(ax1.pb + j1) >= 0);
        const double *cr = coef + (int64_t)row * n2;
        uint16_t *kr = q.keys + (int64_t)row * n2;
        for (int c0 = lane; c0 < n2; c0 += 32 * U) {
            double v[U];
            bool use[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int c = c0 + 32 * k;
                use[k] = c < n2 && (row_fo || (A2 && __ldg(ax2.pb + c) >= 0));
                v[k] = use[k] ? __ldg(cr + c) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < U; k++) {
                const double qa = dmul(v[k], rbin);
                const double r = rint(qa);
                const int ri = (int)r;
                const uint32_t key = ((uint32_t)ri << 1) ^ (uint32_t)(ri >> 31);
                // |r| < half <= 32767.5 bounds |qa| < 2^15, so a fixed 2^-33 margin is stricter than
                // quant_key's |qa| * 2^-49 (one multiply fewer; the rare miss takes the exact path)
                const bool ok = fabs(dsub(qa, r)) < 0.5 - 0x1p-33 && fabs(r) < half;   // (qa - r is exact)
                if (use[k] && ok) {
                    kr[c0 + 32 * k] = (uint16_t)key;
                    if (sh_ok) atomicAdd(&sh_hist[key], 1u);
                    else atomicAdd(&q.hist[key], 1ULL);
                } else if (use[k]) {
                    quant_node(v[k], q, rbin, (int64_t)row * n2 + c0 + 32 * k, fl, sh_hist, sh_ok);
                }
            }
        }
    }
    if (fl) atomicOr(q.flags, fl);
    __syncthreads();
    if (sh_ok)
        for (uint32_t k = threadIdx.x; k < q.dict; k += blockDim.x) {
            const uint32_t c = sh_hist[k];
            if (c) atomicAdd(&q.hist[k], (unsigned long long)c);
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
        else if (fabs(v / qbin(q)) >= 4611686018427387904.0) fl |= 2;
        if (fl) atomicOr(q.flags, fl);
        q.keys[idx[k]] = 0;
    }
    if (k == 0) atomicAdd(&q.hist[0], (unsigned long long)n);
}

// ---------------------------------------------------------------------------------- pass 2
// Z0 (m0, n1, n2) -> B (m0, nc1, nc2): axis-1 LPK as a march over rows streamed through a
// cp.async ring, axis-2 LPK across the block through shared memory.
constexpr int kP2Threads = 256;
constexpr int kP2Out = (kP2Threads - 4) / 2;   // coarse outputs along axis 2 per block
constexpr int kP2Ring = 8;
constexpr int kP2MaxRows = 272;   // fine rows per pass-2 slab (<= 130 coarse outputs + stencil)

template <bool A1, bool A2>
__global__ void __launch_bounds__(kP2Threads) k_level_pass2(const double *__restrict__ Z0, int m0, int n1, int n2,
                                                            DevAxis ax1, DevAxis ax2, double *__restrict__ B,
                                                            int slabs1, int p_base) {
    __shared__ double sw[kP2Threads];
    __shared__ double sy[kP2Threads];
    __shared__ __align__(16) double ring[kP2Ring][kP2Threads];
    __shared__ __align__(16) PlaneInfo ptab[A1 ? kP2MaxRows : 1];   // axis-1 records of the slab's rows
    const int t = threadIdx.x;
    const int p = p_base + blockIdx.y;
    const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
    int c2_lo = 0, c2_cnt = 0, base;
    if (A2) {
        c2_lo = blockIdx.x * kP2Out;
        c2_cnt = min(kP2Out, nc2 - c2_lo);
        base = __ldg(ax2.r0 + c2_lo) - 2;
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
    // per-thread constants of the axis-2 stencil
    double md2 = 0, ml2 = 0, mu2 = 0, wr2 = 0, wl2 = 0;
    int r02 = 0, rr2 = -1, rl2 = -1;
    if (A2 && in) {
        md2 = __ldg(ax2.md + j2);
        ml2 = __ldg(ax2.ml + j2);
        mu2 = __ldg(ax2.mu + j2);
    }
    if (A2 && t < c2_cnt) {
        const int c2 = c2_lo + t;
        r02 = __ldg(ax2.r0 + c2) - base;
        rr2 = __ldg(ax2.rr + c2);
        rl2 = __ldg(ax2.rl + c2);
        wr2 = __ldg(ax2.wr + c2);
        wl2 = __ldg(ax2.wl + c2);
    }
    auto out_row = [&](int c1, double w) {
        if (!A2) {
            if (in) bp[(int64_t)c1 * nc2 + j2] = w;
            return;
        }
        sw[t] = w;
        __syncthreads();
        double y = 0.0;
        if (in) {
            y = dmul(md2, sw[t]);
            if (j2 >= 1 && t >= 1) y = dadd(y, dmul(ml2, sw[t - 1]));
            if (j2 + 1 < n2 && t + 1 < kP2Threads) y = dadd(y, dmul(mu2, sw[t + 1]));
        }
        sy[t] = y;
        __syncthreads();
        if (t < c2_cnt) {
            double z = sy[r02];
            if (rr2 >= 0) z = dadd(z, dmul(wr2, sy[rr2 - base]));
            if (rl2 >= 0) z = dadd(z, dmul(wl2, sy[rl2 - base]));
            bp[(int64_t)c1 * nc2 + c2_lo + t] = z;
        }
    };
    int j_start, j_end;
    if (A1) {
        j_start = max(0, __ldg(ax1.r0 + c_lo) - 2);
        j_end = min(n1 - 1, __ldg(ax1.r0 + c_hi - 1) + 2);
    } else {
        j_start = c_lo;
        j_end = c_hi - 1;
    }
    // the slab's axis-1 PlaneInfo records, loaded once (the launcher bounds the rows per slab)
    const PlaneInfo *P1 = ax1.pi;
    if (A1 && j_end - j_start + 1 <= kP2MaxRows) {
        const int nrec = j_end - j_start + 1;
        const int4 *src = reinterpret_cast<const int4 *>(ax1.pi + j_start);
        int4 *dst = reinterpret_cast<int4 *>(ptab);
        for (int i = t; i < nrec * 5; i += kP2Threads) dst[i] = __ldg(src + i);
        __syncthreads();
        P1 = ptab - j_start;   // record k at P1 + k
    }
    const bool p1_shared = P1 != ax1.pi;
    // each thread streams its own column: no barrier needed for the ring itself
    auto issue = [&](int r) {
        if (r <= j_end && in) cp_async<8>(&ring[r % kP2Ring][t], zp + (int64_t)r * n2 + j2);
        cp_async_commit();
    };
    for (int k = 0; k < kP2Ring - 1; k++) issue(j_start + k);
    March M;
    march_init(M, c_lo, c_hi);
    for (int j = j_start; j <= j_end; j++) {
        cp_async_wait<kP2Ring - 2>();   // row j has landed (own copies)
        const double x = in ? ring[j % kP2Ring][t] : 0.0;
        issue(j + kP2Ring - 1);          // into the slot of row j - 1
        if (A1) {
            if (p1_shared) march_push<-1, false>(M, P1, n1, j, j_start, x, out_row);
            else march_push(M, ax1.pi, n1, j, j_start, x, out_row);
        } else {
            out_row(j, x);
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------- pass 2, 2 columns
// k_level_pass2<true, true> with two adjacent fine columns per thread (512 per block): the axis-1
// march control (record reads, emission test, ring wait) and the two barriers of each emitted row
// are paid once per two columns.  Same operation order.
constexpr int kP2Out2 = (2 * kP2Threads - 4) / 2;   // coarse outputs along axis 2 per block
constexpr int kP2Ring2 = 6;                         // rows in flight (shared memory < 48 KB)
constexpr int kP2MaxRows2 = 136;                    // fine rows per slab (<= 66 coarse outputs + stencil)

struct March2 {
    double m1[2], m2[2];
    double ya[2], yb[2], yc[2];
};

__global__ void __launch_bounds__(kP2Threads) k_level_pass2_x2(const double *__restrict__ Z0, int m0, int n1, int n2,
                                                               DevAxis ax1, DevAxis ax2, double *__restrict__ B,
                                                               int slabs1, int p_base) {
    constexpr int W = 2 * kP2Threads;
    __shared__ double sw[W];
    __shared__ double sy[W];
    __shared__ __align__(16) double ring[kP2Ring2][W];
    __shared__ __align__(16) PlaneInfo ptab[kP2MaxRows2];
    const int t = threadIdx.x;
    const int p = p_base + blockIdx.y;
    const int nc1 = ax1.nc, nc2 = ax2.nc;
    const int c2_lo = blockIdx.x * kP2Out2;
    const int c2_cnt = min(kP2Out2, nc2 - c2_lo);
    const int base = __ldg(ax2.r0 + c2_lo) - 2;
    const int jA = base + 2 * t, jB = jA + 1;   // this thread's fine columns
    const bool inA = jA >= 0 && jA < n2, inB = jB >= 0 && jB < n2;
    int c_lo, c_hi;
    slab_range(nc1, slabs1, blockIdx.z, c_lo, c_hi);
    if (c_lo >= c_hi) return;   // uniform across the block
    const double *zp = Z0 + (int64_t)p * n1 * n2;
    double *bp = B + (int64_t)p * nc1 * nc2;
    // axis-2 stencil constants: mass bands at the two columns, restriction of output t
    double md2[2] = {0, 0}, ml2[2] = {0, 0}, mu2[2] = {0, 0};
    if (inA) { md2[0] = __ldg(ax2.md + jA); ml2[0] = __ldg(ax2.ml + jA); mu2[0] = __ldg(ax2.mu + jA); }
    if (inB) { md2[1] = __ldg(ax2.md + jB); ml2[1] = __ldg(ax2.ml + jB); mu2[1] = __ldg(ax2.mu + jB); }
    double wr2 = 0, wl2 = 0;
    int r02 = 0, rr2 = -1, rl2 = -1;
    if (t < c2_cnt) {
        const int c2 = c2_lo + t;
        r02 = __ldg(ax2.r0 + c2) - base;
        rr2 = __ldg(ax2.rr + c2);
        rl2 = __ldg(ax2.rl + c2);
        wr2 = __ldg(ax2.wr + c2);
        wl2 = __ldg(ax2.wl + c2);
    }
    auto out_row = [&](int c1, double w0, double w1) {
        sw[2 * t] = w0;
        sw[2 * t + 1] = w1;
        __syncthreads();
        double y0 = 0.0, y1 = 0.0;
        const int l0 = 2 * t, l1 = 2 * t + 1;
        if (inA) {
            y0 = dmul(md2[0], sw[l0]);
            if (jA >= 1 && l0 >= 1) y0 = dadd(y0, dmul(ml2[0], sw[l0 - 1]));
            if (jA + 1 < n2) y0 = dadd(y0, dmul(mu2[0], sw[l0 + 1]));
        }
        if (inB) {
            y1 = dmul(md2[1], sw[l1]);
            if (jB >= 1) y1 = dadd(y1, dmul(ml2[1], sw[l1 - 1]));
            if (jB + 1 < n2 && l1 + 1 < W) y1 = dadd(y1, dmul(mu2[1], sw[l1 + 1]));
        }
        sy[l0] = y0;
        sy[l1] = y1;
        __syncthreads();
        if (t < c2_cnt) {
            double z = sy[r02];
            if (rr2 >= 0) z = dadd(z, dmul(wr2, sy[rr2 - base]));
            if (rl2 >= 0) z = dadd(z, dmul(wl2, sy[rl2 - base]));
            bp[(int64_t)c1 * nc2 + c2_lo + t] = z;
        }
    };
    const int j_start = max(0, __ldg(ax1.r0 + c_lo) - 2);
    const int j_end = min(n1 - 1, __ldg(ax1.r0 + c_hi - 1) + 2);
    {   // the slab's axis-1 records (the launcher bounds the rows per slab)
        const int nrec = j_end - j_start + 1;
        const int4 *src = reinterpret_cast<const int4 *>(ax1.pi + j_start);
        int4 *dst = reinterpret_cast<int4 *>(ptab);
        for (int i = t; i < nrec * 5; i += kP2Threads) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const PlaneInfo *P1 = ptab - j_start;   // record k at P1 + k
    const bool vec = ((((int64_t)n2 | base) & 1) == 0);   // 16-byte aligned column pairs
    auto issue = [&](int r) {
        if (r <= j_end) {
            const double *g = zp + (int64_t)r * n2 + jA;
            double *d = &ring[r % kP2Ring2][2 * t];
            if (vec && inA && inB) cp_async<16>(d, g);
            else {
                if (inA) cp_async<8>(d, g);
                if (inB) cp_async<8>(d + 1, g + 1);
            }
        }
        cp_async_commit();
    };
    for (int k = 0; k < kP2Ring2 - 1; k++) issue(j_start + k);
    March2 M;
#pragma unroll
    for (int k = 0; k < 2; k++) M.m1[k] = M.m2[k] = M.ya[k] = M.yb[k] = M.yc[k] = 0.0;
    // y(kk) for both columns and its emission (march_emit_y of fused.cu, two columns)
    auto emit_y = [&](int kk, const double *xk, const double *xkm1, const double *xkp1, bool has_up) {
        const PlaneInfo *pr = P1 + kk;
        double v[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            v[k] = dmul(pr->md, xk[k]);
            if (kk >= 1) v[k] = dadd(v[k], dmul(pr->ml, xkm1[k]));
            if (has_up) v[k] = dadd(v[k], dmul(pr->mu, xkp1[k]));
        }
        const int4 e = *reinterpret_cast<const int4 *>(&pr->fo);   // fo, emit, e_rr, e_rl
#pragma unroll
        for (int k = 0; k < 2; k++) {
            M.ya[k] = M.yb[k];
            M.yb[k] = M.yc[k];
            M.yc[k] = v[k];
        }
        if (e.y >= c_lo && e.y < c_hi) {
            const double wr = pr->ewr, wl = pr->ewl;
            double z[2];
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (e.z) {
                    z[k] = dadd(M.yb[k], dmul(wr, M.yc[k]));
                    if (e.w) z[k] = dadd(z[k], dmul(wl, M.ya[k]));
                } else {
                    z[k] = M.yc[k];
                    if (e.w) z[k] = dadd(z[k], dmul(wl, M.yb[k]));
                }
            }
            out_row(e.y, z[0], z[1]);
        }
    };
    for (int j = j_start; j <= j_end; j++) {
        cp_async_wait<kP2Ring2 - 2>();   // row j has landed (own copies)
        double x[2];
        x[0] = inA ? ring[j % kP2Ring2][2 * t] : 0.0;
        x[1] = inB ? ring[j % kP2Ring2][2 * t + 1] : 0.0;
        issue(j + kP2Ring2 - 1);          // into the slot of row j - 1
        // march_push: y(j - 1) once x(j) is known, y(j) at the last row
        if (j >= (j_start == 0 ? 1 : j_start + 2)) emit_y(j - 1, M.m1, M.m2, x, true);
        if (j == n1 - 1 && (j > j_start || j == 0)) {
            const double zero[2] = {0.0, 0.0};
            emit_y(j, x, M.m1, zero, false);
        }
#pragma unroll
        for (int k = 0; k < 2; k++) {
            M.m2[k] = M.m1[k];
            M.m1[k] = x[k];
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------- final
// Recompose output of one transition: D(j) = P(cv)(j) + mc(j) (transform.py:346-347), P the
// nested lerps over the corrected coarse values cv (nc0, nc1, nc2), mc from the coefficients.
// Each thread prefetches its own coefficient column through a private cp.async ring.
constexpr int kFRing = 8;

template <bool A0, bool A1, bool A2, typename TOut>
__global__ void __launch_bounds__(256) k_level_final(const double *__restrict__ cv, const double *__restrict__ corr,
                                                     int n0, int n1, int n2,
                                                     DevAxis ax0, DevAxis ax1, DevAxis ax2, LevelMap lm,
                                                     const double *__restrict__ coef, TOut *__restrict__ D, int j_base,
                                                     int j_count) {
    __shared__ __align__(16) double ring[kFRing][256];
    __shared__ double sP0[2][256];   // axis-0 GPK over the tile's coarse footprint, per plane (double-buffered)
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
    const int j2 = x0 + threadIdx.x, j1 = y0 + threadIdx.y;
    const bool act = j1 < n1 && j2 < n2;
    const int nc1 = A1 ? ax1.nc : n1, nc2 = A2 ? ax2.nc : n2;
    // coarse footprint of the tile: rows [r_lo, r_lo + R), columns [c_lo, c_lo + C)
    const int ylast = min(y0 + 7, n1 - 1), xlast = min(x0 + 31, n2 - 1);
    int r_lo = y0, r_hi = ylast, c_lo = x0, c_hi = xlast;
    if (A1) {
        r_lo = __ldg(ax1.pa + y0);
        const int pb = __ldg(ax1.pb + ylast);
        r_hi = max(__ldg(ax1.pa + ylast), pb);
    }
    if (A2) {
        c_lo = __ldg(ax2.pa + x0);
        const int pb = __ldg(ax2.pb + xlast);
        c_hi = max(__ldg(ax2.pa + xlast), pb);
    }
    const int C = c_hi - c_lo + 1, RC = (r_hi - r_lo + 1) * C;   // <= 6 x 18 (8 x 32 when an axis is inactive)
    const int fr = tid / max(C, 1), fc = tid - fr * max(C, 1);
    const int64_t cplane = (int64_t)nc1 * nc2;
    const int64_t foff = (int64_t)(r_lo + fr) * nc2 + (c_lo + fc);
    Nb b1{}, b2{};
    if (act) {
        b1 = neighbours<A1>(ax1, j1);
        b2 = neighbours<A2>(ax2, j2);
    }
    const int oa = (b1.ca - r_lo) * C, ob = (b1.cb - r_lo) * C, xa = b2.ca - c_lo, xb = b2.cb - c_lo;
    int lo, hi;
    slab_range(j_count, gridDim.z, blockIdx.z, lo, hi);   // fine planes [j_base, j_base + j_count)
    lo += j_base;
    hi += j_base;
    const int64_t col = (int64_t)j1 * n2 + j2;
    const int64_t fcol = act ? ((int64_t)__ldg(lm.m1 + j1)) * lm.D2 + __ldg(lm.m2 + j2) : 0;
    const int64_t fplane = lm.D1 * lm.D2;
    const bool col_fo = b1.fo || b2.fo;
    auto issue = [&](int j) {
        if (j < hi && act) {
            const bool fo0 = A0 && __ldg(ax0.pb + j) >= 0;
            if (fo0 || col_fo) cp_async<8>(&ring[j % kFRing][tid], coef + (int64_t)__ldg(lm.m0 + j) * fplane + fcol);
        }
        cp_async_commit();
    };
    // P0 of plane j over the footprint (transform.py:264-268: axis 0 first).  Each footprint thread
    // keeps the last two coarse planes it read (slot c & 1), so a coarse plane shared by consecutive
    // fine planes is loaded once; with corr the cached value is coarse - corr (the elementwise k_sub
    // of transform.py:345 folded in).
    int cc0 = -1, cc1 = -1;
    double cv0 = 0.0, cv1 = 0.0;
    auto coarse = [&](int c) -> double {
        if (c == cc0) return cv0;
        if (c == cc1) return cv1;
        const int64_t i = (int64_t)c * cplane + foff;
        double v = __ldg(cv + i);
        if (corr) v = dsub(v, __ldg(corr + i));
        if (c & 1) {
            cc1 = c;
            cv1 = v;
        } else {
            cc0 = c;
            cv0 = v;
        }
        return v;
    };
    auto stage = [&](int j) {
        if (j >= hi || tid >= RC) return;
        const Nb b0 = neighbours<A0>(ax0, j);
        const double va = coarse(b0.ca);
        sP0[j & 1][tid] = b0.fo ? lerp(va, coarse(b0.cb), b0.t) : va;
    };
    for (int k = 0; k < kFRing - 1; k++) issue(lo + k);
    stage(lo);
    for (int j = lo; j < hi; j++) {
        __syncthreads();                 // P0(j) visible; buffer (j + 1) & 1 free
        stage(j + 1);
        const bool fo0 = A0 && __ldg(ax0.pb + j) >= 0;
        double pred = 0.0;
        if (act) {
            const double *P = sP0[j & 1];
            double p1a = P[oa + xa];
            if (b1.fo) p1a = lerp(p1a, P[ob + xa], b1.t);
            pred = p1a;
            if (b2.fo) {
                double p1b = P[oa + xb];
                if (b1.fo) p1b = lerp(p1b, P[ob + xb], b1.t);
                pred = lerp(p1a, p1b, b2.t);
            }
        }
        const bool coarse_node = !fo0 && !col_fo;
        cp_async_wait<kFRing - 2>();
        const double mc = coarse_node ? 0.0 : ring[j % kFRing][tid];
        issue(j + kFRing - 1);
        if (act) D[(int64_t)j * n1 * n2 + col] = (TOut)dadd(pred, mc);
    }
    cp_async_wait<0>();
}

int slabs_for(int64_t cols, int planes) {
    const int64_t target = 148LL * 2048 * 2;
    int64_t s = (target + cols - 1) / std::max<int64_t>(cols, 1);
    return (int)std::max<int64_t>(1, std::min<int64_t>(s, std::max(planes, 1)));
}

template <int MODE, typename TIn>
void launch_pass1(int act, const TIn *F, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1,
                  const DevAxis &a2, const LevelMap &lm, double *coef, const double *coef_in, double *Z0, double *Cg,
                  const QuantOut &q, int c_base, int c_count, cudaStream_t s) {
    if (c_count <= 0) return;
    dim3 block(kTX, kTY);
    // two rows per thread for the all-active 3-D recompose transition (ncu at 513^3: 458 vs 509 us;
    // the quantizing decompose pass is faster with one row, 1297 vs 1466 us: register pressure)
    static const bool one_row = getenv("HPDR_P1_ONE_ROW") != nullptr;
    static const bool two_row_q = getenv("HPDR_P1_TWO_ROW") != nullptr;
    if constexpr (MODE == 1 || sizeof(TIn) == 4) {   // static shared memory < 48 KB
        if ((MODE == 1 || two_row_q) && !one_row && act == 7) {
            dim3 grid2((n2 + kTX - 1) / kTX, (n1 + kTY2 - 1) / kTY2, slabs_for((int64_t)n1 * n2, c_count));
            k_level_pass1_2r<MODE, true, true, true, TIn><<<grid2, block, 0, s>>>(
                F, n0, n1, n2, a0, a1, a2, lm, coef, coef_in, Z0, Cg, q, c_base, c_count);
            LAUNCH_CHECK();
            return;
        }
    }
    dim3 grid((n2 + kTX - 1) / kTX, (n1 + kTY - 1) / kTY, slabs_for((int64_t)n1 * n2, c_count));
    static const bool separable = getenv("HPDR_P1_SEPARABLE") != nullptr;
#define P1L(M)                                                                                                     \
    case M:                                                                                                        \
        if (MODE == 1 || !separable)                                                                               \
            k_level_pass1<MODE, (M & 1) != 0, (M & 2) != 0, (M & 4) != 0, TIn><<<grid, block, 0, s>>>(          \
                F, n0, n1, n2, a0, a1, a2, lm, coef, coef_in, Z0, Cg, q, c_base, c_count);                         \
        else                                                                                                       \
            k_level_pass1s<MODE == 1 ? 0 : MODE, (M & 1) != 0, (M & 2) != 0, (M & 4) != 0, TIn>                   \
                <<<grid, block, 0, s>>>(F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count);          \
        break;
    switch (act) { P1L(1) P1L(2) P1L(3) P1L(4) P1L(5) P1L(6) P1L(7) default: break; }
#undef P1L
    LAUNCH_CHECK();
}

void launch_pass2(int act, const double *Z0, int m0, int n1, int n2, const DevAxis &a1, const DevAxis &a2, double *B,
                  int p_base, int p_count, cudaStream_t s) {
    if (p_count <= 0) return;
    const bool A1 = act & 2, A2 = act & 4;
    const int nc1 = A1 ? a1.nc : n1, nc2 = A2 ? a2.nc : n2;
    const unsigned gx = A2 ? (unsigned)((nc2 + kP2Out - 1) / kP2Out) : (unsigned)((n2 + kP2Threads - 1) / kP2Threads);
    const int64_t cols = (int64_t)m0 * gx * kP2Threads;
    // enough slabs that a slab's rows fit the shared record table (<= 130 coarse rows each)
    const int slabs = std::max(slabs_for(cols, nc1), A1 ? (nc1 + 129) / 130 : 1);
    static const bool one_col = getenv("HPDR_P2_ONE_COL") != nullptr;
    if (A1 && A2 && !one_col) {   // two columns per thread
        const unsigned gx2 = (unsigned)((nc2 + kP2Out2 - 1) / kP2Out2);
        const int slabs2 = std::max(slabs_for((int64_t)m0 * gx2 * kP2Threads, nc1), (nc1 + 65) / 66);
        k_level_pass2_x2<<<dim3(gx2, (unsigned)p_count, (unsigned)slabs2), kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B,
                                                                                             slabs2, p_base);
        LAUNCH_CHECK();
        return;
    }
    dim3 grid(gx, (unsigned)p_count, (unsigned)slabs);
    if (A1 && A2) k_level_pass2<true, true><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs, p_base);
    else if (A1) k_level_pass2<true, false><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs, p_base);
    else if (A2) k_level_pass2<false, true><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs, p_base);
    else k_level_pass2<false, false><<<grid, kP2Threads, 0, s>>>(Z0, m0, n1, n2, a1, a2, B, slabs, p_base);
    LAUNCH_CHECK();
}

template <typename TOut>
void launch_final(int act, const double *cv, const double *corr, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1,
                  const DevAxis &a2, const LevelMap &lm, const double *coef, TOut *D, int j_base, int j_count,
                  cudaStream_t s) {
    if (j_count <= 0) return;
    dim3 grid((n2 + 31) / 32, (n1 + 7) / 8, slabs_for((int64_t)n1 * n2, j_count));
    dim3 block(32, 8);
#define FL(M)                                                                                                      \
    case M:                                                                                                        \
        k_level_final<(M & 1) != 0, (M & 2) != 0, (M & 4) != 0, TOut><<<grid, block, 0, s>>>(cv, corr, n0, n1, n2, a0, \
                                                                                              a1, a2, lm, coef, D, j_base, j_count); \
        break;
    switch (act) { FL(1) FL(2) FL(3) FL(4) FL(5) FL(6) FL(7) default: break; }
#undef FL
    LAUNCH_CHECK();
}

struct View {
    int n0, n1, n2, act;
    LevelMap lm;
};

View view_of(const DevPlan &p, int st_i) {
    const DevStep &st = p.steps[st_i];
    View v;
    v.n0 = (int)st.fsh.n[1];
    v.n1 = (int)st.fsh.n[2];
    v.n2 = (int)st.fsh.n[3];
    v.act = (st.ax[1].active ? 1 : 0) | (st.ax[2].active ? 2 : 0) | (st.ax[3].active ? 4 : 0);
    v.lm = LevelMap{p.map[1][st_i], p.map[2][st_i], p.map[3][st_i], p.dims.n[2], p.dims.n[3]};
    return v;
}

int64_t z0_size(const DevPlan &p, int st_i) {
    const DevStep &st = p.steps[st_i];
    return (int64_t)(st.ax[1].active ? st.ax[1].nc : st.fsh.n[1]) * st.fsh.n[2] * st.fsh.n[3];
}

}  // namespace

bool fused_supported(const DevPlan &p) { return p.dims.n[0] == 1; }

int fused_out_planes(const DevPlan &p, int st_i) {
    const DevStep &st = p.steps[st_i];
    return (int)(st.ax[1].active ? st.ax[1].nc : st.fsh.n[1]);
}

namespace {
int clamp_hi(const DevPlan &p, int st_i, int c_hi) {
    const int m = fused_out_planes(p, st_i);
    return c_hi < 0 || c_hi > m ? m : c_hi;
}
}  // namespace

void fused_pass1_decompose(const DevPlan &p, int st_i, const void *F, bool f32, double *coef, double *Z0, double *Cg,
                           cudaStream_t s, int c_lo, int c_hi) {
    const DevStep &st = p.steps[st_i];
    const View v = view_of(p, st_i);
    c_hi = clamp_hi(p, st_i, c_hi);
    const double frac = (double)(c_hi - c_lo) / fused_out_planes(p, st_i);
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    KPROF("k_level_pass1", frac * ((f32 ? 4.0 : 8.0) * nf + 8.0 * (nf - nc) + 8.0 * nc + 8.0 * z0_size(p, st_i)), s);
    const QuantOut q{};
    if (v.act == 7 && quad_eligible(p, st_i)) {
        if (f32) launch_pass1_quad<0, float>((const float *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                             coef, Z0, Cg, q, c_lo, c_hi - c_lo, s);
        else launch_pass1_quad<0, double>((const double *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                          coef, Z0, Cg, q, c_lo, c_hi - c_lo, s);
        return;
    }
    if (f32) launch_pass1<0, float>(v.act, (const float *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                    coef, nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
    else launch_pass1<0, double>(v.act, (const double *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                 coef, nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
}

void fused_pass1_quantize(const DevPlan &p, int st_i, const void *F, bool f32, const QuantOut &q, double *Z0,
                          double *Cg, cudaStream_t s, int c_lo, int c_hi) {
    const DevStep &st = p.steps[st_i];
    const View v = view_of(p, st_i);
    c_hi = clamp_hi(p, st_i, c_hi);
    const double frac = (double)(c_hi - c_lo) / fused_out_planes(p, st_i);
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    KPROF(st_i == 0 ? "k_level_pass1q" : "k_level_pass1q_coarse", frac * ((f32 ? 4.0 : 8.0) * nf + 2.0 * (nf - nc) + 8.0 * nc + 8.0 * z0_size(p, st_i)), s);
    // the quad kernel's plane ring pays off on large levels; tiny ones (latency-bound) take the
    // single-node kernel (HPDR_QUAD_MIN: smallest fine level, in nodes, that uses quads)
    static const int64_t quad_min = getenv("HPDR_QUAD_MIN") ? atoll(getenv("HPDR_QUAD_MIN")) : (1LL << 18);
    if (v.act == 7 && nf >= quad_min && quad_eligible(p, st_i)) {
        if (f32) launch_pass1_quad<2, float>((const float *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                             nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
        else launch_pass1_quad<2, double>((const double *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                          nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
        return;
    }
    if (f32) launch_pass1<2, float>(v.act, (const float *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                    nullptr, nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
    else launch_pass1<2, double>(v.act, (const double *)F, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm,
                                 nullptr, nullptr, Z0, Cg, q, c_lo, c_hi - c_lo, s);
}

void fused_pass1_recompose(const DevPlan &p, int st_i, const double *coef, double *Z0, cudaStream_t s, int c_lo,
                           int c_hi) {
    const DevStep &st = p.steps[st_i];
    const View v = view_of(p, st_i);
    c_hi = clamp_hi(p, st_i, c_hi);
    const double frac = (double)(c_hi - c_lo) / fused_out_planes(p, st_i);
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    KPROF("k_level_pass1r", frac * (8.0 * (nf - nc) + 8.0 * z0_size(p, st_i)), s);
    const QuantOut q{};
    // the finest transition (coef is dense in its own layout there): quads over coef planes
    static const bool no_quad_p1r = getenv("HPDR_NO_QUAD_P1R") != nullptr;
    if (st_i == 0 && v.act == 7 && !no_quad_p1r && quad_eligible(p, 0)) {
        launch_pass1_quad<1, double>(coef, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, nullptr, Z0, nullptr, q,
                                     c_lo, c_hi - c_lo, s);
        return;
    }
    launch_pass1<1, double>(v.act, nullptr, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, nullptr, coef, Z0,
                            nullptr, q, c_lo, c_hi - c_lo, s);
}

void quantize_fine(const DevPlan &p, const double *coef, const QuantOut &q, cudaStream_t s) {
    const DevStep &st = p.steps[0];
    const View v = view_of(p, 0);
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    KPROF("k_quantize_fine", 10.0 * (nf - nc), s);
    static const bool cols = getenv("HPDR_QF_COLUMNS") != nullptr;   // A/B: the column-walking kernel
    if (!cols && (int64_t)v.n0 * v.n1 < (1LL << 31)) {
        const unsigned g = (unsigned)kNumSMs * 8;
#define QR(M)                                                                                                      \
    case M:                                                                                                        \
        k_quantize_fine_rows<(M & 1) != 0, (M & 2) != 0, (M & 4) != 0><<<g, 256, 0, s>>>(coef, v.n0, v.n1, v.n2,   \
                                                                                        st.ax[1], st.ax[2],       \
                                                                                        st.ax[3], q);             \
        break;
        switch (v.act) { QR(1) QR(2) QR(3) QR(4) QR(5) QR(6) QR(7) default: break; }
#undef QR
        LAUNCH_CHECK();
        return;
    }
    dim3 grid((v.n2 + 31) / 32, (v.n1 + 7) / 8, slabs_for((int64_t)v.n1 * v.n2, v.n0));
    dim3 block(32, 8);
#define QF(M)                                                                                                      \
    case M:                                                                                                        \
        k_quantize_fine<(M & 1) != 0, (M & 2) != 0, (M & 4) != 0><<<grid, block, 0, s>>>(coef, v.n0, v.n1, v.n2,  \
                                                                                         st.ax[1], st.ax[2],      \
                                                                                         st.ax[3], q);            \
        break;
    switch (v.act) { QF(1) QF(2) QF(3) QF(4) QF(5) QF(6) QF(7) default: break; }
#undef QF
    LAUNCH_CHECK();
}

void quantize_coarsest(const DevPlan &p, const double *coarsest_vals, const QuantOut &q, cudaStream_t s) {
    const int n = (int)p.host.coarsest.size();
    KPROF("k_quantize_coarsest", 16.0 * n, s);
    k_quantize_coarsest<<<1, 32, 0, s>>>(coarsest_vals, p.coarsest, n, q);
    LAUNCH_CHECK();
}

void fused_pass2(const DevPlan &p, int st_i, const double *Z0, double *B, cudaStream_t s, int p_lo, int p_hi) {
    const DevStep &st = p.steps[st_i];
    const View v = view_of(p, st_i);
    const int m0 = fused_out_planes(p, st_i);
    p_hi = p_hi < 0 || p_hi > m0 ? m0 : p_hi;
    const double frac = (double)(p_hi - p_lo) / m0;
    KPROF("k_level_pass2", frac * (8.0 * m0 * v.n1 * v.n2 + 8.0 * st.csh.size()), s);
    launch_pass2(v.act, Z0, m0, v.n1, v.n2, st.ax[2], st.ax[3], B, p_lo, p_hi - p_lo, s);
}

void fused_final(const DevPlan &p, int st_i, const double *cv, const double *coef, void *D, int out_dtype,
                 cudaStream_t s, int j_lo, int j_hi, const double *corr) {
    const DevStep &st = p.steps[st_i];
    const View v = view_of(p, st_i);
    const int64_t nf = st.fsh.size(), nc = st.csh.size();
    if (j_hi < 0 || j_hi > v.n0) j_hi = v.n0;
    const double frac = (double)(j_hi - j_lo) / v.n0;
    KPROF("k_level_final", frac * ((corr ? 16.0 : 8.0) * nc + 8.0 * (nf - nc) + (out_dtype == 0 ? 4.0 : 8.0) * nf), s);
    static const bool no_quad_final = getenv("HPDR_NO_QUAD_FINAL") != nullptr;
    if (v.act == 7 && !no_quad_final && quad_eligible(p, st_i)) {
        if (out_dtype == 0)
            launch_final_quad<float>(cv, corr, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, coef, (float *)D,
                                     j_lo, j_hi - j_lo, s);
        else
            launch_final_quad<double>(cv, corr, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, coef, (double *)D,
                                      j_lo, j_hi - j_lo, s);
        return;
    }
    if (out_dtype == 0)
        launch_final<float>(v.act, cv, corr, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, coef, (float *)D, j_lo,
                            j_hi - j_lo, s);
    else
        launch_final<double>(v.act, cv, corr, v.n0, v.n1, v.n2, st.ax[1], st.ax[2], st.ax[3], v.lm, coef, (double *)D, j_lo,
                             j_hi - j_lo, s);
}

}  // namespace hpdr
