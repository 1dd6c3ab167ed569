// quad.cu -- the decomposition pass 1 of an all-axes-active 3-D transition with one 2 x 2 node quad
// per thread (k_pass1_quad), for the finest level and every coarser level whose axes are regular.
//
// Same contract and operation order as k_level_pass1 MODE 0 / 2 (fused.cu): mc = F - P(F) with
// the nested lerps of transform.py:264-268 (axis 0, then 1, then 2), the coarse-node gather, the
// coefficient write or quantize-on-write (quantize.py:73-84) + histogram, and the axis-0
// mass-multiply + restriction march (transform.py:206-226 then :181-203) -> Z0.
//
// Why a quad: on a regular axis (hierarchy.py:86-92: fine-only nodes are the odd j < n - 1, their
// coarse neighbours j - 1 and j + 1) the interpolant of the quad (r0, c0) .. (r0 + 1, c0 + 1), r0 and
// c0 even, only ever reads the axis-0 interpolant P0 at the four corners (r0 | rB) x (c0 | cB),
// rB = r0 + 2 (or r0 + 1 when that row is the coarse tail).  One thread evaluates those four P0
// values, the two axis-1 lerps and the two axis-2 lerps for all four nodes, and runs their four
// axis-0 marches with one copy of the per-plane control (record reads, emission test, ring wait).
// The per-node issue cost drops from ~300 to ~60 thread instructions (k_level_pass1 is issue-bound).
//
// Plane tiles (32 columns x 16 rows + one halo row / column on the high side) stream through an
// 8-slot shared-memory ring five planes ahead of the march:
//   TMA = true   one elected thread loads each plane with cp.async.bulk.tensor (3-D tensor map,
//                OOB zero fill) plus the plane's PlaneInfo record with cp.async.bulk, completing on
//                the slot's `full` mbarrier; warps release slots through `empty` mbarriers, so the
//                loop has no block-wide barrier.  Needs 16-byte aligned rows (n2 * sizeof(T) % 16 == 0).
//   TMA = false  every thread cp.async-copies its share of the tile (rows of any alignment, e.g.
//                513^3 fp32 or the dense fp64 coarse levels) and one __syncthreads per plane.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "level_dev.cuh"

namespace hpdr {

namespace {

using namespace lvl;

constexpr int kQX = 16, kQY = 8;                        // quads per block (x, y): 128 threads
constexpr int kQThreads = kQX * kQY;
constexpr int kTileX = 2 * kQX, kTileY = 2 * kQY;       // 32 x 16 nodes
constexpr int kRows = kTileY + 1;                       // + one halo row
constexpr int kQHist = 4096;

// Ring geometry (static shared memory, < 48 KB): fp32 planes 8 slots / 5 ahead, fp64 6 / 3.
template <typename T>
struct QuadGeom {
    static constexpr int pitch = sizeof(T) == 4 ? 36 : 34;   // row pitch: 33 used, 16-byte multiple
    static constexpr int slot_bytes = (kRows * pitch * (int)sizeof(T) + 127) / 128 * 128;
    static constexpr int slot_elems = slot_bytes / (int)sizeof(T);
    static constexpr int R = sizeof(T) == 4 ? 8 : 6;          // slots
    static constexpr int LA = R - 3;                          // planes issued ahead of the march
    static constexpr unsigned tile_bytes = kRows * pitch * sizeof(T);
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap *map, int x, int y, int z, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Predicated stores / shared-histogram increments (no branch, no reconvergence point).
__device__ __forceinline__ void st_u16_if(uint16_t *p, uint32_t v, bool c) {
    asm volatile("{.reg .pred p; setp.ne.b32 p, %2, 0; @p st.global.u16 [%0], %1;}" ::"l"(p), "h"((unsigned short)v),
                 "r"((int)c));
}
__device__ __forceinline__ void st_f64_if(double *p, double v, bool c) {
    asm volatile("{.reg .pred p; setp.ne.b32 p, %2, 0; @p st.global.f64 [%0], %1;}" ::"l"(p), "d"(v), "r"((int)c));
}
// A 64-bit base the compiler cannot re-associate with the per-node 32-bit offsets (one IMAD.WIDE each).
template <typename T>
__device__ __forceinline__ T *opaque(T *p) {
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

// (v0, v1) at an even element offset of a ring slot, widened to double.
__device__ __forceinline__ void ld2(const float *s, double &a, double &b) {
    const float2 v = *reinterpret_cast<const float2 *>(s);
    a = (double)v.x;
    b = (double)v.y;
}
__device__ __forceinline__ void ld2(const double *s, double &a, double &b) {
    const double2 v = *reinterpret_cast<const double2 *>(s);
    a = v.x;
    b = v.y;
}

// 4 blocks (16 warps) per SM; the cp.async producer needs more registers than 128, so that
// variant runs 3 blocks per SM without spills
template <int MODE, typename TIn, bool TMA, bool SH>
__global__ void __launch_bounds__(kQThreads, TMA ? 4 : 3)
    k_pass1_quad(const __grid_constant__ CUtensorMap tmap, const TIn *__restrict__ F, int n0, int n1, int n2,
                 DevAxis ax0, DevAxis ax1, DevAxis ax2, LevelMap lm, double *__restrict__ coef, double *__restrict__ Z0,
                 double *__restrict__ Cg, QuantOut q, int c_base, int c_count, int z0_vec) {
    using G = QuadGeom<TIn>;
    constexpr int R = G::R, LA = G::LA;
    __shared__ __align__(128) TIn ring[R * G::slot_elems];
    __shared__ __align__(16) PlaneInfo piring[R];
    __shared__ uint32_t sh_hist[MODE == 2 ? kQHist + 1 : 1];   // + a dummy bin
    __shared__ __align__(8) unsigned long long bars[2 * R];   // full[R], empty[R]
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr bool sh_ok = MODE == 2 && SH;   // dict <= 4096: shared-memory histogram
    const double rbin = MODE == 2 ? 1.0 / qbin(q) : 0.0;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += kQThreads) sh_hist[k] = 0;
    if (TMA && tid == 0) {
        for (int s = 0; s < R; s++) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[R + s]), kQThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int qx = tid & (kQX - 1), qy = tid / kQX;
    const int X0 = blockIdx.x * kTileX, Y0 = blockIdx.y * kTileY;
    const int c0 = X0 + 2 * qx, r0 = Y0 + 2 * qy;
    int c_lo, c_hi;
    slab_range(c_count, gridDim.z, blockIdx.z, c_lo, c_hi);
    c_lo += c_base;
    c_hi += c_base;
    int fl = 0;
    if (c_lo < c_hi) {   // uniform across the block
        int j_start, j_end, own_lo, own_hi;
        slab_planes<true>(ax0, n0, ax0.nc, c_lo, c_hi, j_start, j_end, own_lo, own_hi);
        const int nplanes = j_end - j_start + 1;
        const int plane = n1 * n2;   // < 2^31 (checked by the launcher)
        // ---- per-thread quad geometry (constant over the march)
        // node k: 0 (r0, c0), 1 (r0, c0 + 1), 2 (r0 + 1, c0), 3 (r0 + 1, c0 + 1); rows / columns r0, c0
        // are coarse (even), r0 + 1 / c0 + 1 fine-only unless they are the coarse tail
        const bool a00 = r0 < n1 && c0 < n2;
        const bool rowB = a00 && r0 + 1 < n1, colB = a00 && c0 + 1 < n2;
        const bool rowfo = rowB && __ldg(ax1.pb + r0 + 1) >= 0;
        const bool colfo = colB && __ldg(ax2.pb + c0 + 1) >= 0;
        const double t1 = rowfo ? __ldg(ax1.pt + r0 + 1) : 0.0;
        const double t2 = colfo ? __ldg(ax2.pt + c0 + 1) : 0.0;
        const int rB = rowfo ? r0 + 2 : (rowB ? r0 + 1 : r0);
        const int dcB = colfo ? 2 : (colB ? 1 : 0);
        // act: active nodes; nfo: fine-only within the plane (nodes 1-3), coarse nodes are 0 and the tails
        const unsigned act = (a00 ? 1u : 0u) | (colB ? 2u : 0u) | (rowB ? 4u : 0u) | (rowB && colB ? 8u : 0u);
        const unsigned nfo = (colfo ? 2u : 0u) | (rowfo ? 4u : 0u) | (rowfo || colfo ? 8u : 0u);
        const int so_r0 = (r0 - Y0) * G::pitch + (c0 - X0);   // element offsets within a slot
        const int so_rB = (rB - Y0) * G::pitch + (c0 - X0);
        const int col0 = r0 * n2 + c0;
        int fcol0 = 0, fd1 = 0, fd2 = 0, cgc0 = 0;
        if (a00) {
            const int m1a = __ldg(lm.m1 + r0), m2a = __ldg(lm.m2 + c0);
            fcol0 = m1a * (int)lm.D2 + m2a;
            if (rowB) fd1 = (__ldg(lm.m1 + r0 + 1) - m1a) * (int)lm.D2;
            if (colB) fd2 = __ldg(lm.m2 + c0 + 1) - m2a;
            cgc0 = __ldg(ax1.pa + r0) * ax2.nc + __ldg(ax2.pa + c0);
        }
        const int fcol[4] = {fcol0, fcol0 + fd2, fcol0 + fd1, fcol0 + fd1 + fd2};
        const int cgc[4] = {cgc0, cgc0 + 1, cgc0 + ax2.nc, cgc0 + ax2.nc + 1};   // consecutive coarse nodes
        const int64_t fplane = lm.D1 * lm.D2;
        const int64_t cgplane = (int64_t)ax1.nc * ax2.nc;

        // ---- producer side (non-TMA: warp w copies tile rows w, w + 4, ..., lane l column l, lane 0 also
        // column 32; row offsets are recomputed per plane, which is cheaper than holding them)
        const int warp = tid >> 5;
        const bool lane_in = X0 + lane < n2, col32_in = lane == 0 && X0 + kTileX < n2;
        const unsigned ring_s = smem_u32(ring), pir_s = smem_u32(piring);
        const unsigned full_s = smem_u32(bars), empty_s = full_s + R * 8;
        auto issue = [&](int i) {   // plane j_start + i into slot i % R
            const int p = j_start + i;
            const int s = i % R;
            if (TMA) {
                if (tid == 0 && i < nplanes) {
                    if (i >= R) mbar_wait(empty_s + s * 8, ((i / R) + 1) & 1);   // plane i - R released
                    const unsigned fb = full_s + s * 8;
                    mbar_expect_tx(fb, G::tile_bytes + (unsigned)sizeof(PlaneInfo));
                    tma_load_3d(ring_s + s * G::slot_bytes, &tmap, X0, Y0, p, fb);
                    bulk_load(pir_s + s * (unsigned)sizeof(PlaneInfo), ax0.pi + p, (unsigned)sizeof(PlaneInfo), fb);
                }
            } else {
                if (i < nplanes) {
                    const TIn *gp = F + (int64_t)p * plane + X0 + lane;
                    const unsigned sb = ring_s + s * G::slot_bytes + lane * (unsigned)sizeof(TIn);
#pragma unroll
                    for (int k = 0; k < (kRows + 3) / 4; k++) {
                        const int r = warp + 4 * k;
                        if (r < kRows && Y0 + r < n1) {
                            const TIn *g = gp + (Y0 + r) * n2;
                            const unsigned so = sb + r * G::pitch * (unsigned)sizeof(TIn);
                            if (lane_in) cp_async_s<sizeof(TIn)>(so, g);
                            if (col32_in) cp_async_s<sizeof(TIn)>(so + kTileX * (unsigned)sizeof(TIn), g + kTileX);
                        }
                    }
                    if (tid < 5)
                        cp_async_s<16>(pir_s + s * (unsigned)sizeof(PlaneInfo) + tid * 16,
                                       reinterpret_cast<const char *>(ax0.pi + p) + tid * 16);
                }
                cp_async_commit();
            }
        };

        // Four axis-0 marches (march_push of fused.cu).  Planes alternate parity, so the window
        // x(j-1), x(j-2) and y(k-2), y(k-1) is kept by parity (X[p], Y[p]) instead of shifted: every
        // step is instantiated for its parity and no march value is ever copied.
        double X[2][4], Y[2][4];
#pragma unroll
        for (int k = 0; k < 4; k++) X[0][k] = X[1][k] = Y[0][k] = Y[1][k] = 0.0;
        const int y_from = j_start == 0 ? 1 : j_start + 2;   // first j whose y(j - 1) is computable

        // restriction z(e.y) = (y(r0) + wr y(rr)) + wl y(rl) from the window (ya, yb, yc), stored to Z0
        auto restrict_out = [&](const PlaneInfo &P, const double *ya, const double *yb, const double *yc) {
            const int4 e = *reinterpret_cast<const int4 *>(&P.fo);   // fo, emit, e_rr, e_rl
            if (e.y >= c_lo && e.y < c_hi) {
                const double wr = P.ewr, wl = P.ewl;
                double z[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (e.z) {
                        z[k] = dadd(yb[k], dmul(wr, yc[k]));
                        if (e.w) z[k] = dadd(z[k], dmul(wl, ya[k]));
                    } else {
                        z[k] = yc[k];
                        if (e.w) z[k] = dadd(z[k], dmul(wl, yb[k]));
                    }
                }
                double *zp = Z0 + (int64_t)e.y * plane + col0;
                if (z0_vec) {   // rows even-aligned: (c0, c0 + 1) pairs as 16-byte stores
                    if (act & 2) *reinterpret_cast<double2 *>(zp) = make_double2(z[0], z[1]);
                    else if (act & 1) zp[0] = z[0];
                    if (act & 8) *reinterpret_cast<double2 *>(zp + n2) = make_double2(z[2], z[3]);
                    else if (act & 4) zp[n2] = z[2];
                } else {
                    if (act & 1) zp[0] = z[0];
                    if (act & 2) zp[1] = z[1];
                    if (act & 4) zp[n2] = z[2];
                    if (act & 8) zp[n2 + 1] = z[3];
                }
            }
        };
        // y(kk) = (md x(kk) + ml x(kk-1)) + mu x(kk+1) for the four marches
        auto y_of = [&](const PlaneInfo &P, int kk, const double *xk, const double *xkm1, const double *xkp1,
                        bool has_up, double *v) {
            const double md = P.md, ml = P.ml, mu = P.mu;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                v[k] = dmul(md, xk[k]);
                if (kk >= 1) v[k] = dadd(v[k], dmul(ml, xkm1[k]));
                if (has_up) v[k] = dadd(v[k], dmul(mu, xkp1[k]));
            }
        };

        // ---- prologue
#pragma unroll 1
        for (int i = 0; i < LA; i++) issue(i);
        if (!TMA) {
            cp_async_wait<LA - 1>();   // plane 0
            __syncthreads();
        } else {
            mbar_wait(full_s, 0);
        }
        int m0_next = __ldg(lm.m0 + j_start);

        auto step = [&](auto parity, int i) {
            constexpr int pe = decltype(parity)::value, po = 1 - pe;   // parity of j, of j - 1
            const int j = j_start + i;
            if (TMA) {
                issue(i + LA);
                if (i + 1 < nplanes) mbar_wait(full_s + ((unsigned)(i + 1) % R) * 8, ((unsigned)(i + 1) / R) & 1);
            } else {
                cp_async_wait<LA - 2>();   // planes <= i + 1 landed (own copies)
                __syncthreads();           // ... everyone's; slots of planes <= i - 2 free
                issue(i + LA);
            }
            const int m0j = m0_next;
            if (i + 1 < nplanes) m0_next = __ldg(lm.m0 + j + 1);
            const PlaneInfo &pj = piring[(unsigned)i % R];
            const int4 hd = *reinterpret_cast<const int4 *>(&pj);   // fa, fb, ca, cb
            const bool pfo = pj.fo != 0;
            const TIn *so = ring + ((unsigned)i % R) * G::slot_elems;
            double own[4], P00 = 0.0, P0B = 0.0, PB0 = 0.0, PBB = 0.0;
            ld2(so + so_r0, own[0], own[1]);
            ld2(so + so_r0 + G::pitch, own[2], own[3]);
            double mc[4];
            if constexpr (MODE == 1) {   // recompose: the coefficients of this level's fine-only nodes, 0 elsewhere
                const unsigned fm = act & (pfo ? 15u : nfo);
#pragma unroll
                for (int k = 0; k < 4; k++) mc[k] = ((fm >> k) & 1u) ? own[k] : 0.0;
            } else if (pfo) {   // fine-only plane: P0 = lerp(F[fa], F[fb], t0) at the four corners
                const double t0 = pj.t;
                const TIn *sa = ring + ((unsigned)(hd.x - j_start) % R) * G::slot_elems;
                const TIn *sb = ring + ((unsigned)(hd.y - j_start) % R) * G::slot_elems;
                P00 = lerp((double)sa[so_r0], (double)sb[so_r0], t0);
                P0B = lerp((double)sa[so_r0 + dcB], (double)sb[so_r0 + dcB], t0);
                PB0 = lerp((double)sa[so_rB], (double)sb[so_rB], t0);
                PBB = lerp((double)sa[so_rB + dcB], (double)sb[so_rB + dcB], t0);
            } else {
                P00 = own[0];
                P0B = (double)so[so_r0 + dcB];
                PB0 = (double)so[so_rB];
                PBB = (double)so[so_rB + dcB];
            }
            (void)P00, (void)P0B, (void)PB0, (void)PBB;   // MODE 1 interpolates nothing
            if constexpr (MODE != 1) {
                const double p1a = rowfo ? lerp(P00, PB0, t1) : PB0;
                const double p1b = rowfo ? lerp(P0B, PBB, t1) : PBB;
                mc[0] = dsub(own[0], P00);
                mc[1] = dsub(own[1], colfo ? lerp(P00, P0B, t2) : P0B);
                mc[2] = dsub(own[2], p1a);
                mc[3] = dsub(own[3], colfo ? lerp(p1a, p1b, t2) : p1b);
            }
            if (MODE != 1 && j >= own_lo && j < own_hi) {   // uniform
                const int64_t fb = (int64_t)m0j * fplane;
                const unsigned fine = act & (pfo ? 15u : nfo), coarse = act & ~fine;
                if (coarse) {
                    double *cgp = opaque(Cg + (int64_t)hd.z * cgplane);
#pragma unroll
                    for (int k = 0; k < 4; k++) st_f64_if(cgp + cgc[k], own[k], coarse & (1u << k));
                }
                if constexpr (MODE == 0) {
                    double *cp = opaque(coef + fb);
#pragma unroll
                    for (int k = 0; k < 4; k++) st_f64_if(cp + (unsigned)fcol[k], mc[k], fine & (1u << k));
                } else {
                    // fast path (quant_node for an in-range, comfortably rounded quotient), branch-free
                    uint16_t *kp = opaque(q.keys + fb);
                    unsigned slow = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const double qa = dmul(mc[k], rbin);
                        const double r = rint(qa);
                        // |r| < half bounds |qa| < 2^15: the fixed 2^-33 margin is stricter than quant_key's
                        // |qa| * 2^-49 (one multiply fewer; near-half quotients take the exact path)
                        const bool ok = fabs(dsub(qa, r)) < 0.5 - 0x1p-33 && fabs(r) < (double)q.half;   // (qa - r is exact)
                        const int ri = (int)r;
                        const uint32_t key = ((uint32_t)ri << 1) ^ (uint32_t)(ri >> 31);
                        const bool fk = (fine >> k) & 1u;
                        st_u16_if(kp + (unsigned)fcol[k], key, fk && ok);
                        if (sh_ok) atomicAdd(&sh_hist[fk && ok ? key : (uint32_t)kQHist], 1u);
                        else if (fk && ok) atomicAdd(&q.hist[key], 1ULL);
                        slow |= (fk && !ok) ? 1u << k : 0u;
                    }
                    if (slow) {   // outliers, near-half quotients, non-finite values: the full rule
#pragma unroll 1
                        for (int k = 0; k < 4; k++)
                            if (slow & (1u << k)) {
                                const double mk = k == 0 ? mc[0] : k == 1 ? mc[1] : k == 2 ? mc[2] : mc[3];
                                const int fk = fcol0 + ((k & 1) ? fd2 : 0) + ((k & 2) ? fd1 : 0);
                                quant_node(mk, q, rbin, fb + fk, fl, sh_hist, sh_ok);
                            }
                    }
                }
            }
            // axis-0 marches (march_push): y(j - 1) once x(j) is known, y(j) at the last plane
            if (j >= y_from) {
                const PlaneInfo &pm = piring[(unsigned)(i + R - 1) % R];
                double v[4];
                y_of(pm, j - 1, X[po], X[pe], mc, true, v);
                restrict_out(pm, Y[po], Y[pe], v);   // window y(j-3), y(j-2), y(j-1)
#pragma unroll
                for (int k = 0; k < 4; k++) Y[po][k] = v[k];
            }
            if (j == n0 - 1 && (j > j_start || j == 0)) {
                double v[4];
                y_of(pj, j, mc, X[po], mc, false, v);
                restrict_out(pj, Y[pe], Y[po], v);   // window y(j-2), y(j-1), y(j)
            }
#pragma unroll
            for (int k = 0; k < 4; k++) X[pe][k] = mc[k];
            if (TMA && i >= 1) {   // plane i - 1 is no longer read by this warp
                __syncwarp();
                if (lane == 0) mbar_arrive(empty_s + ((unsigned)(i - 1) % R) * 8);
            }
        };
        using P0 = std::integral_constant<int, 0>;
        using P1 = std::integral_constant<int, 1>;
        int i0 = 0;
        if (j_start & 1) step(P1{}, i0++);   // a slab may start on an odd plane (single-plane chunks)
#pragma unroll 1
        for (; i0 + 1 < nplanes; i0 += 2) {
            step(P0{}, i0);
            step(P1{}, i0 + 1);
        }
        if (i0 < nplanes) step(P0{}, i0);
        if (!TMA) cp_async_wait<0>();
    }
    if (MODE == 2) {
        if (fl) atomicOr(q.flags, fl);
        __syncthreads();
        if (sh_ok)
            for (uint32_t k = tid; k < q.dict; k += kQThreads) {
                const uint32_t c = sh_hist[k];
                if (c) atomicAdd(&q.hist[k], (unsigned long long)c);
            }
    }
}

// ---- host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &qr) !=
                cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <typename TIn>
bool make_tmap(CUtensorMap &m, const TIn *F, int n0, int n1, int n2) {
    auto enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
    const cuuint64_t strides[2] = {(cuuint64_t)n2 * sizeof(TIn), (cuuint64_t)n1 * n2 * sizeof(TIn)};
    const cuuint32_t box[3] = {(cuuint32_t)QuadGeom<TIn>::pitch, (cuuint32_t)kRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&m, sizeof(TIn) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                           const_cast<TIn *>(F), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int MODE, typename TIn, bool TMA, bool SH>
void launch_one(dim3 grid, const CUtensorMap &tm, const TIn *F, int n0, int n1, int n2, const DevAxis &a0,
                const DevAxis &a1, const DevAxis &a2, const LevelMap &lm, double *coef, double *Z0, double *Cg,
                const QuantOut &q, int c_base, int c_count, int z0_vec, cudaStream_t s) {
    k_pass1_quad<MODE, TIn, TMA, SH><<<grid, kQThreads, 0, s>>>(tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q,
                                                               c_base, c_count, z0_vec);
}

// Every axis regular: fine-only nodes are odd with coarse neighbours j -/+ 1, other nodes their own.
bool axis_regular(const AxisTables &t) {
    if (!t.active) return false;
    for (int64_t j = 0; j < t.n; j++) {
        const bool fo = t.pb[j] >= 0;
        if (fo ? ((j & 1) == 0 || t.fa[j] != j - 1 || t.fb[j] != j + 1) : (t.fa[j] != j || t.fb[j] != j))
            return false;
    }
    return true;
}

// ---------------------------------------------------------------------------------- final (quads)
// Recompose output of a regular all-active transition, one 2 x 2 node quad per thread:
// D = P(cv - corr) + mc (transform.py:345-347) with P the nested lerps of transform.py:264-268.
// The quad's interpolant reads the axis-0 interpolant P0 only at its four coarse corners, so each
// thread forms those itself from the two coarse planes around the fine plane (cv - corr, cached per
// corner for the next fine plane) -- no shared footprint and no barrier -- and the coefficients of
// the next plane are loaded one plane ahead.  Same values and operation order as k_level_final.
// block shape: 64 x 2 quads (128 x 4 nodes): a row of the tile is 1 KB of contiguous coefficients
constexpr int kFQX = 64, kFQY = 2;
template <typename TOut>
__global__ void __launch_bounds__(kQThreads) k_final_quad(const double *__restrict__ cv, const double *__restrict__ corr,
                                                         int n0, int n1, int n2, DevAxis ax0, DevAxis ax1, DevAxis ax2,
                                                         LevelMap lm, const double *__restrict__ coef,
                                                         TOut *__restrict__ D, int j_base, int j_count) {
    const int tid = threadIdx.x;
    const int qx = tid & (kFQX - 1), qy = tid / kFQX;
    const int c0 = blockIdx.x * (2 * kFQX) + 2 * qx, r0 = blockIdx.y * (2 * kFQY) + 2 * qy;
    if (r0 >= n1 || c0 >= n2) return;   // no barriers below
    int lo, hi;
    slab_range(j_count, gridDim.z, blockIdx.z, lo, hi);
    lo += j_base;
    hi += j_base;
    const bool rowB = r0 + 1 < n1, colB = c0 + 1 < n2;
    const bool rowfo = rowB && __ldg(ax1.pb + r0 + 1) >= 0;
    const bool colfo = colB && __ldg(ax2.pb + c0 + 1) >= 0;
    const double t1 = rowfo ? __ldg(ax1.pt + r0 + 1) : 0.0;
    const double t2 = colfo ? __ldg(ax2.pt + c0 + 1) : 0.0;
    // coarse corners: rows cy0 / cyB, columns cx0 / cxB (the coarse neighbours of r0 + 1 / c0 + 1)
    const int nc2 = ax2.nc;
    const int cy0 = __ldg(ax1.pa + r0), cx0 = __ldg(ax2.pa + c0);
    const int cyB = rowfo ? __ldg(ax1.pb + r0 + 1) : (rowB ? __ldg(ax1.pa + r0 + 1) : cy0);
    const int cxB = colfo ? __ldg(ax2.pb + c0 + 1) : (colB ? __ldg(ax2.pa + c0 + 1) : cx0);
    const int64_t cplane = (int64_t)ax1.nc * nc2;
    const int64_t co[4] = {(int64_t)cy0 * nc2 + cx0, (int64_t)cy0 * nc2 + cxB, (int64_t)cyB * nc2 + cx0,
                           (int64_t)cyB * nc2 + cxB};
    // finest offsets of the four nodes within a finest plane; node k: (r0 | r0 + 1) x (c0 | c0 + 1)
    const int64_t m1a = __ldg(lm.m1 + r0), m2a = __ldg(lm.m2 + c0);
    const int64_t f00 = m1a * lm.D2 + m2a;
    const int64_t fd1 = rowB ? (__ldg(lm.m1 + r0 + 1) - m1a) * lm.D2 : 0, fd2 = colB ? __ldg(lm.m2 + c0 + 1) - m2a : 0;
    const unsigned act = 1u | (colB ? 2u : 0u) | (rowB ? 4u : 0u) | (rowB && colB ? 8u : 0u);
    const unsigned cfo = (colfo ? 2u : 0u) | (rowfo ? 4u : 0u) | (rowfo || colfo ? 8u : 0u);   // fine-only in-plane
    const int64_t fplane = lm.D1 * lm.D2;
    // coarse - corr at the four corners of coarse plane c; the even and the odd plane last read are
    // kept (a coarse plane serves up to three consecutive fine planes)
    int ce = -1, cod = -1;
    double ve[4], vo[4];
    auto fetch = [&](int c, double *v) {
        const double *b = cv + (int64_t)c * cplane;
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = __ldg(b + co[k]);
        if (corr) {   // coarse - corr (the elementwise k_sub folded in)
            const double *r = corr + (int64_t)c * cplane;
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = dsub(v[k], __ldg(r + co[k]));
        }
    };
    auto corners = [&](int c, double *v) {
        if (c & 1) {
            if (cod != c) {
                cod = c;
                fetch(c, vo);
            }
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = vo[k];
        } else {
            if (ce != c) {
                ce = c;
                fetch(c, ve);
            }
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = ve[k];
        }
    };
    auto load_mc = [&](int j, double *m) {
        const unsigned need = act & (__ldg(ax0.pb + j) >= 0 ? 15u : cfo);
        const double *cp = coef + (int64_t)__ldg(lm.m0 + j) * fplane;
        m[0] = (need & 1u) ? __ldg(cp + f00) : 0.0;
        m[1] = (need & 2u) ? __ldg(cp + f00 + fd2) : 0.0;
        m[2] = (need & 4u) ? __ldg(cp + f00 + fd1) : 0.0;
        m[3] = (need & 8u) ? __ldg(cp + f00 + fd1 + fd2) : 0.0;
    };
    double mcn[4];
    if (lo < hi) load_mc(lo, mcn);
    for (int j = lo; j < hi; j++) {
        double mc[4];
#pragma unroll
        for (int k = 0; k < 4; k++) mc[k] = mcn[k];
        if (j + 1 < hi) load_mc(j + 1, mcn);   // one plane ahead
        const int pb0 = __ldg(ax0.pb + j);
        const int ca = __ldg(ax0.pa + j);
        double P[4];
        corners(ca, P);
        if (pb0 >= 0) {   // fine-only plane: P0 = lerp(cv[ca], cv[cb], t0) at the corners
            const double t0 = __ldg(ax0.pt + j);
            double Q[4];
            corners(pb0, Q);
#pragma unroll
            for (int k = 0; k < 4; k++) P[k] = lerp(P[k], Q[k], t0);
        }
        // P[0] = P00, P[1] = P0B, P[2] = PB0, P[3] = PBB
        const double p1a = rowfo ? lerp(P[0], P[2], t1) : P[2];
        const double p1b = rowfo ? lerp(P[1], P[3], t1) : P[3];
        const double pred[4] = {P[0], colfo ? lerp(P[0], P[1], t2) : P[1], p1a, colfo ? lerp(p1a, p1b, t2) : p1b};
        TOut *dp = D + (int64_t)j * n1 * n2 + (int64_t)r0 * n2 + c0;
        dp[0] = (TOut)dadd(pred[0], mc[0]);
        if (act & 2u) dp[1] = (TOut)dadd(pred[1], mc[1]);
        if (act & 4u) dp[n2] = (TOut)dadd(pred[2], mc[2]);
        if (act & 8u) dp[n2 + 1] = (TOut)dadd(pred[3], mc[3]);
    }
}

}  // namespace

bool quad_eligible(const DevPlan &p, int st_i) {
    const StepTables &h = p.host.steps[st_i];
    const DevStep &st = p.steps[st_i];
    if (p.dims.n[0] != 1) return false;
    const int64_t n1 = st.fsh.n[2], n2 = st.fsh.n[3];
    if (n1 * n2 >= (1LL << 31) || p.dims.n[2] * p.dims.n[3] >= (1LL << 31)) return false;
    if (getenv("HPDR_NO_QUAD")) return false;
    return axis_regular(h.ax[1]) && axis_regular(h.ax[2]) && axis_regular(h.ax[3]);
}

template <typename TOut>
void launch_final_quad(const double *cv, const double *corr, int n0, int n1, int n2, const DevAxis &a0,
                       const DevAxis &a1, const DevAxis &a2, const LevelMap &lm, const double *coef, TOut *D, int j_base,
                       int j_count, cudaStream_t s) {
    if (j_count <= 0) return;
    const unsigned gx = (n2 + 2 * kFQX - 1) / (2 * kFQX), gy = (n1 + 2 * kFQY - 1) / (2 * kFQY);
    const int64_t want = 148LL * 12 * 4;   // >= 4 waves of 12 resident blocks per SM
    const int slabs = (int)std::max<int64_t>(1, std::min<int64_t>(j_count, (want + (int64_t)gx * gy - 1) / ((int64_t)gx * gy)));
    k_final_quad<TOut><<<dim3(gx, gy, (unsigned)slabs), kQThreads, 0, s>>>(cv, corr, n0, n1, n2, a0, a1, a2, lm, coef, D,
                                                                          j_base, j_count);
    LAUNCH_CHECK();
}
template void launch_final_quad<float>(const double *, const double *, int, int, int, const DevAxis &, const DevAxis &,
                                       const DevAxis &, const LevelMap &, const double *, float *, int, int, cudaStream_t);
template void launch_final_quad<double>(const double *, const double *, int, int, int, const DevAxis &, const DevAxis &,
                                        const DevAxis &, const LevelMap &, const double *, double *, int, int,
                                        cudaStream_t);

template <int MODE, typename TIn>
void launch_pass1_quad(const TIn *F, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1, const DevAxis &a2,
                       const LevelMap &lm, double *coef, double *Z0, double *Cg, const QuantOut &q, int c_base,
                       int c_count, cudaStream_t s) {
    if (c_count <= 0) return;
    const unsigned gx = (n2 + kTileX - 1) / kTileX, gy = (n1 + kTileY - 1) / kTileY;
    static const int slab_env = getenv("HPDR_QUAD_SLABS") ? atoi(getenv("HPDR_QUAD_SLABS")) : 0;
    const int64_t want = 148LL * 4 * 8;   // >= 8 waves of 4 resident blocks per SM
    int slabs = slab_env > 0 ? slab_env : (int)((want + (int64_t)gx * gy - 1) / ((int64_t)gx * gy));
    // >= 8 coarse planes per slab when that still fills the GPU; small grids (latency-bound marches)
    // go down to 2
    const int min_planes = (int64_t)gx * gy * std::max(1, c_count / 8) >= want ? 8 : 2;
    slabs = std::max(1, std::min(slabs, std::max(1, c_count / min_planes)));
    // every block flushes its shared histogram: no more than ~4 blocks per SM on small grids
    if (slab_env <= 0 && min_planes == 2)
        slabs = std::max(1, std::min<int>(slabs, (int)std::max<int64_t>(1, 148LL * 4 / ((int64_t)gx * gy))));
    const dim3 grid(gx, gy, (unsigned)slabs);
    const int z0_vec = ((int64_t)n1 * n2 % 2 == 0 && n2 % 2 == 0) ? 1 : 0;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    static const bool no_tma = getenv("HPDR_NO_TMA") != nullptr;
    const bool tma = !no_tma && ((int64_t)n2 * sizeof(TIn)) % 16 == 0 && ((uintptr_t)F & 15) == 0 &&
                     make_tmap(tm, F, n0, n1, n2);
    const bool sh = MODE == 2 && q.dict <= (uint32_t)kQHist;
    if (tma) {
        if (sh) launch_one<MODE, TIn, true, true>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec, s);
        else launch_one<MODE, TIn, true, false>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec, s);
    } else {
        if (sh) launch_one<MODE, TIn, false, true>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec, s);
        else launch_one<MODE, TIn, false, false>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec, s);
    }
    LAUNCH_CHECK();
}

template void launch_pass1_quad<0, float>(const float *, int, int, int, const DevAxis &, const DevAxis &,
                                          const DevAxis &, const LevelMap &, double *, double *, double *,
                                          const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<0, double>(const double *, int, int, int, const DevAxis &, const DevAxis &,
                                           const DevAxis &, const LevelMap &, double *, double *, double *,
                                           const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<1, double>(const double *, int, int, int, const DevAxis &, const DevAxis &,
                                           const DevAxis &, const LevelMap &, double *, double *, double *,
                                           const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<2, float>(const float *, int, int, int, const DevAxis &, const DevAxis &,
                                          const DevAxis &, const LevelMap &, double *, double *, double *,
                                          const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<2, double>(const double *, int, int, int, const DevAxis &, const DevAxis &,
                                           const DevAxis &, const LevelMap &, double *, double *, double *,
                                           const QuantOut &, int, int, cudaStream_t);

}  // namespace hpdr
