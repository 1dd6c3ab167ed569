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

#include <mutex>

#include "level_dev.cuh"

namespace hpdr {

namespace {

using namespace lvl;

constexpr int kQX = 16, kQY = 8;                        // quads per block (x, y): 128 threads
constexpr int kTileX = 2 * kQX, kTileY = 2 * kQY;       // 32 x 16 nodes
constexpr int kRows = kTileY + 1;                       // + one halo row
constexpr int kQRing = 8;                               // ring slots (power of two)
constexpr int kLook = 5;                                // planes issued ahead of the march
constexpr int kQHist = 4096;

template <typename T>
struct QuadGeom {
    static constexpr int pitch = sizeof(T) == 4 ? 36 : 34;   // row pitch: 33 used, 16-byte multiple
    static constexpr int slot_elems = kRows * pitch;
    static constexpr int slot_bytes = (slot_elems * (int)sizeof(T) + 127) / 128 * 128;
    static constexpr int ring_bytes = kQRing * slot_bytes;
    static constexpr int pi_off = ring_bytes;                           // PlaneInfo ring
    static constexpr int hist_off = pi_off + kQRing * (int)sizeof(PlaneInfo);
    static constexpr int bar_off = hist_off + kQHist * 4;               // full[8], empty[8]
    static constexpr int smem = bar_off + 2 * kQRing * 8;
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

template <typename T>
__device__ __forceinline__ double ld1(const T *s) { return (double)*s; }

// Four marches along axis 0 sharing one PlaneInfo stream (march_push of fused.cu, unrolled x4).
struct Quad4 {
    double m1[4], m2[4], ya[4], yb[4], yc[4];
};

template <int MODE, typename TIn, bool TMA>
__global__ void __launch_bounds__(kQX *kQY, 4)
    k_pass1_quad(const __grid_constant__ CUtensorMap tmap, const TIn *__restrict__ F, int n0, int n1, int n2,
                 DevAxis ax0, DevAxis ax1, DevAxis ax2, LevelMap lm, double *__restrict__ coef, double *__restrict__ Z0,
                 double *__restrict__ Cg, QuantOut q, int c_base, int c_count, int z0_vec) {
    using G = QuadGeom<TIn>;
    extern __shared__ __align__(128) unsigned char smem[];
    TIn *ring = reinterpret_cast<TIn *>(smem);
    const PlaneInfo *piring = reinterpret_cast<const PlaneInfo *>(smem + G::pi_off);
    uint32_t *sh_hist = reinterpret_cast<uint32_t *>(smem + G::hist_off);
    const unsigned ring_s = smem_u32(smem), pir_s = ring_s + G::pi_off;
    const unsigned full_s = ring_s + G::bar_off, empty_s = full_s + kQRing * 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool sh_ok = MODE == 2 && q.dict <= kQHist;
    const double rbin = MODE == 2 ? 1.0 / qbin(q) : 0.0;
    if (MODE == 2 && sh_ok)
        for (uint32_t k = tid; k < q.dict; k += kQX * kQY) sh_hist[k] = 0;
    if (TMA && tid == 0) {
        for (int s = 0; s < kQRing; s++) {
            mbar_init(full_s + s * 8, 1);
            mbar_init(empty_s + s * 8, (kQX * kQY) / 32);
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
        const bool a00 = r0 < n1 && c0 < n2;
        const bool rowB = r0 + 1 < n1, colB = c0 + 1 < n2;
        bool rowfo = false, colfo = false;
        double t1 = 0.0, t2 = 0.0;
        if (a00 && rowB) {
            rowfo = __ldg(ax1.pb + r0 + 1) >= 0;
            if (rowfo) t1 = __ldg(ax1.pt + r0 + 1);
        }
        if (a00 && colB) {
            colfo = __ldg(ax2.pb + c0 + 1) >= 0;
            if (colfo) t2 = __ldg(ax2.pt + c0 + 1);
        }
        const int rB = rowfo ? r0 + 2 : (rowB ? r0 + 1 : r0);
        const int cB = colfo ? c0 + 2 : (colB ? c0 + 1 : c0);
        // node k: 0 (r0, c0), 1 (r0, c0 + 1), 2 (r0 + 1, c0), 3 (r0 + 1, c0 + 1)
        bool act[4];
        act[0] = a00;
        act[1] = a00 && colB;
        act[2] = a00 && rowB;
        act[3] = a00 && rowB && colB;
        const bool nfo[4] = {false, colfo, rowfo, rowfo || colfo};   // fine-only within the plane
        const int so_r0 = (r0 - Y0) * G::pitch + (c0 - X0);          // smem offsets within a slot
        const int so_r1 = so_r0 + G::pitch;
        const int so_rB = (rB - Y0) * G::pitch + (c0 - X0);
        const int dcB = cB - c0;
        int col[4], fcol[4], cgc[4];
        {
            const int rr[4] = {r0, r0, r0 + 1, r0 + 1}, cc[4] = {c0, c0 + 1, c0, c0 + 1};
            const int nc2 = ax2.nc;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                col[k] = rr[k] * n2 + cc[k];
                fcol[k] = act[k] ? __ldg(lm.m1 + rr[k]) * (int)lm.D2 + __ldg(lm.m2 + cc[k]) : 0;
                cgc[k] = act[k] ? __ldg(ax1.pa + rr[k]) * nc2 + __ldg(ax2.pa + cc[k]) : 0;
            }
        }
        const int64_t fplane = lm.D1 * lm.D2;
        const int64_t cgplane = (int64_t)ax1.nc * ax2.nc;

        // ---- producer side
        auto slot_of = [&](int i) { return i & (kQRing - 1); };
        // non-TMA: this thread's share of a tile (33 columns x 17 rows)
        constexpr int kTileElems = kRows * (kTileX + 1);
        constexpr int kPer = (kTileElems + kQX * kQY - 1) / (kQX * kQY);
        int ld_s[kPer], ld_g[kPer];
        if (!TMA) {
#pragma unroll
            for (int k = 0; k < kPer; k++) {
                const int e = tid + k * kQX * kQY;
                const int yy = e / (kTileX + 1), xx = e - yy * (kTileX + 1);
                const bool ok = e < kTileElems && Y0 + yy < n1 && X0 + xx < n2;
                ld_s[k] = ok ? (yy * G::pitch + xx) * (int)sizeof(TIn) : -1;
                ld_g[k] = (Y0 + yy) * n2 + X0 + xx;
            }
        }
        auto issue = [&](int i) {   // plane j_start + i into its slot
            const int p = j_start + i;
            const int s = slot_of(i);
            if (TMA) {
                if (tid == 0 && i < nplanes) {
                    if (i >= kQRing) mbar_wait(empty_s + s * 8, ((i >> 3) + 1) & 1);   // plane i - 8 released
                    const unsigned fb = full_s + s * 8;
                    mbar_expect_tx(fb, (unsigned)(kRows * G::pitch * sizeof(TIn) + sizeof(PlaneInfo)));
                    tma_load_3d(ring_s + s * G::slot_bytes, &tmap, X0, Y0, p, fb);
                    bulk_load(pir_s + s * (unsigned)sizeof(PlaneInfo), ax0.pi + p, (unsigned)sizeof(PlaneInfo), fb);
                }
            } else {
                if (i < nplanes) {
                    const TIn *gp = F + (int64_t)p * plane;
                    const unsigned sb = ring_s + s * G::slot_bytes;
#pragma unroll
                    for (int k = 0; k < kPer; k++)
                        if (ld_s[k] >= 0) cp_async_s<sizeof(TIn)>(sb + ld_s[k], gp + ld_g[k]);
                    if (tid < 5)
                        cp_async_s<16>(pir_s + s * (unsigned)sizeof(PlaneInfo) + tid * 16,
                                       reinterpret_cast<const char *>(ax0.pi + p) + tid * 16);
                }
                cp_async_commit();
            }
        };
        auto wait_plane = [&](int i) {   // TMA: plane i has landed
            if (TMA && i < nplanes) mbar_wait(full_s + slot_of(i) * 8, (i >> 3) & 1);
        };

        Quad4 M;
#pragma unroll
        for (int k = 0; k < 4; k++) M.m1[k] = M.m2[k] = M.ya[k] = M.yb[k] = M.yc[k] = 0.0;
        const int y_from = j_start == 0 ? 1 : j_start + 2;   // first j whose y(j - 1) is computable

        // one y(k) per march from record P: y = (md x_k + ml x_{k-1}) + mu x_{k+1}, then emission
        auto emit_y = [&](const PlaneInfo *P, int kk, const double *xk, const double *xkm1, const double *xkp1,
                          bool has_up) {
            const double md = P->md, ml = P->ml, mu = P->mu;
            const int4 e = *reinterpret_cast<const int4 *>(&P->fo);   // fo, emit, e_rr, e_rl
            double v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                v[k] = dmul(md, xk[k]);
                if (kk >= 1) v[k] = dadd(v[k], dmul(ml, xkm1[k]));
                if (has_up) v[k] = dadd(v[k], dmul(mu, xkp1[k]));
                M.ya[k] = M.yb[k];
                M.yb[k] = M.yc[k];
                M.yc[k] = v[k];
            }
            if (e.y >= c_lo && e.y < c_hi) {
                const double wr = P->ewr, wl = P->ewl;
                double z[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (e.z) {
                        z[k] = dadd(M.yb[k], dmul(wr, M.yc[k]));
                        if (e.w) z[k] = dadd(z[k], dmul(wl, M.ya[k]));
                    } else {
                        z[k] = M.yc[k];
                        if (e.w) z[k] = dadd(z[k], dmul(wl, M.yb[k]));
                    }
                }
                double *zp = Z0 + (int64_t)e.y * plane;
                if (z0_vec) {   // rows even-aligned: (c0, c0 + 1) pairs as 16-byte stores
                    if (act[1]) *reinterpret_cast<double2 *>(zp + col[0]) = make_double2(z[0], z[1]);
                    else if (act[0]) zp[col[0]] = z[0];
                    if (act[3]) *reinterpret_cast<double2 *>(zp + col[2]) = make_double2(z[2], z[3]);
                    else if (act[2]) zp[col[2]] = z[2];
                } else {
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        if (act[k]) zp[col[k]] = z[k];
                }
            }
        };

        // ---- prologue
#pragma unroll 1
        for (int i = 0; i < kLook; i++) issue(i);
        if (!TMA) {
            cp_async_wait<kLook - 1>();   // plane 0
            __syncthreads();
        }
        wait_plane(0);

#pragma unroll 1
        for (int i = 0; i < nplanes; i++) {
            const int j = j_start + i;
            if (TMA) {
                issue(i + kLook);
                wait_plane(i + 1);
            } else {
                cp_async_wait<kLook - 2>();   // planes <= i + 1 landed (own copies)
                __syncthreads();              // ... everyone's; slots of planes <= i - 2 free
                issue(i + kLook);
            }
            const PlaneInfo *pj = piring + slot_of(i);
            const int4 hd = *reinterpret_cast<const int4 *>(pj);   // fa, fb, ca, cb
            const bool pfo = pj->fo != 0;
            const TIn *so = ring + slot_of(i) * (G::slot_bytes / (int)sizeof(TIn));
            double own[4], P00, P0B, PB0, PBB;
            own[0] = ld1(so + so_r0);
            own[1] = ld1(so + so_r0 + 1);
            own[2] = ld1(so + so_r1);
            own[3] = ld1(so + so_r1 + 1);
            if (pfo) {   // fine-only plane: P0 = lerp(F[fa], F[fb], t0) at the four corners
                const double t0 = pj->t;
                const TIn *sa = ring + slot_of(hd.x - j_start) * (G::slot_bytes / (int)sizeof(TIn));
                const TIn *sb = ring + slot_of(hd.y - j_start) * (G::slot_bytes / (int)sizeof(TIn));
                P00 = lerp(ld1(sa + so_r0), ld1(sb + so_r0), t0);
                P0B = lerp(ld1(sa + so_r0 + dcB), ld1(sb + so_r0 + dcB), t0);
                PB0 = lerp(ld1(sa + so_rB), ld1(sb + so_rB), t0);
                PBB = lerp(ld1(sa + so_rB + dcB), ld1(sb + so_rB + dcB), t0);
            } else {
                P00 = own[0];
                P0B = ld1(so + so_r0 + dcB);
                PB0 = ld1(so + so_rB);
                PBB = ld1(so + so_rB + dcB);
            }
            double mc[4];
            {
                const double p1a = rowfo ? lerp(P00, PB0, t1) : PB0;
                const double p1b = rowfo ? lerp(P0B, PBB, t1) : PBB;
                mc[0] = dsub(own[0], P00);
                mc[1] = dsub(own[1], colfo ? lerp(P00, P0B, t2) : P0B);
                mc[2] = dsub(own[2], p1a);
                mc[3] = dsub(own[3], colfo ? lerp(p1a, p1b, t2) : p1b);
            }
            if (j >= own_lo && j < own_hi) {
                const int64_t fb = (int64_t)__ldg(lm.m0 + j) * fplane;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (!act[k]) continue;
                    if (!pfo && !nfo[k]) {
                        Cg[(int64_t)hd.z * cgplane + cgc[k]] = own[k];
                    } else if (MODE == 0) {
                        coef[fb + fcol[k]] = mc[k];
                    } else {
                        quant_node(mc[k], q, rbin, fb + fcol[k], fl, sh_hist, sh_ok);
                    }
                }
            }
            // axis-0 marches (march_push): y(j - 1) once x(j) is known, y(j) at the last plane
            if (j >= y_from) emit_y(piring + slot_of(i - 1), j - 1, M.m1, M.m2, mc, true);
            if (j == n0 - 1 && (j > j_start || j == 0)) emit_y(pj, j, mc, M.m1, mc, false);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                M.m2[k] = M.m1[k];
                M.m1[k] = mc[k];
            }
            if (TMA && i >= 1) {   // plane i - 1 is no longer read by this warp
                __syncwarp();
                if (lane == 0) mbar_arrive(empty_s + slot_of(i - 1) * 8);
            }
        }
        if (!TMA) cp_async_wait<0>();
    }
    if (MODE == 2) {
        if (fl) atomicOr(q.flags, fl);
        __syncthreads();
        if (sh_ok)
            for (uint32_t k = tid; k < q.dict; k += kQX * kQY) {
                const uint32_t c = sh_hist[k];
                if (c) atomicAdd(&q.hist[k], (unsigned long long)c);
            }
    }
    (void)warp;
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

template <int MODE, typename TIn, bool TMA>
void launch_one(dim3 grid, const CUtensorMap &tm, const TIn *F, int n0, int n1, int n2, const DevAxis &a0,
                const DevAxis &a1, const DevAxis &a2, const LevelMap &lm, double *coef, double *Z0, double *Cg,
                const QuantOut &q, int c_base, int c_count, int z0_vec, cudaStream_t s) {
    constexpr int smem = QuadGeom<TIn>::smem;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(k_pass1_quad<MODE, TIn, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    k_pass1_quad<MODE, TIn, TMA><<<grid, kQX * kQY, smem, s>>>(tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q,
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

template <int MODE, typename TIn>
void launch_pass1_quad(const TIn *F, int n0, int n1, int n2, const DevAxis &a0, const DevAxis &a1, const DevAxis &a2,
                       const LevelMap &lm, double *coef, double *Z0, double *Cg, const QuantOut &q, int c_base,
                       int c_count, cudaStream_t s) {
    if (c_count <= 0) return;
    const unsigned gx = (n2 + kTileX - 1) / kTileX, gy = (n1 + kTileY - 1) / kTileY;
    static const int slab_env = getenv("HPDR_QUAD_SLABS") ? atoi(getenv("HPDR_QUAD_SLABS")) : 0;
    const int64_t want = 148LL * 4 * 8;   // >= 8 waves of 4 resident blocks per SM
    int slabs = slab_env > 0 ? slab_env : (int)((want + (int64_t)gx * gy - 1) / ((int64_t)gx * gy));
    slabs = std::max(1, std::min(slabs, std::max(1, c_count / 8)));
    const dim3 grid(gx, gy, (unsigned)slabs);
    const int z0_vec = ((int64_t)n1 * n2 % 2 == 0 && n2 % 2 == 0) ? 1 : 0;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    static const bool no_tma = getenv("HPDR_NO_TMA") != nullptr;
    const bool tma = !no_tma && ((int64_t)n2 * sizeof(TIn)) % 16 == 0 && ((uintptr_t)F & 15) == 0 &&
                     make_tmap(tm, F, n0, n1, n2);
    if (tma)
        launch_one<MODE, TIn, true>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec,
                                    s);
    else
        launch_one<MODE, TIn, false>(grid, tm, F, n0, n1, n2, a0, a1, a2, lm, coef, Z0, Cg, q, c_base, c_count, z0_vec,
                                     s);
    LAUNCH_CHECK();
}

template void launch_pass1_quad<0, float>(const float *, int, int, int, const DevAxis &, const DevAxis &,
                                          const DevAxis &, const LevelMap &, double *, double *, double *,
                                          const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<0, double>(const double *, int, int, int, const DevAxis &, const DevAxis &,
                                           const DevAxis &, const LevelMap &, double *, double *, double *,
                                           const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<2, float>(const float *, int, int, int, const DevAxis &, const DevAxis &,
                                          const DevAxis &, const LevelMap &, double *, double *, double *,
                                          const QuantOut &, int, int, cudaStream_t);
template void launch_pass1_quad<2, double>(const double *, int, int, int, const DevAxis &, const DevAxis &,
                                           const DevAxis &, const LevelMap &, double *, double *, double *,
                                           const QuantOut &, int, int, cudaStream_t);

}  // namespace hpdr
