// tiny.cu -- the small end of a hierarchy in one CTA.
//
// Once a level has at most kTinyMaxNodes nodes, every remaining transition of a decomposition
// (GPK residual + quantize-on-write, LPK correction, IPK Thomas, coarse + corr; transform.py:
// 287-323) or of a recomposition (correction, coarse - corr, GPK + mc; transform.py:326-348) is
// latency-bound: a handful of launches per level, each moving a few KB.  Here one 512-thread block
// runs them all with the levels resident in shared memory, phase by phase with block barriers,
// in exactly the generic per-axis path's operation order (transform.cu k_prolong,
// k_mass_restrict, Thomas), so results are bit-identical to the multi-launch chain.
#include "fused.cuh"
#include "level_dev.cuh"
#include "transform.cuh"

namespace hpdr {

namespace {

using namespace lvl;

constexpr int kTinySteps = 10;
constexpr int kTinyMaxNodes = 1024;   // fine nodes of the first transition run here (9^3, 32^2)
constexpr int kTinyHist = 4096;       // shared key histogram (dict sizes up to this)
constexpr int kTinyThreads = 512;

struct TinyStep {
    Shape4 fsh, csh;
    DevAxis ax[4];
    const int32_t *map[4];   // fine-level index -> finest index, per axis
};

struct TinyArgs {
    int nsteps;              // transitions st_a .. st_a + nsteps - 1
    TinyStep st[kTinySteps];
    Shape4 dims;             // finest shape
    const int32_t *cmap[4];  // coarsest level -> finest index (recompose)
    Shape4 shL;              // coarsest level shape
};

// q = e / n, r = e % n for 0 <= e < 2^23 through a float reciprocal and a one-step fix-up (the
// integer divisions of a naive index decode dominated these latency-bound phases)
__device__ __forceinline__ int fdiv(int e, int n, float inv, int &r) {
    int q = __float2int_rz((float)e * inv);
    r = e - q * n;
    if (r < 0) {
        q--;
        r += n;
    } else if (r >= n) {
        q++;
        r -= n;
    }
    return q;
}

__device__ __forceinline__ void coords4(int e, const Shape4 &s, int c[4]) {
    const int n1 = (int)s.n[1], n2 = (int)s.n[2], n3 = (int)s.n[3];
    int t = fdiv(e, n3, 1.0f / (float)n3, c[3]);
    t = fdiv(t, n2, 1.0f / (float)n2, c[2]);
    c[0] = fdiv(t, n1, 1.0f / (float)n1, c[1]);
}

__device__ __forceinline__ int lin4(const Shape4 &s, const int c[4]) {
    return ((c[0] * (int)s.n[1] + c[1]) * (int)s.n[2] + c[2]) * (int)s.n[3] + c[3];
}

__device__ __forceinline__ int64_t finest(const Shape4 &dims, const int32_t *const map[4], const int c[4]) {
    return (((int64_t)__ldg(map[0] + c[0]) * dims.n[1] + __ldg(map[1] + c[1])) * dims.n[2] + __ldg(map[2] + c[2])) *
               dims.n[3] +
           __ldg(map[3] + c[3]);
}

// dst(csh) = src(fsh)[sel] with sel = r0 along active axes (k_gather_coarse)
__device__ void t_gather_coarse(const double *src, const TinyStep &st, double *dst) {
    const int N = (int)st.csh.size();
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        int c[4];
        coords4(e, st.csh, c);
        for (int d = 0; d < 4; d++)
            if (st.ax[d].active) c[d] = __ldg(st.ax[d].r0 + c[d]);
        dst[e] = src[lin4(st.fsh, c)];
    }
}

// one GPK axis (k_prolong): src shape sh (axis a at nc) -> dst (axis a at n); MODE 1 dst = aux - pred,
// MODE 2 dst = pred + aux, MODE 0 dst = pred
template <int MODE>
__device__ void t_prolong(const double *src, double *dst, const double *aux, const Shape4 &sh, int a,
                          const DevAxis &ax) {
    Shape4 dsh = sh;
    dsh.n[a] = ax.n;
    const int N = (int)dsh.size();
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        int c[4];
        coords4(e, dsh, c);
        const int j = c[a];
        const int pa = __ldg(ax.pa + j), pb = __ldg(ax.pb + j);
        c[a] = pa;
        const double va = src[lin4(sh, c)];
        double v = va;
        if (pb >= 0) {
            c[a] = pb;
            const double vb = src[lin4(sh, c)];
            v = dadd(va, dmul(__ldg(ax.pt + j), dsub(vb, va)));
        }
        if (MODE == 1) v = dsub(aux[e], v);
        if (MODE == 2) v = dadd(v, aux[e]);
        dst[e] = v;
    }
}

// interpolate (transform.py:261-268): the active axes in order, the last one fused with the
// residual (MODE 1) or the add (MODE 2).  cur (csh) -> out (fsh); A, B scratch.
template <int MODE>
__device__ void t_interpolate(const TinyStep &st, const double *coarse, double *out, const double *aux, double *A,
                              double *B) {
    int na = 0;
    for (int a = 0; a < 4; a++) na += st.ax[a].active;
    const double *cur = coarse;
    Shape4 sh = st.csh;
    int k = 0;
    for (int a = 0; a < 4; a++) {
        if (!st.ax[a].active) continue;
        const bool last = k == na - 1;
        double *dst = last ? out : ((k % 2 == 0) ? A : B);
        if (last) t_prolong<MODE>(cur, dst, aux, sh, a, st.ax[a]);
        else t_prolong<0>(cur, dst, nullptr, sh, a, st.ax[a]);
        __syncthreads();
        sh.n[a] = st.fsh.n[a];
        cur = dst;
        k++;
    }
}

__device__ __forceinline__ double t_mass(const double *x, int s, int j, int n, const DevAxis &ax) {
    double v = dmul(__ldg(ax.md + j), x[j * s]);
    if (j >= 1) v = dadd(v, dmul(__ldg(ax.ml + j), x[(j - 1) * s]));
    if (j + 1 < n) v = dadd(v, dmul(__ldg(ax.mu + j), x[(j + 1) * s]));
    return v;
}

// one LPK axis (k_mass_restrict): src shape sh (axis a at n) -> dst (axis a at nc)
__device__ void t_mass_restrict(const double *src, double *dst, const Shape4 &sh, int a, const DevAxis &ax) {
    Shape4 dsh = sh;
    dsh.n[a] = ax.nc;
    int stride = 1;
    for (int d = a + 1; d < 4; d++) stride *= (int)sh.n[d];
    const int N = (int)dsh.size(), n = ax.n;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        int c[4];
        coords4(e, dsh, c);
        const int cc = c[a];
        c[a] = 0;
        const double *x = src + lin4(sh, c);
        double v = t_mass(x, stride, __ldg(ax.r0 + cc), n, ax);
        const int r = __ldg(ax.rr + cc);
        if (r >= 0) v = dadd(v, dmul(__ldg(ax.wr + cc), t_mass(x, stride, r, n, ax)));
        const int l = __ldg(ax.rl + cc);
        if (l >= 0) v = dadd(v, dmul(__ldg(ax.wl + cc), t_mass(x, stride, l, n, ax)));
        dst[e] = v;
    }
}

// IPK along axis a of the coarse grid sh (transform.py:229-245), one thread per line
__device__ void t_thomas(double *x0, const Shape4 &sh, int a, const DevAxis &ax) {
    int inner = 1, outer = 1;
    for (int d = 0; d < a; d++) outer *= (int)sh.n[d];
    for (int d = a + 1; d < 4; d++) inner *= (int)sh.n[d];
    const int n = ax.nc, lines = outer * inner;
    for (int ln = threadIdx.x; ln < lines; ln += blockDim.x) {
        int q;
        const int p = fdiv(ln, inner, 1.0f / (float)inner, q);
        double *x = x0 + p * n * inner + q;
        double prev = x[0];
        for (int i = 1; i < n; i++) {
            prev = dsub(x[i * inner], dmul(__ldg(ax.tw + i), prev));
            x[i * inner] = prev;
        }
        auto div = [](double v, double b, double r) {
            bool bad = false;
            const double q = div_fast(v, b, r, bad);
            return bad ? ddiv(v, b) : q;
        };
        double last = div(prev, __ldg(ax.tb + n - 1), __ldg(ax.tr + n - 1));
        x[(n - 1) * inner] = last;
        for (int i = n - 2; i >= 0; i--) {
            last = div(dsub(x[i * inner], dmul(__ldg(ax.tu + i), last)), __ldg(ax.tb + i), __ldg(ax.tr + i));
            x[i * inner] = last;
        }
    }
}

// correction (transform.py:251-260): mass + restrict per active axis, then Thomas per active
// axis.  mc (fsh) -> returned buffer (csh), one of A / B.
__device__ double *t_correction(const TinyStep &st, const double *mc, double *A, double *B) {
    const double *cur = mc;
    double *out = A;
    Shape4 sh = st.fsh;
    int k = 0;
    for (int a = 0; a < 4; a++) {
        if (!st.ax[a].active) continue;
        out = (k++ % 2 == 0) ? A : B;
        t_mass_restrict(cur, out, sh, a, st.ax[a]);
        __syncthreads();
        sh.n[a] = st.csh.n[a];
        cur = out;
    }
    for (int a = 0; a < 4; a++) {
        if (!st.ax[a].active) continue;
        t_thomas(out, sh, a, st.ax[a]);
        __syncthreads();
    }
    return out;
}

// A step's record (shapes, axis tables, maps) into shared memory: the per-element reads of a
// dynamically indexed kernel parameter otherwise go to the constant bank with a computed address.
__device__ __forceinline__ void load_step(TinyStep &dst, const TinyStep &src) {
    __syncthreads();   // the previous step's readers are done
    static_assert(sizeof(TinyStep) % 8 == 0, "");
    for (int i = threadIdx.x; i < (int)(sizeof(TinyStep) / 8); i += blockDim.x)
        reinterpret_cast<long long *>(&dst)[i] = reinterpret_cast<const long long *>(&src)[i];
    __syncthreads();
}

// Every operator table of every step into L1 up front (a few KB, all lines in flight at once), so
// the per-phase table reads hit L1 instead of paying a cold global-memory latency each.
__device__ void t_prefetch_tables(const TinyArgs &T) {
    auto pf = [](const void *p, int bytes) {
        if (!p) return;
        for (int o = threadIdx.x * 128; o < bytes; o += blockDim.x * 128)
            asm volatile("prefetch.global.L1 [%0];" ::"l"((const char *)p + o));
    };
    for (int k = 0; k < T.nsteps; k++)
        for (int d = 0; d < 4; d++) {
            const DevAxis &a = T.st[k].ax[d];
            if (a.active) {
                const int n = a.n * 8, nc = a.nc * 8;
                pf(a.pa, n / 2), pf(a.pb, n / 2), pf(a.pt, n), pf(a.md, n), pf(a.ml, n), pf(a.mu, n);
                pf(a.r0, nc / 2), pf(a.rr, nc / 2), pf(a.rl, nc / 2), pf(a.wr, nc), pf(a.wl, nc);
                pf(a.tw, nc), pf(a.tb, nc), pf(a.tu, nc), pf(a.tr, nc);
            }
            pf(T.st[k].map[d], (int)T.st[k].fsh.n[d] * 4);
        }
}

__device__ __forceinline__ bool t_is_coarse(const TinyStep &st, const int c[4]) {
    for (int d = 0; d < 4; d++)
        if (st.ax[d].active && __ldg(st.ax[d].pb + c[d]) >= 0) return false;
    return true;
}

// Decomposition with quantize-on-write of transitions st_a .. (the caller's last), starting from
// the dense level F0 (fp64, device); the coarsest level is written to DL and quantized raw.
__global__ void __launch_bounds__(kTinyThreads) k_tiny_decompose(TinyArgs T, const double *__restrict__ F0,
                                                                 double *__restrict__ DL, QuantOut q,
                                                                 const long long *__restrict__ cidx, int n_co) {
    extern __shared__ double tsm[];
    const int nmax = (int)T.st[0].fsh.size();
    double *F = tsm, *M = F + nmax, *A = M + nmax, *B = A + nmax, *Cg = B + nmax;
    // keys concentrate on a few values: count them in shared memory, flush once (one global
    // atomic per used bin instead of one per node on the same few addresses)
    uint32_t *sh_hist = reinterpret_cast<uint32_t *>(Cg + nmax / 2 + 1);
    const bool sh_ok = q.dict <= (uint32_t)kTinyHist;
    if (sh_ok)
        for (uint32_t k = threadIdx.x; k < q.dict; k += blockDim.x) sh_hist[k] = 0;
    t_prefetch_tables(T);
    for (int i = threadIdx.x; i < nmax; i += blockDim.x) F[i] = F0[i];
    __syncthreads();
    const double rbin = 1.0 / qbin(q);
    int fl = 0;
    __shared__ __align__(16) TinyStep sst;   // the current step's tables, off the parameter bank
    for (int s = 0; s < T.nsteps; s++) {
        load_step(sst, T.st[s]);
        const TinyStep &st = sst;
        t_gather_coarse(F, st, Cg);
        __syncthreads();
        t_interpolate<1>(st, Cg, M, F, A, B);   // M = F - pred
        // fine-only nodes: quantize-on-write at their finest positions (quantize.py:73-84)
        const int nf = (int)st.fsh.size();
        for (int e = threadIdx.x; e < nf; e += blockDim.x) {
            int c[4];
            coords4(e, st.fsh, c);
            if (!t_is_coarse(st, c)) quant_node(M[e], q, rbin, finest(T.dims, st.map, c), fl, sh_hist, sh_ok);
        }
        const double *corr = t_correction(st, M, A, B);
        const int nc = (int)st.csh.size();
        for (int e = threadIdx.x; e < nc; e += blockDim.x) F[e] = dadd(Cg[e], corr[e]);   // coarse + corr
        __syncthreads();
    }
    // the coarsest level: to DL (the blob's raw coarse values), its nodes keyed 0 after the
    // bin-limit / finiteness check (quantize.py:64-77; k_quantize_coarsest)
    const int nL = (int)T.st[T.nsteps - 1].csh.size();
    for (int i = threadIdx.x; i < nL; i += blockDim.x) DL[i] = F[i];
    const double bin = qbin(q);
    for (int k = threadIdx.x; k < n_co; k += blockDim.x) {
        const double v = F[k];
        if (!isfinite(v)) fl |= 1;
        else if (fabs(v / bin) >= 4611686018427387904.0) fl |= 2;
        q.keys[cidx[k]] = 0;
    }
    if (threadIdx.x == 0 && n_co) atomicAdd(&q.hist[0], (unsigned long long)n_co);
    if (fl) atomicOr(q.flags, fl);
    if (sh_ok) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < q.dict; k += blockDim.x)
            if (sh_hist[k]) atomicAdd(&q.hist[k], (unsigned long long)sh_hist[k]);
    }
}

// Recomposition of transitions (the caller's last) .. st_a from the coefficient set: the coarsest
// level gathered from coef, then per transition (coarser first) corr, coarse - corr and
// pred + mc; the finest level of the range (T.st[0].fsh) is written to D (fp64).
__global__ void __launch_bounds__(kTinyThreads) k_tiny_recompose(TinyArgs T, const double *__restrict__ coef,
                                                                 double *__restrict__ D) {
    extern __shared__ double tsm[];
    const int nmax = (int)T.st[0].fsh.size();
    double *F = tsm, *M = F + nmax, *A = M + nmax, *B = A + nmax, *Cg = B + nmax;
    t_prefetch_tables(T);
    {
        const int nL = (int)T.shL.size();
        for (int e = threadIdx.x; e < nL; e += blockDim.x) {
            int c[4];
            coords4(e, T.shL, c);
            F[e] = coef[finest(T.dims, T.cmap, c)];
        }
    }
    __syncthreads();
    __shared__ __align__(16) TinyStep sst;
    for (int s = T.nsteps - 1; s >= 0; s--) {
        load_step(sst, T.st[s]);
        const TinyStep &st = sst;
        // mc of this level, zero at the next-coarser level's nodes (k_gather_level)
        const int nf = (int)st.fsh.size();
        for (int e = threadIdx.x; e < nf; e += blockDim.x) {
            int c[4];
            coords4(e, st.fsh, c);
            M[e] = t_is_coarse(st, c) ? 0.0 : coef[finest(T.dims, st.map, c)];
        }
        __syncthreads();
        const double *corr = t_correction(st, M, A, B);
        const int nc = (int)st.csh.size();
        for (int e = threadIdx.x; e < nc; e += blockDim.x) Cg[e] = dsub(F[e], corr[e]);   // coarse - corr
        __syncthreads();
        t_interpolate<2>(st, Cg, F, M, A, B);   // F = pred + mc
    }
    for (int i = threadIdx.x; i < nmax; i += blockDim.x) D[i] = F[i];
}

}  // namespace

// Host side --------------------------------------------------------------------------------------

// First transition index >= st_min whose fine level fits one block (-1: none, or too many left).
int tiny_start(const DevPlan &p, int st_min) {
    static const bool off = getenv("HPDR_NO_TINY") != nullptr;
    const int L = p.host.L;
    if (off || L < 2) return -1;
    for (int st = std::max(st_min, 0); st + 1 < L; st++)
        if (p.steps[st].fsh.size() <= kTinyMaxNodes) return (L - 1 - st) <= kTinySteps ? st : -1;
    return -1;
}

namespace {
TinyArgs tiny_args(const DevPlan &p, int st_a) {
    TinyArgs T{};
    const int L = p.host.L;
    T.nsteps = L - 1 - st_a;
    for (int k = 0; k < T.nsteps; k++) {
        const DevStep &s = p.steps[st_a + k];
        T.st[k].fsh = s.fsh;
        T.st[k].csh = s.csh;
        for (int d = 0; d < 4; d++) {
            T.st[k].ax[d] = s.ax[d];
            T.st[k].map[d] = p.map[d][st_a + k];
        }
    }
    T.dims = p.dims;
    for (int d = 0; d < 4; d++) {
        T.cmap[d] = p.map[d][L - 1];
        T.shL.n[d] = p.host.cnt[d][L - 1];
    }
    return T;
}

size_t tiny_smem(const DevPlan &p, int st_a) {   // F, M, A, B (fine), Cg (<= fine / 2 + 1), histogram
    const int64_t nf = p.steps[st_a].fsh.size();
    return (size_t)(4 * nf + nf / 2 + 1) * 8 + kTinyHist * 4;
}

void tiny_attr() {
    static bool done = false;
    if (done) return;
    const int mx = (4 * kTinyMaxNodes + kTinyMaxNodes / 2 + 1) * 8 + kTinyHist * 4;   // 200 KB
    CUDA_CHECK(cudaFuncSetAttribute(k_tiny_decompose, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CUDA_CHECK(cudaFuncSetAttribute(k_tiny_recompose, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    done = true;
}
}  // namespace

void tiny_decompose_quantize(const DevPlan &p, int st_a, const double *F0, double *DL, const QuantOut &q,
                             cudaStream_t s) {
    tiny_attr();
    const TinyArgs T = tiny_args(p, st_a);
    KPROF("k_tiny_decompose", 8.0 * (p.steps[st_a].fsh.size() + p.steps[p.host.L - 2].csh.size()), s);
    k_tiny_decompose<<<1, kTinyThreads, tiny_smem(p, st_a), s>>>(T, F0, DL, q, p.coarsest,
                                                                 (int)p.host.coarsest.size());
    LAUNCH_CHECK();
}

void tiny_recompose(const DevPlan &p, int st_a, const double *coef, double *D, cudaStream_t s) {
    tiny_attr();
    const TinyArgs T = tiny_args(p, st_a);
    KPROF("k_tiny_recompose", 16.0 * p.steps[st_a].fsh.size(), s);
    k_tiny_recompose<<<1, kTinyThreads, tiny_smem(p, st_a), s>>>(T, coef, D);
    LAUNCH_CHECK();
}

}  // namespace hpdr
