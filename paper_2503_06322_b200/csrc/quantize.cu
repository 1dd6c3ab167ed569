// quantize.cu -- level-wise linear quantization fused with the key histogram, and the
// order-preserving outlier compaction (quantize.py:50-98, huffman.py:74-104).
#include <cub/cub.cuh>

#include "stages.cuh"

namespace hpdr {

namespace {

constexpr int kQThreads = 256;
constexpr int kSmemHistMax = 16384;          // u32 shared counters (64 KB)
constexpr int kChunkWords = 1024;            // outlier-mask words per compaction block (large masks)

// Compaction block size: 1024 mask words, down to 256 (one scan step) for small masks so that the
// latency-bound compaction still spreads over every SM.
int chunk_words(int64_t words) {
    int cw = kChunkWords;
    while (cw > 256 && words / cw < 2 * kNumSMs) cw /= 2;
    return cw;
}
constexpr double kBinLimit = 4611686018427387904.0;   // 2^62, quantize.py:21

struct Coarsest {
    long long idx[16];
    int n;
};

// Warp-aggregated increment: lanes with equal keys add once (key 0 dominates real data).
__device__ __forceinline__ void hist_add(uint32_t *sh, unsigned long long *g, bool use_sh, uint32_t key, unsigned mask) {
    unsigned peers = __match_any_sync(mask, key);
    int lane = threadIdx.x & 31;
    if (lane == __ffs(peers) - 1) {
        if (use_sh) atomicAdd(&sh[key], (uint32_t)__popc(peers));
        else atomicAdd(&g[key], (unsigned long long)__popc(peers));
    }
}

__global__ void __launch_bounds__(kQThreads) k_quantize(const double *__restrict__ coef, int64_t n, Coarsest co,
                                                        double bin, long long half, uint32_t dict,
                                                        uint16_t *__restrict__ keys, uint32_t *__restrict__ omask,
                                                        unsigned long long *__restrict__ hist, int *__restrict__ flags) {
    extern __shared__ uint32_t sh_hist[];
    const bool use_sh = dict <= kSmemHistMax;
    if (use_sh)
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) sh_hist[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const double rbin = 1.0 / bin;
    const double half_d = (double)half;
    int fl = 0;
    // U warp-rows of 32 coefficients in flight per lane before any is quantized
    constexpr int U = 4;
    const int64_t step = warps_total * 32;
    for (int64_t w0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < n; w0 += U * step) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = w0 + u * step + lane;
            v[u] = i < n ? __ldg(coef + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t wbase = w0 + u * step;
            if (wbase >= n) break;
            const int64_t i = wbase + lane;
            const bool valid = i < n;
            // b = rint(c / bin) as an integral double (quantize.py:73-76; exact, see fused.cu quant_node)
            double r = 0.0;
            if (valid) {
                if (!isfinite(v[u])) {
                    fl |= 1;
                } else {
                    const double qa = __dmul_rn(v[u], rbin);
                    r = rint(qa);
                    const double dist = 0.5 - fabs(__dsub_rn(qa, r));
                    if (!(dist > fabs(qa) * 0x1p-49 && fabs(qa) < 0x1p61)) {
                        const double sc = v[u] / bin;   // IEEE division
                        if (fabs(sc) >= kBinLimit) {
                            fl |= 2;
                            r = 0.0;
                        } else {
                            r = rint(sc);
                        }
                    }
                }
            }
            // coarsest nodes are carried raw (:77): warp-uniform test first
            bool any = false;
#pragma unroll
            for (int k = 0; k < 16; k++) any |= k < co.n && (co.idx[k] >> 5) == (wbase >> 5);
            if (any) {
#pragma unroll
                for (int k = 0; k < 16; k++)
                    if (k < co.n && i == co.idx[k]) r = 0.0;
            }
            const bool out = valid && fabs(r) >= half_d;
            const unsigned om = __ballot_sync(0xffffffffu, out);
            if (lane == 0) omask[wbase >> 5] = om;
            const uint32_t key = out ? 0u : (uint32_t)(r >= 0.0 ? 2.0 * r : -2.0 * r - 1.0);   // zigzag
            if (valid) {
                keys[i] = (uint16_t)key;
                if (use_sh) atomicAdd(&sh_hist[key], 1u);
                else atomicAdd(&hist[key], 1ULL);
            }
        }
    }
    if (fl) atomicOr(flags, fl);
    if (use_sh) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) {
            uint32_t c = sh_hist[k];
            if (c) atomicAdd(&hist[k], (unsigned long long)c);
        }
    }
}

__global__ void k_chunk_counts(const uint32_t *__restrict__ omask, int64_t words, int cw, unsigned long long *__restrict__ counts) {
    typedef cub::BlockReduce<unsigned, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    const int64_t c = blockIdx.x;
    unsigned s = 0;
    for (int64_t w = c * cw + threadIdx.x; w < min64(words, (c + 1) * cw); w += blockDim.x)
        s += __popc(omask[w]);
    unsigned tot = BR(tmp).Sum(s);
    if (threadIdx.x == 0) counts[c] = tot;
}

// Ordered outlier compaction (quantize.py:80-83: ascending flat index).  Per 256-word step the block
// scans the words' popcounts; then each warp takes whole words with one lane per node, so the
// index / bin writes and the sparse-bin reads are coalesced (consecutive positions / nodes).
__global__ void k_write_outliers(const uint32_t *__restrict__ omask, int64_t words, int cw, const double *__restrict__ coef,
                                 const long long *__restrict__ sparse, double bin, const unsigned long long *__restrict__ chunk_off,
                                 uint64_t *__restrict__ oidx, int64_t *__restrict__ obins) {
    typedef cub::BlockScan<unsigned, 256> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint32_t smask[256];
    __shared__ unsigned spre[256];
    const int64_t c = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long base = chunk_off[c];
    const int64_t w_end = min64(words, (c + 1) * cw);
    for (int64_t w0 = c * cw; w0 < w_end; w0 += blockDim.x) {
        const int64_t w = w0 + threadIdx.x;
        const uint32_t m = w < w_end ? omask[w] : 0u;
        if (!__syncthreads_or(m != 0u)) continue;   // no outlier in these 256 words (the common case)
        unsigned pre, tot;
        BS(tmp).ExclusiveSum((unsigned)__popc(m), pre, tot);
        smask[threadIdx.x] = m;
        spre[threadIdx.x] = pre;
        __syncthreads();
        for (int k = warp; k < 256; k += 8) {
            const uint32_t mk = smask[k];
            if (!mk) continue;
            if ((mk >> lane) & 1u) {
                const unsigned long long pos = base + spre[k] + __popc(mk & ((1u << lane) - 1u));
                const int64_t i = (w0 + k) * 32 + lane;
                oidx[pos] = (uint64_t)i;
                obins[pos] = sparse ? sparse[i] : (long long)rint(coef[i] / bin);
            }
        }
        base += tot;
        __syncthreads();
    }
}

__global__ void k_histogram(const uint32_t *__restrict__ keys, int64_t n, uint32_t dict,
                            unsigned long long *__restrict__ hist, int *__restrict__ bad) {
    extern __shared__ uint32_t sh_hist[];
    const bool use_sh = dict <= kSmemHistMax;
    if (use_sh)
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) sh_hist[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t wbase = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; wbase < n;
         wbase += warps_total * 32) {
        const int64_t i = wbase + lane;
        uint32_t key = i < n ? keys[i] : 0u;
        bool ok = i < n && key < dict;
        if (i < n && key >= dict) atomicOr(bad, 1);
        unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) hist_add(sh_hist, hist, use_sh, key, m);
    }
    if (use_sh) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) {
            uint32_t c = sh_hist[k];
            if (c) atomicAdd(&hist[k], (unsigned long long)c);
        }
    }
}

}  // namespace

void quantize_device(hpdr_ctx *ctx, const double *coef, int64_t n, const std::vector<int64_t> &coarsest,
                     double bin_width, uint32_t dict_size, uint16_t *keys, QuantResult &res, cudaStream_t s) {
    const int64_t words = (n + 31) / 32;
    uint32_t *omask = (uint32_t *)ctx->dbuf("omask", words * 4);
    unsigned long long *hist = (unsigned long long *)ctx->dbuf("hist", (size_t)dict_size * 8);
    int *flags = (int *)ctx->dbuf("qflags", 16);
    zero_async(hist, (size_t)dict_size * 8, s);
    zero_async(flags, 16, s);
    Coarsest co;
    co.n = (int)coarsest.size();
    for (int k = 0; k < 16; k++) co.idx[k] = k < co.n ? coarsest[k] : -1;
    const long long half = dict_size / 2;
    size_t smem = dict_size <= kSmemHistMax ? (size_t)dict_size * 4 : 0;
    if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_quantize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned grid = grid_for(n, kQThreads, 148 * 4);
    {
        KPROF("k_quantize", 10.0 * n + n / 8.0, s);
        k_quantize<<<grid, kQThreads, smem, s>>>(coef, n, co, bin_width, half, dict_size, keys, omask, hist, flags);
        LAUNCH_CHECK();
    }
    quantize_finish(ctx, n, dict_size, bin_width, coef, nullptr, res, s);
}

void quantize_finish(hpdr_ctx *ctx, int64_t n, uint32_t dict_size, double bin_width, const double *coef,
                     const long long *obins_sparse, QuantResult &res, cudaStream_t s) {
    const int64_t words = (n + 31) / 32;
    const int cw = chunk_words(words);
    const int64_t chunks = (words + cw - 1) / cw;
    uint32_t *omask = (uint32_t *)ctx->dbuf("omask", words * 4);
    unsigned long long *hist = (unsigned long long *)ctx->dbuf("hist", (size_t)dict_size * 8);
    int *flags = (int *)ctx->dbuf("qflags", 16);
    unsigned long long *ccount = (unsigned long long *)ctx->dbuf("ochunk", (chunks + 1) * 8);
    unsigned long long *coff = (unsigned long long *)ctx->dbuf("ochunk_off", (chunks + 1) * 8);
    {
        KPROF("k_chunk_counts", 4.0 * words, s);
        k_chunk_counts<<<(unsigned)chunks, 256, 0, s>>>(omask, words, cw, ccount);
        LAUNCH_CHECK();
    }
    size_t tmp_bytes = 0;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, ccount, coff, (int)(chunks + 1), s));
    void *tmp = ctx->dbuf("cub_tmp", tmp_bytes);
    zero_async(ccount + chunks, 8, s);
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ccount, coff, (int)(chunks + 1), s));
    count_launch();
    uint64_t *h = (uint64_t *)ctx->hbuf("q_readback", (size_t)dict_size * 8 + 64);
    small_copy(h, coff + chunks, 8, s);
    small_copy(h + 1, flags, 4, s);
    small_copy(h + 2, hist, (size_t)dict_size * 8, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    res.n_outliers = h[0];
    int fl;
    memcpy(&fl, h + 1, 4);
    res.flags = fl;
    res.hist.assign(h + 2, h + 2 + dict_size);
    if (fl) return;
    res.d_outlier_idx = (uint64_t *)ctx->dbuf(ctx->oname("oidx"), res.n_outliers * 8);
    res.d_outlier_bins = (int64_t *)ctx->dbuf(ctx->oname("obins"), res.n_outliers * 8);
    if (res.n_outliers) {
        KPROF("k_write_outliers", 4.0 * words + 24.0 * res.n_outliers, s);
        k_write_outliers<<<(unsigned)chunks, 256, 0, s>>>(omask, words, cw, coef, obins_sparse, bin_width, coff,
                                                          res.d_outlier_idx, res.d_outlier_bins);
        LAUNCH_CHECK();
    }
}

void histogram_device(hpdr_ctx *ctx, const uint32_t *keys, int64_t n, uint32_t dict_size, std::vector<uint64_t> &hist,
                      bool *bad, cudaStream_t s) {
    unsigned long long *d = (unsigned long long *)ctx->dbuf("hist", (size_t)dict_size * 8);
    int *flags = (int *)ctx->dbuf("qflags", 16);
    zero_async(d, (size_t)dict_size * 8, s);
    zero_async(flags, 16, s);
    size_t smem = dict_size <= kSmemHistMax ? (size_t)dict_size * 4 : 0;
    if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_histogram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (n > 0) {
        KPROF("k_histogram", 4.0 * n, s);
        k_histogram<<<grid_for(n, 256, 148 * 4), 256, smem, s>>>(keys, n, dict_size, d, flags);
        LAUNCH_CHECK();
    }
    uint64_t *h = (uint64_t *)ctx->hbuf("q_readback", (size_t)dict_size * 8 + 64);
    small_copy(h, flags, 4, s);
    small_copy(h + 1, d, (size_t)dict_size * 8, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    int fl;
    memcpy(&fl, h, 4);
    *bad = fl != 0;
    hist.assign(h + 1, h + 1 + dict_size);
}

}  // namespace hpdr
