// huffman.cu -- canonical Huffman: host codebook (huffman.py:107-204) and device
// encode (huffman.py:228-289) / decode (huffman.py:207-358) kernels.
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <cub/cub.cuh>
#include <numeric>

#include "stages.cuh"

namespace hpdr {

// ===================================================================== host codebook
namespace {

// Moffat-Katajainen in-place code lengths over weights sorted ascending by (count, key)
// (huffman.py:107-157).  a[] is overwritten with leaf lengths, slot i = leaf i.
void mk_lengths(std::vector<int64_t> &a) {
    const int64_t n = (int64_t)a.size();
    if (n == 1) { a[0] = 1; return; }
    int64_t leaf = 0, node = 0;
    for (int64_t t = 0; t < n - 1; t++) {
        for (int child = 0; child < 2; child++) {
            // a leaf wins ties (strict <), huffman.py:122 / :130
            const bool take_node = leaf >= n || (node < t && a[node] < a[leaf]);
            int64_t w;
            if (take_node) { w = a[node]; a[node] = t; node++; }
            else { w = a[leaf]; leaf++; }
            a[t] = child == 0 ? w : a[t] + w;
        }
    }
    a[n - 2] = 0;                                            // root depth
    for (int64_t t = n - 3; t >= 0; t--) a[t] = a[a[t]] + 1;  // parent links -> depths
    int64_t avail = 1, used = 0, depth = 0, t = n - 2, x = n - 1;
    while (avail > 0) {
        while (t >= 0 && a[t] == depth) { used++; t--; }
        while (avail > used) { a[x--] = depth; avail--; }
        avail = 2 * used;
        used = 0;
        depth++;
    }
}

}  // namespace

namespace {
// Canonical codes in (length, key) order (huffman.py:188-204) over the present keys `keys`
// (ascending): a counting sort by length, then the reference's code recurrence.
int canonical_from(const uint8_t *lengths, const uint32_t *keys, size_t n, uint32_t *codes) {
    if (!n) return HPDR_OK;
    uint32_t cnt[4][256];   // interleaved counters: no store-to-load chain on runs of equal lengths
    memset(cnt, 0, sizeof(cnt));
    for (size_t i = 0; i < n; i++) cnt[i & 3][lengths[keys[i]]]++;
    uint32_t start[256], acc = 0;
    for (int L = 0; L < 256; L++) {
        start[L] = acc;
        acc += cnt[0][L] + cnt[1][L] + cnt[2][L] + cnt[3][L];
    }
    static thread_local std::vector<uint32_t> order;
    order.resize(n);
    for (size_t i = 0; i < n; i++) order[start[lengths[keys[i]]]++] = keys[i];
    uint64_t code = 0;
    int prev = lengths[order[0]];
    for (uint32_t k : order) {
        const int sh = lengths[k] - prev;
        if (code) {
            if (sh >= 32) return HPDR_ERR_OVERFLOW;   // Python int >= 2^32 into a uint32 array
            code <<= sh;
        }
        if (code >> 32) return HPDR_ERR_OVERFLOW;
        codes[k] = (uint32_t)code;
        code++;
        prev = lengths[k];
    }
    return HPDR_OK;
}
}  // namespace

int canonical_codes(const uint8_t *lengths, uint32_t dict_size, uint32_t *codes) {
    static thread_local std::vector<uint32_t> keys;
    keys.resize(dict_size);
    size_t n = 0;
    for (uint32_t k = 0; k < dict_size; k++) {
        codes[k] = 0;
        keys[n] = k;
        n += lengths[k] != 0;
    }
    return canonical_from(lengths, keys.data(), n, codes);
}

int build_codebook(const uint64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes, std::string &err) {
    // Present keys in stable ascending (count, key) order (huffman.py:174): collected in key order,
    // then a stable LSD radix sort on the count bits alone (ceil(bits / 11) passes).
    static thread_local std::vector<uint64_t> v, tmp;
    static thread_local std::vector<int64_t> a;
    static thread_local std::vector<uint32_t> pk;   // present keys, ascending
    memset(lengths, 0, dict_size);
    memset(codes, 0, (size_t)dict_size * 4);
    v.resize(dict_size);
    size_t n = 0;
    uint64_t mx = 0;
    for (uint32_t k = 0; k < dict_size; k++) {
        const uint64_t c = counts[k];
        v[n] = (c << 16) | k;
        n += c != 0;
        mx |= c;
    }
    if (n == 0) { err = "frequency table has no nonzero counts"; return HPDR_ERR_VALIDATION; }
    if (n == 1) { lengths[v[0] & 0xffff] = 1; return HPDR_OK; }
    pk.resize(n);
    for (size_t i = 0; i < n; i++) pk[i] = (uint32_t)(v[i] & 0xffff);
    a.resize(n);
    if (mx >> 48) {   // counts beyond 2^48: comparison sort on (count, key)
        std::vector<uint32_t> present;
        for (uint32_t k = 0; k < dict_size; k++)
            if (counts[k]) present.push_back(k);
        std::stable_sort(present.begin(), present.end(), [&](uint32_t x, uint32_t y) { return counts[x] < counts[y]; });
        for (size_t i = 0; i < n; i++) {
            a[i] = (int64_t)counts[present[i]];
            v[i] = present[i];
        }
    } else {
        int cb = 1;
        while (cb < 48 && (mx >> cb)) cb++;
        const int passes = (cb + 10) / 11, digit = (cb + passes - 1) / passes;
        const uint32_t mask = (1u << digit) - 1;
        tmp.resize(n);
        static thread_local std::vector<uint32_t> cbuf;
        cbuf.resize(4 * 2049);
        uint32_t *c = cbuf.data();
        for (int ps = 0, sh = 16; ps < passes; ps++, sh += digit) {
            memset(c, 0, sizeof(uint32_t) * 4 * 2049);
            for (size_t i = 0; i < n; i++) c[(i & 3) * 2049 + ((v[i] >> sh) & mask) + 1]++;
            for (uint32_t d = 0; d <= mask; d++) c[d + 1] += c[d] + c[2049 + d + 1] + c[2 * 2049 + d + 1] + c[3 * 2049 + d + 1];
            for (size_t i = 0; i < n; i++) tmp[c[(v[i] >> sh) & mask]++] = v[i];
            v.swap(tmp);
        }
        for (size_t i = 0; i < n; i++) a[i] = (int64_t)(v[i] >> 16);
    }
    mk_lengths(a);
    int64_t mxl = 0;
    for (size_t i = 0; i < n; i++) {
        lengths[v[i] & 0xffff] = (uint8_t)std::min<int64_t>(a[i], 255);
        mxl = std::max(mxl, a[i]);
    }
    if (mxl > kMaxCodeLen) {
        err = "codeword length " + std::to_string(mxl) + " exceeds " + std::to_string(kMaxCodeLen);
        return HPDR_ERR_VALIDATION;
    }
    return canonical_from(lengths, pk.data(), n, codes);
}

// ===================================================================== encode
namespace {

constexpr int kEncThreads = 256;
constexpr int kSymPerThread = kBlockSymbols / kEncThreads;   // 16
constexpr int kSmemTableMax = 8192;
constexpr int kEncTableMax = 4096;     // codes + lengths + the unit's word buffer fit 48 KB

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Per-unit bit totals.  One block per unit; 16 consecutive symbols per thread.
// Keys are 16 bits (dict_size <= 65535, quantize.py:61): a thread's 16 consecutive keys are two
// 16-byte loads.
__device__ __forceinline__ void load_keys16(const uint16_t *p, uint32_t k[16]) {
    const uint4 *v4 = reinterpret_cast<const uint4 *>(p);
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const uint4 v = v4[h];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            k[8 * h + 2 * i] = w[i] & 0xffffu;
            k[8 * h + 2 * i + 1] = w[i] >> 16;
        }
    }
}

__global__ void __launch_bounds__(kEncThreads) k_unit_bits(const uint16_t *__restrict__ keys, int64_t n,
                                                           const uint8_t *__restrict__ lens, uint32_t dict,
                                                           uint64_t *__restrict__ ubits, int64_t units) {
    __shared__ uint8_t sl[kSmemTableMax];
    const bool sm = dict <= kSmemTableMax;
    if (sm)
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) sl[k] = lens[k];
    __syncthreads();
    typedef cub::BlockReduce<unsigned, kEncThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t lo = u * kBlockSymbols + (int64_t)threadIdx.x * kSymPerThread;
        unsigned s = 0;
        if (lo + kSymPerThread <= n) {
            uint32_t k[kSymPerThread];
            load_keys16(keys + lo, k);
#pragma unroll
            for (int q = 0; q < kSymPerThread; q++) s += sm ? sl[k[q]] : lens[k[q]];
        } else {
            for (int64_t i = lo; i < min64(n, lo + kSymPerThread); i++) s += sm ? sl[keys[i]] : lens[keys[i]];
        }
        unsigned tot = BR(tmp).Sum(s);
        if (threadIdx.x == 0) ubits[u] = tot;
        __syncthreads();
    }
}

// Pack one unit per block: per-thread bit offsets by block scan, codewords OR-ed into a
// shared word buffer aligned to the unit's global word, then streamed out (boundary words
// shared with the neighbouring units use atomicOr on a zeroed buffer).
__global__ void __launch_bounds__(kEncThreads) k_encode(const uint16_t *__restrict__ keys, int64_t n,
                                                        const uint8_t *__restrict__ lens,
                                                        const uint32_t *__restrict__ codes, uint32_t dict,
                                                        const uint64_t *__restrict__ uoff,
                                                        const uint64_t *__restrict__ ubits,
                                                        uint32_t *__restrict__ out, int64_t u_lo, int64_t u_hi) {
    __shared__ uint32_t words[kBlockSymbols + 2];
    __shared__ uint8_t sl[kEncTableMax];
    __shared__ uint32_t sc[kEncTableMax];
    const bool sm = dict <= kEncTableMax;
    if (sm)
        for (uint32_t k = threadIdx.x; k < dict; k += blockDim.x) { sl[k] = lens[k]; sc[k] = codes[k]; }
    typedef cub::BlockScan<unsigned, kEncThreads> BS;
    __shared__ typename BS::TempStorage tmp;
    for (int64_t u = u_lo + blockIdx.x; u < u_hi; u += gridDim.x) {
        for (int w = threadIdx.x; w < kBlockSymbols + 2; w += blockDim.x) words[w] = 0;
        __syncthreads();
        const int64_t lo = u * kBlockSymbols + (int64_t)threadIdx.x * kSymPerThread;
        uint32_t k16[kSymPerThread];
        int cnt = 0;
        if (lo + kSymPerThread <= n) {
            load_keys16(keys + lo, k16);
            cnt = kSymPerThread;
        } else {
            for (int64_t i = lo; i < min64(n, lo + kSymPerThread); i++) k16[cnt++] = keys[i];
        }
        unsigned mybits = 0;
#pragma unroll
        for (int q = 0; q < kSymPerThread; q++)
            if (q < cnt) mybits += sm ? sl[k16[q]] : lens[k16[q]];
        unsigned start;
        BS(tmp).ExclusiveSum(mybits, start);
        const uint64_t g = uoff[u];
        uint32_t pos = (uint32_t)(g & 31) + start;
#pragma unroll
        for (int q = 0; q < kSymPerThread; q++) {
            if (q >= cnt) break;
            const uint32_t key = k16[q];
            const int L = sm ? sl[key] : lens[key];
            const uint32_t c = sm ? sc[key] : codes[key];
            // left-align the L-bit code in a 64-bit window at bit (pos & 31) of word pos >> 5
            const uint64_t v = ((uint64_t)c << (64 - L)) >> (pos & 31);
            const uint32_t hi = (uint32_t)(v >> 32), lo32 = (uint32_t)v;
            atomicOr(&words[pos >> 5], hi);
            if (lo32) atomicOr(&words[(pos >> 5) + 1], lo32);
            pos += L;
        }
        __syncthreads();
        const uint32_t nw = (uint32_t)(((g & 31) + ubits[u] + 31) >> 5);
        uint32_t *dst = out + (g >> 5);
        for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) {
            const uint32_t val = bswap32(words[w]);
            if (w == 0 || w == nw - 1) atomicOr(&dst[w], val);
            else dst[w] = val;
        }
        __syncthreads();
    }
}

// The words k_encode merges with atomicOr -- each unit's first and last word -- are cleared; every
// other word of the stream is written whole by exactly one unit (no full-buffer memset).
__global__ void k_zero_unit_bounds(const uint64_t *__restrict__ uoff, const uint64_t *__restrict__ ubits,
                                   uint32_t *__restrict__ out, int64_t units) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units; u += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t b = ubits[u];
        if (b) {
            const uint64_t g = uoff[u];
            out[g >> 5] = 0;
            out[(g + b - 1) >> 5] = 0;
        }
    }
}

}  // namespace

void encode_device(hpdr_ctx *ctx, const uint16_t *keys, int64_t n, uint32_t dict_size, const uint8_t *lengths,
                   const uint32_t *codes, EncodeResult &res, cudaStream_t s, const EncodeHooks *hooks,
                   const uint64_t *hist) {
    const int64_t units = (n + kBlockSymbols - 1) / kBlockSymbols;
    res.n_units = units;
    uint8_t *d_len = (uint8_t *)ctx->dbuf("enc_len", dict_size + 16);
    uint32_t *d_code = (uint32_t *)ctx->dbuf("enc_code", (size_t)dict_size * 4 + 16);
    uint64_t *ubits = (uint64_t *)ctx->dbuf("enc_ubits", (units + 1) * 8);
    uint64_t *uoff = (uint64_t *)ctx->dbuf(ctx->oname("enc_uoff"), (units + 1) * 8);
    {   // the codebook through pinned staging + an SM copy (see small_copy)
        uint8_t *ht = (uint8_t *)ctx->hbuf("enc_tabs_h", (size_t)dict_size * 5 + 16);
        memcpy(ht, codes, (size_t)dict_size * 4);
        memcpy(ht + (size_t)dict_size * 4, lengths, dict_size);
        small_copy(d_code, ht, (size_t)dict_size * 4, s);
        small_copy(d_len, ht + (size_t)dict_size * 4, dict_size, s);
    }
    {
        KPROF("k_unit_bits", 2.0 * n + 8.0 * units, s);
        k_unit_bits<<<(unsigned)std::min<int64_t>(units, 148 * 16), kEncThreads, 0, s>>>(keys, n, d_len, dict_size, ubits,
                                                                                          units);
        LAUNCH_CHECK();
    }
    zero_async(ubits + units, 8, s);
    size_t tb = 0;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, ubits, uoff, (int)(units + 1), s));
    void *tmp = ctx->dbuf("cub_tmp", tb);
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, ubits, uoff, (int)(units + 1), s));
    count_launch();
    // unit groups: the encode runs in G launches so the caller can stream finished byte ranges out
    const int G = hooks && hooks->groups > 1 ? (int)std::min<int64_t>(hooks->groups, std::max<int64_t>(1, units)) : 1;
    std::vector<int64_t> ub(G + 1);
    for (int g = 0; g <= G; g++) ub[g] = units * g / G;
    std::vector<uint64_t> gbit(G + 1, 0);
    if (hist && G == 1) {   // sum of count x length: the stream size is known without waiting for the scan
        uint64_t tot = 0;
        for (uint32_t k = 0; k < dict_size; k++) tot += hist[k] * lengths[k];
        res.total_bits = gbit[1] = tot;
    } else {   // group boundaries (bit offsets) for the streamed fetch
        uint64_t *h = (uint64_t *)ctx->hbuf("enc_total", 8 * (G + 2));
        for (int g = 0; g <= G; g++) small_copy(h + g, uoff + ub[g], 8, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
        res.total_bits = h[G];
        gbit.assign(h, h + G + 1);
    }
    const size_t words = (size_t)((res.total_bits + 31) / 32) + 2;
    res.d_words = (uint32_t *)ctx->dbuf(ctx->oname("enc_words"), words * 4);
    res.d_offsets = uoff;
    {
        static const bool full_zero = getenv("HPDR_ENC_FULL_ZERO") != nullptr;
        if (full_zero) {
            zero_async(res.d_words, words * 4, s);
        } else {
            KPROF("k_zero_unit_bounds", 24.0 * units, s);
            k_zero_unit_bounds<<<grid_for(units, 256, 148 * 4), 256, 0, s>>>(uoff, ubits, res.d_words, units);
            LAUNCH_CHECK();
        }
    }
    if (hooks && hooks->ready) hooks->ready(res);
    const uint64_t pbytes = (res.total_bits + 7) / 8;
    for (int g = 0; g < G; g++) {
        const int64_t cnt = ub[g + 1] - ub[g];
        if (cnt > 0) {
            KPROF("k_encode", (2.0 * n + 16.0 * units + res.total_bits / 8.0) * ((double)cnt / (double)units), s);
            k_encode<<<(unsigned)std::min<int64_t>(cnt, 148 * 8), kEncThreads, 0, s>>>(keys, n, d_len, d_code, dict_size,
                                                                                      uoff, ubits, res.d_words, ub[g],
                                                                                      ub[g + 1]);
            LAUNCH_CHECK();
        }
        if (hooks && hooks->group_done) {
            // bytes [lo, hi) are final: the word shared with the next group is left to that group
            const uint64_t lo = (gbit[g] >> 5) * 4, hi = g + 1 < G ? std::min<uint64_t>((gbit[g + 1] >> 5) * 4, pbytes) : pbytes;
            hooks->group_done(g, std::min(lo, hi), hi);
        }
    }
}

// ===================================================================== decode
namespace {

constexpr int kLutSize = 1 << kLutBits;

struct DecTables {
    long long first_code[258];
    long long first_rank[258];
    long long cnt[258];
    int max_len;
};

__device__ __forceinline__ uint32_t load_be(const uint32_t *w, uint64_t i) {
    return __byte_perm(__ldg(w + i), 0, 0x0123);
}

// ---------------------------------------------------------------- warp-cooperative decode
// One warp per 4096-symbol unit.  The unit's bit range [off_u, off_u+1) is split into 32 lane
// segments; every lane decodes its segment from a guessed start and the guesses are repaired by
// self-synchronisation: each round a lane restarts from where its left neighbour's decode left
// the neighbour's segment, until no start moves (lane 0 starts on the true boundary, so after
// round r lanes 0..r are exact; canonical codes resynchronise within a few codewords, so one or
// two rounds suffice in practice).  Symbol counts are then scanned across the warp and every lane
// re-decodes its exact range, staging 32 symbols per lane in shared memory so the warp writes
// the dequantized coefficients (quantize.py:110-111) with coalesced stores.
// A unit whose walk ends anywhere but exactly on the next unit's offset with exactly its symbol
// count (or that hits an invalid codeword, or max_len > 32) is a non-canonical / corrupted
// stream: lane 0 redoes it with the reference's bit-serial walk (huffman.py:292-313), which also
// produces the reference's error offsets.
constexpr int kDWWarps = 8;
constexpr int kDWStage = 33;    // padded 32-symbol staging row per lane
// per-warp shared payload window, chosen per stream from its largest unit: 1024 / 2048 / 4096 words
// (4096 x 8 / 16 / 32-bit codes); larger units read global memory

// canonical lookup of the codeword at the top of `win` (len 0: no codeword)
__device__ __forceinline__ uint32_t dw_lookup(uint32_t win, const uint32_t *lut, const DecTables &T,
                                              const uint32_t *__restrict__ sym_by_rank, int max_len, int &L) {
    const uint32_t e = lut[win >> (32 - kLutBits)];
    L = (int)(e & 0xffu);
    if (L) return e >> 8;
    // longer codes: the entry holds the shortest code length that has this kLutBits-bit prefix
    // (0: no codeword starts with it); shorter lengths cannot match, so the scan starts there
    const int l0 = (int)((e >> 8) & 0xffu);
    if (!l0) return 0;
    for (int l = l0; l <= max_len; l++) {
        const long long idx = (long long)(win >> (32 - l)) - T.first_code[l];
        if (idx >= 0 && idx < T.cnt[l]) {
            L = l;
            return __ldg(sym_by_rank + T.first_rank[l] + idx);
        }
    }
    L = 0;
    return 0;
}

// Bit positions: SM = the unit's words staged (byte-swapped) in shared memory, positions 32-bit
// and relative to the first staged word; otherwise absolute 64-bit positions over global words.
template <bool SM>
struct DW {
    using Pos = typename std::conditional<SM, uint32_t, uint64_t>::type;
    const uint32_t *w;
    const uint32_t *lut;
    const DecTables *T;
    const uint32_t *sbr;
    int max_len;
    __device__ __forceinline__ uint32_t word(Pos i) const { return SM ? w[i] : load_be(w, (uint64_t)i); }
    // the 32 bits starting at bit p (two independent word loads + funnel shift: no bit buffer)
    __device__ __forceinline__ uint32_t win(Pos p) const {
        const Pos i = p >> 5;
        return __funnelshift_l(word(i + 1), word(i), (uint32_t)p & 31u);
    }
    __device__ __forceinline__ uint32_t sym(Pos p, int &L) const { return dw_lookup(win(p), lut, *T, sbr, max_len, L); }
    // decode from p while p < end; n = symbols; bad = an invalid codeword stopped the walk
    __device__ __forceinline__ Pos scan(Pos p, Pos end, uint32_t &n, bool &bad) const {
        n = 0;
        bad = false;
        while (p < end) {
            int L;
            sym(p, L);
            if (L == 0) {
                bad = true;
                return p;
            }
            p += L;
            n++;
        }
        return p;
    }
    // Re-decode from a new start ns, replaying the previous walk (os -> oe, on symbols) in lockstep:
    // once both walks stand on the same codeword boundary the rest of the old walk is valid.
    __device__ __forceinline__ Pos rescan(Pos ns, Pos os, Pos oe, bool obad, uint32_t on, Pos end, uint32_t &n,
                                          bool &bad) const {
        if (obad || ns >= end) return scan(ns, end, n, bad);
        n = 0;
        bad = false;
        Pos pa = ns, pb = os;
        uint32_t na = 0, nb = 0;
        while (pa < end) {
            if (pa == pb) {
                n = na + (on - nb);
                return oe;
            }
            int L;
            if (pb < pa) {   // valid: the old walk passed here
                sym(pb, L);
                pb += L;
                nb++;
            } else {
                sym(pa, L);
                if (L == 0) {
                    bad = true;
                    return pa;
                }
                pa += L;
                na++;
            }
        }
        n = na;
        return pa;
    }
};

// Self-synchronising decode of one unit whose bits lie in [S, E) (see k_decode_warp), positions
// relative to `base`.  Returns false if the unit is not a canonical layout (the caller falls back
// to the serial walk).  A codeword overrunning E (or the stream limit >= E) shows up as last != E.
template <bool SM>
__device__ __forceinline__ bool dw_unit(const DW<SM> &c, uint64_t base, uint64_t S_, uint64_t E_, uint64_t lo,
                                        uint64_t cnt, uint16_t *st, uint32_t *__restrict__ keys,
                                        double *__restrict__ coef, double bin, unsigned &kmax,
                                        unsigned long long *stats) {
    using Pos = typename DW<SM>::Pos;
    const int lane = threadIdx.x & 31;
    const Pos S = (Pos)(S_ - base), E = (Pos)(E_ - base);
    const Pos seg = (E - S + 31) / 32;
    const Pos send = min(E, (Pos)(S + (Pos)(lane + 1) * seg));
    Pos start = min(E, (Pos)(S + (Pos)lane * seg));
    uint32_t n;
    bool bad;
    Pos exit = c.scan(start, send, n, bad);
    for (int round = 0; round < 32; round++) {
        Pos ns = __shfl_up_sync(0xffffffffu, exit, 1);
        const bool lbad = __shfl_up_sync(0xffffffffu, (int)bad, 1);
        if (lane == 0) ns = S;
        const bool moved = ns != start && (lane == 0 || !lbad);
        if (!__any_sync(0xffffffffu, moved)) break;
        if (stats && lane == 0) atomicAdd(stats + 1, 1ULL);
        if (moved) {
            uint32_t n2;
            bool b2;
            const Pos ex2 = c.rescan(ns, start, exit, bad, n, send, n2, b2);
            start = ns;
            n = n2;
            exit = ex2;
            bad = b2;
        }
    }
    // exact iff every start is its neighbour's exit, no lane failed, the walk ends on E and the
    // unit holds exactly cnt symbols
    Pos left = __shfl_up_sync(0xffffffffu, exit, 1);
    if (lane == 0) left = S;
    uint32_t tot = n;
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const Pos last = __shfl_sync(0xffffffffu, exit, 31);
    if (!(__all_sync(0xffffffffu, left == start && !bad) && last == E && tot == cnt)) return false;
    uint32_t pos = n;   // inclusive scan -> this lane's first output
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, pos, o);
        if (lane >= o) pos += v;
    }
    pos -= n;
    Pos p = start;
    uint32_t done = 0;
    const uint32_t nmax = __reduce_max_sync(0xffffffffu, n);
    for (uint32_t r0 = 0; r0 < nmax; r0 += 32) {
        const uint32_t m = n > r0 ? min(32u, n - r0) : 0u;
        for (uint32_t k = 0; k < m; k++) {
            int L;
            const uint32_t sym = c.sym(p, L);
            p += L;
            st[lane * kDWStage + k] = (uint16_t)sym;   // keys < dict_size <= 65535
            kmax = sym > kmax ? sym : kmax;
        }
        __syncwarp();
        for (int j = 0; j < 32; j++) {
            const uint32_t mj = __shfl_sync(0xffffffffu, m, j);
            const uint32_t bj = __shfl_sync(0xffffffffu, pos + done, j);
            if ((uint32_t)lane < mj) {
                const uint32_t sym = st[j * kDWStage + lane];
                const uint64_t o = lo + bj + lane;
                if (keys) keys[o] = sym;
                if (coef) {
                    const long long b = (long long)(sym >> 1) ^ -(long long)(sym & 1u);
                    coef[o] = __dmul_rn((double)b, bin);
                }
            }
        }
        __syncwarp();
        done += m;
    }
    return true;
}

// The reference walk for one unit (lane 0 of the warp): exact outputs and error offsets.
__device__ void dw_serial_unit(const uint32_t *__restrict__ words, uint64_t limit, uint64_t pos, uint64_t lo,
                               uint64_t cnt, const DecTables &T, const uint32_t *lut,
                               const uint32_t *__restrict__ sym_by_rank, uint32_t *__restrict__ keys,
                               double *__restrict__ coef, double bin, long long &err, unsigned &kmax) {
    const int max_len = T.max_len;
    for (uint64_t i = 0; i < cnt; i++) {
        const uint64_t cw = pos;
        uint32_t sym = 0;
        if (max_len <= 32) {
            if (pos >= limit) { err = (long long)cw; return; }
            const uint64_t wi = pos >> 5;
            const uint64_t win64 = ((uint64_t)load_be(words, wi) << 32) | load_be(words, wi + 1);
            int L;
            sym = dw_lookup((uint32_t)((win64 << (pos & 31)) >> 32), lut, T, sym_by_rank, max_len, L);
            if (L == 0 || pos + (uint64_t)L > limit) { err = (long long)cw; return; }
            pos += L;
        } else {   // wrapping int64 arithmetic of the numba walk (corrupted length arrays only)
            unsigned long long code = 0;
            int len = 0;
            bool ok = false;
            for (;;) {
                if (pos >= limit || len >= max_len) break;
                const uint32_t word = load_be(words, pos >> 5);
                code = (code << 1) | ((word >> (31 - (pos & 31))) & 1u);
                pos++;
                len++;
                const long long idx = (long long)(code - (unsigned long long)T.first_code[len]);
                if (idx >= 0 && idx < T.cnt[len]) {
                    sym = __ldg(sym_by_rank + T.first_rank[len] + idx);
                    ok = true;
                    break;
                }
            }
            if (!ok) { err = (long long)cw; return; }
        }
        kmax = sym > kmax ? sym : kmax;
        if (keys) keys[lo + i] = sym;
        if (coef) {
            const long long b = (long long)(sym >> 1) ^ -(long long)(sym & 1u);
            coef[lo + i] = __dmul_rn((double)b, bin);
        }
    }
}

// ---------------------------------------------------------------- warp-cooperative decode
// One warp per 4096-symbol unit.  The warp stages the unit's payload words in shared memory
// (coalesced), splits its bit range [off_u, off_u+1) into 32 lane segments and decodes every
// segment from a guessed start; guesses are repaired by self-synchronisation (each round a lane
// restarts where its left neighbour's walk left the neighbour's segment, replaying its old walk in
// lockstep until the two meet on a common codeword boundary; lane 0 starts on the true boundary,
// so round r fixes lanes <= r, and canonical codes resynchronise within a few codewords).  Symbol
// counts are scanned across the warp and every lane re-decodes its exact range, staging 32
// symbols per lane in shared memory so the warp writes the dequantized coefficients
// (quantize.py:110-111) with coalesced stores.
// A unit whose walk ends anywhere but exactly on the next unit's offset with exactly its symbol
// count (or that hits an invalid codeword, or max_len > 32) is a non-canonical / corrupted
// stream: lane 0 redoes it with the reference's bit-serial walk (huffman.py:292-313), which also
// produces the reference's error offsets.
size_t dw_smem_bytes(int words) {
    return (size_t)kLutSize * 4 + ((sizeof(DecTables) + 15) & ~size_t(15)) +
           (((size_t)kDWWarps * 32 * kDWStage * 2 + 15) & ~size_t(15)) + (size_t)kDWWarps * words * 4;
}

template <int kDWWords>
__global__ void __launch_bounds__(kDWWarps * 32) k_decode_warp(
    const uint32_t *__restrict__ words, uint64_t limit, const uint64_t *__restrict__ offs, uint64_t nsym,
    int64_t units, const DecTables *__restrict__ tabs_g, const uint32_t *__restrict__ lut_g,
    const uint32_t *__restrict__ sym_by_rank, uint32_t *__restrict__ keys, double *__restrict__ coef, double bin,
    long long *__restrict__ unit_err, unsigned long long *__restrict__ first_bad, unsigned *__restrict__ max_key,
    unsigned long long *__restrict__ stats, int64_t u_lo, int64_t u_hi, int *__restrict__ deferred, int redo) {
    extern __shared__ __align__(16) unsigned char dw_smem[];
    uint32_t *lut = (uint32_t *)dw_smem;
    DecTables &T = *(DecTables *)(dw_smem + kLutSize * 4);
    uint16_t *stage = (uint16_t *)(dw_smem + kLutSize * 4 + ((sizeof(DecTables) + 15) & ~size_t(15)));
    uint32_t *pay = (uint32_t *)((unsigned char *)stage + (((size_t)kDWWarps * 32 * kDWStage * 2 + 15) & ~size_t(15)));
    for (int i = threadIdx.x; i < kLutSize; i += blockDim.x) lut[i] = lut_g[i];
    for (int i = threadIdx.x; i < (int)(sizeof(DecTables) / 8); i += blockDim.x)
        ((long long *)&T)[i] = ((const long long *)tabs_g)[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint16_t *st = stage + wid * 32 * kDWStage;
    uint32_t *pw = pay + wid * kDWWords;
    const int max_len = T.max_len;
    unsigned kmax = 0;
    const int64_t wstride = (int64_t)gridDim.x * kDWWarps;
    for (int64_t u = u_lo + blockIdx.x * (int64_t)kDWWarps + wid; u < u_hi; u += wstride) {
        if (redo && !deferred[u]) continue;   // redo pass: only units deferred by a streamed pass
        const uint64_t lo = (uint64_t)u * kBlockSymbols;
        const uint64_t cnt = nsym - lo < (uint64_t)kBlockSymbols ? nsym - lo : (uint64_t)kBlockSymbols;
        const uint64_t S = __ldg(offs + u);
        const uint64_t E = u + 1 < units ? __ldg(offs + u + 1) : limit;
        bool fast = !redo && max_len <= 32 && S < limit && S <= E && E <= limit && E - S <= cnt * (uint64_t)max_len;
        if (fast) {
            const int64_t w0 = (int64_t)(S >> 5), nw = (int64_t)(E >> 5) + 4 - w0;
            if (nw <= kDWWords) {
                for (int64_t i = lane; i < nw; i += 32) pw[i] = load_be(words, (uint64_t)(w0 + i));
                __syncwarp();
                const DW<true> c{pw, lut, &T, sym_by_rank, max_len};
                fast = dw_unit<true>(c, (uint64_t)w0 * 32, S, E, lo, cnt, st, keys, coef, bin, kmax, stats);
            } else {
                const DW<false> c{words, lut, &T, sym_by_rank, max_len};
                fast = dw_unit<false>(c, 0, S, E, lo, cnt, st, keys, coef, bin, kmax, stats);
                if (stats && lane == 0) atomicAdd(stats + 2, 1ULL);
            }
        }
        if (!fast && deferred && !redo) {   // streamed pass: the walk may need bytes not landed yet
            if (lane == 0) {
                deferred[u] = 1;
                atomicAdd(first_bad + 2, 1ULL);   // deferred-unit count (flag[2])
            }
        } else if (!fast) {
            long long err = -1;
            if (stats && lane == 0) atomicAdd(stats, 1ULL);
            if (lane == 0) {
                dw_serial_unit(words, limit, S, lo, cnt, T, lut, sym_by_rank, keys, coef, bin, err, kmax);
                if (err >= 0) {
                    unit_err[u] = err;
                    atomicMin(first_bad, (unsigned long long)u);
                }
            }
        }
        __syncwarp();
    }
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    if (lane == 0 && kmax) atomicMax(max_key, kmax);
}

__global__ void k_fill(uint32_t *keys, double *coef, int64_t n, uint32_t sym, double val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (keys) keys[i] = sym;
        if (coef) coef[i] = val;
    }
}

}  // namespace

void decode_begin(hpdr_ctx *ctx, const DecodeJob &job, DecodeSession &S, cudaStream_t s, bool copy_payload) {
    // _decode_tables (huffman.py:207-225) and the 12-bit lookup table
    const uint32_t dict = job.dict_size;
    // present keys in (length, key) order: a counting sort over the lengths
    uint32_t lstart[257] = {0};
    int max_len = 0;
    for (uint32_t k = 0; k < dict; k++) {
        lstart[job.lengths[k] + 1]++;
        max_len = std::max<int>(max_len, job.lengths[k]);
    }
    lstart[1] = 0;   // absent keys (length 0) are not ranked
    for (int l = 1; l < 256; l++) lstart[l + 1] += lstart[l];
    std::vector<uint32_t> present(lstart[256]);
    for (uint32_t k = 0; k < dict; k++)
        if (job.lengths[k]) present[lstart[job.lengths[k]]++] = k;
    DecTables *T = (DecTables *)ctx->hbuf("dec_tabs", sizeof(DecTables) + kLutSize * 4 + (present.size() + 1) * 4);
    memset(T, 0, sizeof(DecTables));
    for (uint32_t k : present) T->cnt[job.lengths[k]]++;
    unsigned long long code = 0;
    long long rank = 0;
    for (int ln = 1; ln <= max_len; ln++) {
        if (ln > 1) code <<= 1;
        T->first_code[ln] = (long long)code;
        T->first_rank[ln] = rank;
        code += (unsigned long long)T->cnt[ln];
        rank += T->cnt[ln];
    }
    T->max_len = max_len;
    uint32_t *lut = (uint32_t *)(T + 1);
    uint32_t *sbr = lut + kLutSize;
    for (size_t i = 0; i < present.size(); i++) sbr[i] = present[i];
    // 12-bit lookup: entry v = the shortest code that is a prefix of v (codes of length l fill the
    // entries [c << (12 - l), (c + 1) << (12 - l)); shorter lengths first, filled entries kept)
    const int lut_len = std::min(kLutBits, max_len);
    memset(lut, 0, kLutSize * 4);
    for (int l = 1; l <= lut_len && max_len <= 32; l++) {
        for (long long idx = 0; idx < T->cnt[l]; idx++) {
            const unsigned long long c = (unsigned long long)(T->first_code[l] + idx);
            const unsigned long long lo = c << (kLutBits - l), hi = (c + 1) << (kLutBits - l);
            if (lo >= (unsigned long long)kLutSize) break;
            const uint32_t e = (sbr[T->first_rank[l] + idx] << 8) | (uint32_t)l;
            for (unsigned long long v = lo; v < hi && v < (unsigned long long)kLutSize; v++)
                if (!lut[v]) lut[v] = e;
        }
    }
    // prefixes of codes longer than kLutBits: the shortest such length per prefix (canonical codes
    // of length l cover the prefixes [first >> (l - kLutBits), (first + cnt - 1) >> (l - kLutBits)])
    if (max_len > kLutBits && max_len <= 32)
        for (int l = kLutBits + 1; l <= max_len; l++) {
            if (!T->cnt[l]) continue;
            const unsigned long long f = (unsigned long long)T->first_code[l];
            const unsigned long long lo = f >> (l - kLutBits), hi = (f + T->cnt[l] - 1) >> (l - kLutBits);
            for (unsigned long long v = lo; v <= hi && v < (unsigned long long)kLutSize; v++)
                if (!lut[v]) lut[v] = (uint32_t)l << 8;
        }
    const size_t tab_bytes = sizeof(DecTables) + kLutSize * 4 + (present.size() + 1) * 4;
    char *d_tab = (char *)ctx->dbuf("dec_tabs", tab_bytes);
    small_copy(d_tab, T, tab_bytes, s);

    S.job = job;
    S.max_len = max_len;
    S.d_tab = d_tab;
    S.units = (int64_t)job.n_units;
    const int64_t units = S.units;
    S.d_off = (uint64_t *)ctx->dbuf("dec_off", (units + 1) * 8);
    small_copy(S.d_off, job.offsets, units * 8, s);
    S.pbytes = (size_t)((job.total_bits + 7) / 8);
    S.pwords = ((S.pbytes / 4 + 12) & ~size_t(3));   // zero-padded tail words
    S.d_words = (uint32_t *)ctx->dbuf("dec_words", S.pwords * 4);
    zero_async((char *)S.d_words + (S.pbytes & ~size_t(3)), S.pwords * 4 - (S.pbytes & ~size_t(3)), s);
    S.uerr = (long long *)ctx->dbuf("dec_err", (units + 1) * 8);
    S.flag = (unsigned long long *)ctx->dbuf("dec_flag", 32);
    S.deferred = (int *)ctx->dbuf("dec_defer", (units + 1) * 4);
    zero_async(S.deferred, (units + 1) * 4, s);
    unsigned long long init[4] = {~0ULL, 0ULL, 0ULL, 0ULL};
    unsigned long long *hinit = (unsigned long long *)ctx->hbuf("dec_init", 64);
    memcpy(hinit, init, 32);
    small_copy(S.flag, hinit, 32, s);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_decode_warp<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dw_smem_bytes(1024)));
        CUDA_CHECK(cudaFuncSetAttribute(k_decode_warp<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dw_smem_bytes(2048)));
        CUDA_CHECK(cudaFuncSetAttribute(k_decode_warp<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dw_smem_bytes(4096)));
        attr = true;
    }
    // smallest window holding the largest unit (host offsets: the caller's stream)
    uint64_t max_bits = 0;
    {
        const uint64_t nu = job.n_units;
        uint64_t prev = 0;
        for (uint64_t u = 0; u < nu; u++) {
            uint64_t o;
            memcpy(&o, job.offsets + 8 * u, 8);
            if (u) max_bits = std::max(max_bits, o >= prev ? o - prev : 0);
            prev = o;
        }
        if (nu) max_bits = std::max(max_bits, job.total_bits >= prev ? job.total_bits - prev : 0);
    }
    const uint64_t need_words = max_bits / 32 + 4;
    S.window = need_words <= 1024 ? 1024 : need_words <= 2048 ? 2048 : 4096;
    static const bool want_stats = getenv("HPDR_DECODE_STATS") != nullptr;
    S.stats = nullptr;
    if (want_stats) {
        S.stats = (unsigned long long *)ctx->dbuf("dec_stats", 32);
        zero_async(S.stats, 32, s);
    }
    if (copy_payload && units > 0) {
        if (classify(job.packed) == MemKind::Host && S.pbytes >= (1u << 20)) stage_h2d(ctx, S.d_words, job.packed, S.pbytes, s);
        else CUDA_CHECK(cudaMemcpyAsync(S.d_words, job.packed, S.pbytes, cudaMemcpyDefault, s));
    }
}

void decode_units(const DecodeSession &S, int64_t u_lo, int64_t u_hi, bool streamed, cudaStream_t s, int redo) {
    if (u_hi <= u_lo) return;
    const DecodeJob &job = S.job;
    KPROF("k_decode", (job.total_bits / 8.0 + 8.0 * S.units +
                       (double)job.n_symbols * ((job.keys ? 4 : 0) + (job.coef ? 8 : 0))) *
                          ((double)(u_hi - u_lo) / (double)S.units), s);
    const int per_sm = S.window == 1024 ? 3 : S.window == 2048 ? 2 : 1;   // resident blocks (shared memory)
    const unsigned blocks = (unsigned)std::min<int64_t>((u_hi - u_lo + kDWWarps - 1) / kDWWarps, 148 * per_sm);
#define DWL(W)                                                                                                          \
    k_decode_warp<W><<<blocks, kDWWarps * 32, dw_smem_bytes(W), s>>>(                                                    \
        S.d_words, job.total_bits, S.d_off, job.n_symbols, S.units, (const DecTables *)S.d_tab,                         \
        (const uint32_t *)(S.d_tab + sizeof(DecTables)), (const uint32_t *)(S.d_tab + sizeof(DecTables) + kLutSize * 4), \
        job.keys, job.coef, job.bin_width, S.uerr, S.flag, (unsigned *)(S.flag + 1), S.stats, u_lo, u_hi,              \
        (streamed || redo) ? S.deferred : nullptr, redo)
    if (S.window == 1024) DWL(1024);
    else if (S.window == 2048) DWL(2048);
    else DWL(4096);
#undef DWL
    LAUNCH_CHECK();
}

void decode_end(hpdr_ctx *ctx, const DecodeSession &S, DecodeResult &res, cudaStream_t s, bool streamed) {
    if (streamed) decode_units(S, 0, S.units, false, s, 1);   // deferred units, now with every byte present
    unsigned long long *h = (unsigned long long *)ctx->hbuf("dec_rb", 64);
    small_copy(h, S.flag, 24, s);
    if (S.stats) small_copy(h + 4, S.stats, 16, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (S.stats) fprintf(stderr, "[decode] units %lld fallback %llu rounds %llu deferred %llu\n", (long long)S.units, h[4],
                         h[5], h[2]);
    res.deferred = h[2];
    res.bad_bit = -1;
    if (h[0] != ~0ULL) {
        long long b;
        CUDA_CHECK(cudaMemcpy(&b, S.uerr + h[0], 8, cudaMemcpyDeviceToHost));
        res.bad_bit = b;
    }
    res.max_key = (uint32_t)h[1];
    res.key_out_of_range = res.max_key >= S.job.key_limit;
}

void decode_device(hpdr_ctx *ctx, const DecodeJob &job, DecodeResult &res, cudaStream_t s) {
    DecodeSession S;
    decode_begin(ctx, job, S, s, true);
    decode_units(S, 0, S.units, false, s, 0);
    decode_end(ctx, S, res, s, false);
}

void fill_single(uint32_t *keys, double *coef, int64_t n, uint32_t sym, double bin_width, cudaStream_t s) {
    const long long b = (long long)(sym >> 1) ^ -(long long)(sym & 1u);
    const double val = (double)b * bin_width;
    k_fill<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(keys, coef, n, sym, val);
    LAUNCH_CHECK();
}

}  // namespace hpdr
