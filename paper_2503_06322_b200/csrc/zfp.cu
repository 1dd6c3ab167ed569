// zfp.cu -- the fixed-rate block coder (reference: hpdr/zfp.py) on sm_100a.
//
// Every 4^d block becomes exactly w = 1 + e_bits + rate*4^d bits (zfp.py:64-65), so block b's
// bits start at b*w and the whole stream is a pure function of (dims, dtype, rate).  That makes
// the coder embarrassingly parallel: one thread owns one block end to end (gather with edge
// replication, common exponent, fixed point, reversible lifting, negabinary, bit planes), and a
// CTA of 128 threads owns 128 consecutive blocks = 16*w whole bytes of stream, assembled in
// shared memory and stored with coalesced 32-bit words.  The kernels are HBM-bound
// (4 or 8 B/value in, rate/8 B/value out) -- see DESIGN.md section 10.
//
// The host side streams: the input is copied in dim-0 slabs on the h2d stream, each slab's
// blocks are coded as soon as their planes are resident, and the finished stream bytes go out
// on the d2h stream while the next slab is coded (decompress mirrors it).
#include <algorithm>
#include <cstring>
#include <utility>

#include "context.cuh"

namespace hpdr {
namespace {

constexpr int kZThreads = 128;   // blocks per CTA
constexpr int kZHeader = 3;      // zfp.py:267 "<BBB" rank, dtype code, rate

template <class T>
struct ZSpec;
template <>
struct ZSpec<float> {   // zfp.py:48-49
    using U = uint32_t;
    using S = int32_t;
    static constexpr int q = 32, ebits = 8, bias = 127;
    static constexpr U nb = 0xAAAAAAAAu;
};
template <>
struct ZSpec<double> {   // zfp.py:50-51
    using U = uint64_t;
    using S = int64_t;
    static constexpr int q = 64, ebits = 11, bias = 1023;
    static constexpr U nb = 0xAAAAAAAAAAAAAAAAull;
};

// zfp.py:68-80: k-th block position in sequency order (total per-axis frequency, ties by flat
// index).  Evaluated at compile time so the permutation is free register renaming.
constexpr int seq_perm(int d, int k) {
    const int freq[4] = {0, 3, 1, 2};
    int m = d == 1 ? 4 : d == 2 ? 16 : 64;
    int key[64] = {}, perm[64] = {};
    for (int f = 0; f < m; f++) {
        int s = 0, r = f;
        for (int i = 0; i < d; i++) {
            s += freq[r % 4];
            r /= 4;
        }
        key[f] = s;
        perm[f] = f;
    }
    for (int i = 1; i < m; i++)
        for (int j = i; j > 0 && key[perm[j - 1]] > key[perm[j]]; j--) {
            int t = perm[j];
            perm[j] = perm[j - 1];
            perm[j - 1] = t;
        }
    return perm[k];
}
template <int D, int K>
struct Perm {
    static constexpr int v = seq_perm(D, K);
};

template <class U, class S>
__device__ __forceinline__ U asr1(U v) { return (U)((S)v >> 1); }

// zfp.py:160-180, modulo 2^q (unsigned wrap; >> is the signed arithmetic shift).
template <class U, class S, bool FWD>
__device__ __forceinline__ void lift(U &x, U &y, U &z, U &w) {
    if (FWD) {
        w -= x; x += asr1<U, S>(w);
        y -= z; z += asr1<U, S>(y);
        z -= x; x += asr1<U, S>(z);
        y -= w; w += asr1<U, S>(y);
        w += asr1<U, S>(y); y -= asr1<U, S>(w);
    } else {
        y += asr1<U, S>(w); w -= asr1<U, S>(y);
        w -= asr1<U, S>(y); y += w;
        x -= asr1<U, S>(z); z += x;
        z -= asr1<U, S>(y); y += z;
        x -= asr1<U, S>(w); w += x;
    }
}

// zfp.py:183-201: forward along in-block axes slowest first, inverse in reverse order.
template <int D, class U, class S, bool FWD>
__device__ __forceinline__ void transform(U (&v)[1 << (2 * D)]) {
    constexpr int M = 1 << (2 * D);
#pragma unroll
    for (int t = 0; t < D; t++) {
        const int ax = FWD ? t : D - 1 - t;
        const int st = 1 << (2 * (D - 1 - ax));
#pragma unroll
        for (int f = 0; f < M; f++)
            if (((f / st) & 3) == 0) lift<U, S, FWD>(v[f], v[f + st], v[f + 2 * st], v[f + 3 * st]);
    }
}

template <int D, class U, int... K>
__device__ __forceinline__ void gather_perm(const U (&src)[1 << (2 * D)], U (&dst)[1 << (2 * D)],
                                            std::integer_sequence<int, K...>) {
    ((dst[K] = src[Perm<D, K>::v]), ...);
}
template <int D, class U, int... K>
__device__ __forceinline__ void scatter_perm(const U (&src)[1 << (2 * D)], U (&dst)[1 << (2 * D)],
                                             std::integer_sequence<int, K...>) {
    ((dst[Perm<D, K>::v] = src[K]), ...);
}

// MSB-first bit writer into shared 32-bit words (word 0 bit 31 = first stream bit).  Only a
// thread's first and last words can be shared with its neighbours; atomicOr covers both.
struct BitWriter {
    uint32_t *s;
    uint32_t idx;
    uint64_t acc;
    int n;
    __device__ BitWriter(uint32_t *sm, uint32_t pos) : s(sm), idx(pos >> 5), acc(0), n(pos & 31) {}
    __device__ __forceinline__ void put(uint32_t v, int nb) {   // 1 <= nb <= 32, v < 2^nb
        acc = (acc << nb) | v;   // n + nb <= 63 meaningful bits
        n += nb;
        if (n >= 32) {
            n -= 32;
            atomicOr(&s[idx++], (uint32_t)(acc >> n));
        }
    }
    __device__ __forceinline__ void flush() {
        if (n) atomicOr(&s[idx], (uint32_t)(acc << (32 - n)));
    }
};

struct BitReader {
    const uint32_t *s;
    uint32_t pos;
    __device__ __forceinline__ uint32_t get(int nb) {   // 1 <= nb <= 32; s has one spare word
        const uint32_t w = pos >> 5, o = pos & 31;
        const uint64_t two = ((uint64_t)s[w] << 32) | s[w + 1];
        pos += nb;
        return (uint32_t)((two << o) >> (64 - nb));
    }
};

struct ZGrid {
    int64_t n[3];   // extents padded to rank 3 with leading 1s
    int64_t g[3];   // blocks per axis
};

// Element offsets of the block's 4^D positions, edge-replicated (np.pad mode="edge", zfp.py:98-100).
template <int D>
__device__ __forceinline__ void block_rows(const ZGrid &G, int64_t b, int64_t (&row)[16], int64_t (&col)[4]) {
    const int64_t b2 = b % G.g[2], r = b / G.g[2];
    const int64_t b1 = r % G.g[1], b0 = r / G.g[1];
#pragma unroll
    for (int i = 0; i < 4; i++) col[i] = min64(b2 * 4 + i, G.n[2] - 1);
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int64_t i0 = D == 3 ? min64(b0 * 4 + a, G.n[0] - 1) : 0;
            const int64_t i1 = D >= 2 ? min64(b1 * 4 + (D == 3 ? c : a), G.n[1] - 1) : 0;
            row[a * 4 + c] = (i0 * G.n[1] + i1) * G.n[2];
        }
}

template <int D>
__device__ __forceinline__ int64_t elem_at(const int64_t (&row)[16], const int64_t (&col)[4], int f) {
    // f = flat in-block position, row-major over the block's D axes
    if (D == 3) return row[(f >> 4) * 4 + ((f >> 2) & 3)] + col[f & 3];
    if (D == 2) return row[(f >> 2) * 4] + col[f & 3];
    return row[0] + col[f & 3];
}

// zfp_compress per block (zfp.py:291-303): exp_align :125-150, forward_transform :194-196,
// bitplane_encode :217-241.  Stream words go to out32 (MSB-first bits, byte-swapped on store so
// memory holds the np.packbits byte order).
template <class T, int D>
__global__ void __launch_bounds__(kZThreads) k_zfp_encode(const T *__restrict__ in, ZGrid G, int64_t b_lo,
                                                           int64_t b_hi, int rate, uint32_t *__restrict__ out32,
                                                           unsigned *__restrict__ bad) {
    using Z = ZSpec<T>;
    using U = typename Z::U;
    using S = typename Z::S;
    constexpr int M = 1 << (2 * D);
    extern __shared__ uint32_t zs[];
    const uint32_t w = 1 + Z::ebits + (uint32_t)rate * M;
    const int64_t cta0 = b_lo + (int64_t)blockIdx.x * kZThreads;
    const int nblk = (int)min64(kZThreads, b_hi - cta0);
    const uint32_t words = (uint32_t)(((uint64_t)nblk * w + 31) / 32);
    for (uint32_t i = threadIdx.x; i < words; i += kZThreads) zs[i] = 0;
    __syncthreads();
    if ((int)threadIdx.x < nblk) {
        const int64_t b = cta0 + threadIdx.x;
        int64_t row[16], col[4];
        block_rows<D>(G, b, row, col);
        T v[M];   // widened to double on use (exact), as np.asarray(blocks, float64) does
        double maxabs = 0.0;
        bool finite = true;
#pragma unroll
        for (int f = 0; f < M; f++) {
            v[f] = __ldg(in + elem_at<D>(row, col, f));
            const double a = fabs((double)v[f]);
            finite &= a <= 1.79769313486231570815e308;   // false for inf and NaN
            maxabs = fmax(maxabs, a);
        }
        if (!finite) atomicOr(bad, 1u);
        const bool zero = maxabs == 0.0;
        // floor(log2(maxabs)) exactly (the :139-144 guards make the reference exact too)
        int emax = zero ? 0 : ilogb(maxabs);
        emax = max(emax, -Z::bias);
        const int shift = Z::q - 2 - emax;
        U fx[M];
#pragma unroll
        for (int f = 0; f < M; f++) fx[f] = zero ? (U)0 : (U)(S)rint(ldexp((double)v[f], shift));
        transform<D, U, S, true>(fx);
        U c[M];
        gather_perm<D, U>(fx, c, std::make_integer_sequence<int, M>{});
#pragma unroll
        for (int k = 0; k < M; k++) c[k] = zero ? (U)0 : (U)((c[k] + Z::nb) ^ Z::nb);   // zfp.py:204-208
        BitWriter bw(zs, (uint32_t)threadIdx.x * w);
        bw.put(zero ? 1u : 0u, 1);
        bw.put(zero ? 0u : (uint32_t)(emax + Z::bias), Z::ebits);
        for (int t = 0; t < rate; t++) {
            const int sh = Z::q - 1 - t;
            if (D == 3) {
                uint32_t hi = 0, lo = 0;
#pragma unroll
                for (int k = 0; k < 32; k++) hi |= (uint32_t)((c[k] >> sh) & 1) << (31 - k);
#pragma unroll
                for (int k = 0; k < 32; k++) lo |= (uint32_t)((c[32 + k] >> sh) & 1) << (31 - k);
                bw.put(hi, 32);
                bw.put(lo, 32);
            } else {
                uint32_t p = 0;
#pragma unroll
                for (int k = 0; k < M; k++) p |= (uint32_t)((c[k] >> sh) & 1) << (M - 1 - k);
                bw.put(p, M);
            }
        }
        bw.flush();
    }
    __syncthreads();
    uint32_t *dst = out32 + (uint64_t)(cta0 - b_lo) * w / 32;
    for (uint32_t i = threadIdx.x; i < words; i += kZThreads) dst[i] = __byte_perm(zs[i], 0, 0x0123);
}

// zfp_decompress per block (zfp.py:338-347): bitplane_decode :244-264, inverse_transform,
// exp_restore :153-157 (ldexp in double, then the cast for F32), zero blocks -> 0.0.
template <class T, int D>
__global__ void __launch_bounds__(kZThreads) k_zfp_decode(const uint32_t *__restrict__ in32, ZGrid G, int64_t b_lo,
                                                           int64_t b_hi, int rate, T *__restrict__ out) {
    using Z = ZSpec<T>;
    using U = typename Z::U;
    using S = typename Z::S;
    constexpr int M = 1 << (2 * D);
    extern __shared__ uint32_t zs[];
    const uint32_t w = 1 + Z::ebits + (uint32_t)rate * M;
    const int64_t cta0 = b_lo + (int64_t)blockIdx.x * kZThreads;
    const int nblk = (int)min64(kZThreads, b_hi - cta0);
    const uint32_t words = (uint32_t)(((uint64_t)nblk * w + 31) / 32);
    const uint32_t *src = in32 + (uint64_t)(cta0 - b_lo) * w / 32;
    for (uint32_t i = threadIdx.x; i <= words; i += kZThreads)
        zs[i] = i < words ? __byte_perm(__ldg(src + i), 0, 0x0123) : 0u;
    __syncthreads();
    if ((int)threadIdx.x >= nblk) return;
    const int64_t b = cta0 + threadIdx.x;
    BitReader br{zs, (uint32_t)threadIdx.x * w};
    const bool zero = br.get(1) != 0;
    const int biased = (int)br.get(Z::ebits);
    const int emax = zero ? -Z::bias : biased - Z::bias;
    U c[M];
#pragma unroll
    for (int k = 0; k < M; k++) c[k] = 0;
    for (int t = 0; t < rate; t++) {
        const int sh = Z::q - 1 - t;
        if (D == 3) {
            const uint32_t hi = br.get(32), lo = br.get(32);
#pragma unroll
            for (int k = 0; k < 32; k++) c[k] |= (U)((hi >> (31 - k)) & 1) << sh;
#pragma unroll
            for (int k = 0; k < 32; k++) c[32 + k] |= (U)((lo >> (31 - k)) & 1) << sh;
        } else {
            const uint32_t p = br.get(M);
#pragma unroll
            for (int k = 0; k < M; k++) c[k] |= (U)((p >> (M - 1 - k)) & 1) << sh;
        }
    }
#pragma unroll
    for (int k = 0; k < M; k++) c[k] = (U)((c[k] ^ Z::nb) - Z::nb);   // zfp.py:211-214
    U fx[M];
    scatter_perm<D, U>(c, fx, std::make_integer_sequence<int, M>{});
    transform<D, U, S, false>(fx);
    const int64_t b2 = b % G.g[2], r = b / G.g[2];
    const int64_t b1 = r % G.g[1], b0 = r / G.g[1];
    const int sc = emax - (Z::q - 2);
#pragma unroll
    for (int f = 0; f < M; f++) {
        const int p0 = D == 3 ? f >> 4 : 0, p1 = D == 3 ? (f >> 2) & 3 : D == 2 ? f >> 2 : 0, p2 = f & 3;
        const int64_t i0 = b0 * 4 + p0, i1 = b1 * 4 + p1, i2 = b2 * 4 + p2;
        if (i0 >= G.n[0] || i1 >= G.n[1] || i2 >= G.n[2]) continue;   // padding is discarded
        const double val = zero ? 0.0 : ldexp((double)(S)fx[f], sc);
        out[(i0 * G.n[1] + i1) * G.n[2] + i2] = (T)val;
    }
}

struct ZfpShape {
    int dtype = 0, rank = 0, rate = 0;
    uint64_t dims[3] = {1, 1, 1};
    ZGrid G{};
    int64_t nblk = 0;
    uint32_t w = 0;          // bits per block
    uint64_t payload = 0;    // bytes
    uint64_t total = 0;      // stream bytes
    int64_t blocks_per_plane = 0;   // blocks in one dim-0 block row
};

int zspec_q(int dtype) { return dtype == 0 ? 32 : 64; }

void zfp_shape(int dtype, int rank, const uint64_t *dims, int rate, ZfpShape &z) {
    if (dtype != 0 && dtype != 1) throw Error{HPDR_ERR_VALIDATION, "fix-rate compression needs F32/F64", -1};
    const int q = zspec_q(dtype);
    if (rate < 1 || rate > q)
        throw Error{HPDR_ERR_VALIDATION, "rate must be in [1, " + std::to_string(q) + "], got " + std::to_string(rate), -1};
    if (rank < 1) throw Error{HPDR_ERR_VALIDATION, "dims must be non-empty", -1};
    if (rank > 3) throw Error{HPDR_ERR_VALIDATION, "rank " + std::to_string(rank) + " > 3 unsupported", -1};
    z.dtype = dtype;
    z.rank = rank;
    z.rate = rate;
    for (int i = 0; i < 3; i++) z.G.n[i] = 1;
    for (int i = 0; i < rank; i++) {
        if (dims[i] < 1) throw Error{HPDR_ERR_VALIDATION, "every extent must be >= 1", -1};
        z.dims[i] = dims[i];
        z.G.n[3 - rank + i] = (int64_t)dims[i];
    }
    z.nblk = 1;
    for (int i = 0; i < 3; i++) {
        z.G.g[i] = (z.G.n[i] + 3) / 4;
        z.nblk *= z.G.g[i];
    }
    z.w = 1 + (dtype == 0 ? 8 : 11) + (uint32_t)rate * (1u << (2 * rank));
    z.payload = ((uint64_t)z.nblk * z.w + 7) / 8;
    z.total = kZHeader + 8ull * rank + z.payload;
    z.blocks_per_plane = z.G.g[1] * z.G.g[2];
}

size_t zfp_smem(const ZfpShape &z) { return ((size_t)kZThreads * z.w / 32 + 1) * 4; }

template <class T, int D>
void launch_encode(const ZfpShape &z, const void *in, int64_t lo, int64_t hi, uint32_t *out32, unsigned *bad,
                   cudaStream_t s) {
    if (hi <= lo) return;
    const size_t smem = zfp_smem(z);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_zfp_encode<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
    }
    const unsigned grid = (unsigned)((hi - lo + kZThreads - 1) / kZThreads);
    KPROF("k_zfp_encode", (double)(hi - lo) * ((double)(1 << (2 * D)) * sizeof(T) + z.w / 8.0), s);
    k_zfp_encode<T, D><<<grid, kZThreads, smem, s>>>((const T *)in, z.G, lo, hi, z.rate, out32, bad);
    LAUNCH_CHECK();
}

template <class T, int D>
void launch_decode(const ZfpShape &z, const uint32_t *in32, int64_t lo, int64_t hi, void *out, cudaStream_t s) {
    if (hi <= lo) return;
    const size_t smem = zfp_smem(z) + 4;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_zfp_decode<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
    }
    const unsigned grid = (unsigned)((hi - lo + kZThreads - 1) / kZThreads);
    KPROF("k_zfp_decode", (double)(hi - lo) * ((double)(1 << (2 * D)) * sizeof(T) + z.w / 8.0), s);
    k_zfp_decode<T, D><<<grid, kZThreads, smem, s>>>(in32, z.G, lo, hi, z.rate, (T *)out);
    LAUNCH_CHECK();
}

void encode_range(const ZfpShape &z, const void *in, int64_t lo, int64_t hi, uint32_t *out32, unsigned *bad,
                  cudaStream_t s) {
    if (z.dtype == 0) {
        if (z.rank == 1) launch_encode<float, 1>(z, in, lo, hi, out32, bad, s);
        else if (z.rank == 2) launch_encode<float, 2>(z, in, lo, hi, out32, bad, s);
        else launch_encode<float, 3>(z, in, lo, hi, out32, bad, s);
    } else {
        if (z.rank == 1) launch_encode<double, 1>(z, in, lo, hi, out32, bad, s);
        else if (z.rank == 2) launch_encode<double, 2>(z, in, lo, hi, out32, bad, s);
        else launch_encode<double, 3>(z, in, lo, hi, out32, bad, s);
    }
}

void decode_range(const ZfpShape &z, const uint32_t *in32, int64_t lo, int64_t hi, void *out, cudaStream_t s) {
    if (z.dtype == 0) {
        if (z.rank == 1) launch_decode<float, 1>(z, in32, lo, hi, out, s);
        else if (z.rank == 2) launch_decode<float, 2>(z, in32, lo, hi, out, s);
        else launch_decode<float, 3>(z, in32, lo, hi, out, s);
    } else {
        if (z.rank == 1) launch_decode<double, 1>(z, in32, lo, hi, out, s);
        else if (z.rank == 2) launch_decode<double, 2>(z, in32, lo, hi, out, s);
        else launch_decode<double, 3>(z, in32, lo, hi, out, s);
    }
}

template <class F>
int zguard(F &&f) {
    try {
        f();
        return HPDR_OK;
    } catch (const Error &e) {
        set_error(e.code, e.msg, e.bit_offset);
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error(HPDR_ERR_ALLOCATION, "host allocation failed");
        return HPDR_ERR_ALLOCATION;
    }
}

// Header checks of zfp_decompress, in the reference's order (zfp.py:314-334).
void zfp_parse(const uint8_t *d, uint64_t len, ZfpShape &z) {
    if (len < (uint64_t)kZHeader) throw Error{HPDR_ERR_CORRUPT, "stream shorter than header", -1};
    const int rank = d[0], code = d[1], rate = d[2];
    if (rank < 1 || rank > 3 || code > 6) throw Error{HPDR_ERR_CORRUPT, "bad rank or dtype code", -1};
    if (code != 0 && code != 1) throw Error{HPDR_ERR_CORRUPT, "stored dtype is not a float type", -1};
    const int q = zspec_q(code);
    if (rate < 1 || rate > q)
        throw Error{HPDR_ERR_VALIDATION, "rate must be in [1, " + std::to_string(q) + "], got " + std::to_string(rate), -1};
    // the reference's struct.unpack_from raises struct.error here; reported as a corrupt stream
    if (len < (uint64_t)kZHeader + 8ull * rank) throw Error{HPDR_ERR_CORRUPT, "stream truncated in dims", -1};
    uint64_t dims[3];
    memcpy(dims, d + kZHeader, 8ull * rank);
    for (int i = 0; i < rank; i++)
        if (dims[i] < 1 || dims[i] > (1ull << 40)) throw Error{HPDR_ERR_CORRUPT, "bad extent in header", -1};
    zfp_shape(code, rank, dims, rate, z);
    if (len - (kZHeader + 8ull * rank) < z.payload)
        throw Error{HPDR_ERR_CORRUPT, "payload truncated: need " + std::to_string(z.payload) + " bytes", -1};
}

// Slab schedule of the streamed paths: about `want` slabs along dim 0, with every boundary a
// multiple of kZThreads blocks so each slab's stream starts on a 32-bit word (128*w bits).
std::vector<int64_t> zfp_slabs(const ZfpShape &z, int want) {
    std::vector<int64_t> cut{0};
    const int64_t rows = z.G.g[0];
    for (int k = 1; k < want; k++) {
        int64_t b = rows * k / want * z.blocks_per_plane;
        b = b / kZThreads * kZThreads;
        if (b > cut.back() && b < z.nblk) cut.push_back(b);
    }
    cut.push_back(z.nblk);
    return cut;
}

int zfp_slab_count(const ZfpShape &z, uint64_t in_bytes) {
    static const char *e = getenv("HPDR_ZFP_SLABS");
    if (e) return std::max(1, atoi(e));
    // ~32 MB of input per slab, at most 16 slabs
    return (int)std::min<uint64_t>(16, std::max<uint64_t>(1, in_bytes / (32ull << 20)));
}

}  // namespace
}  // namespace hpdr

using namespace hpdr;

extern "C" {

int hpdr_zfp_compressed_size(int dtype, int rank, const uint64_t *dims, uint32_t rate, uint64_t *size) {
    return zguard([&] {
        ZfpShape z;
        zfp_shape(dtype, rank, dims, (int)std::min<uint32_t>(rate, 1u << 20), z);
        *size = z.total;
    });
}

int hpdr_zfp_peek(const void *stream, uint64_t len, int *dtype, int *rank, uint64_t *dims, uint32_t *rate) {
    return zguard([&] {
        uint8_t head[kZHeader + 24];
        const uint8_t *d = (const uint8_t *)stream;
        if (stream && classify(stream) == MemKind::Device) {
            CUDA_CHECK(cudaMemcpy(head, stream, std::min<uint64_t>(len, sizeof(head)), cudaMemcpyDeviceToHost));
            d = head;
        }
        ZfpShape z;
        zfp_parse(d, len, z);
        *dtype = z.dtype;
        *rank = z.rank;
        *rate = (uint32_t)z.rate;
        for (int i = 0; i < z.rank; i++) dims[i] = z.dims[i];
    });
}

int hpdr_zfp_compress(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, uint32_t rate,
                      void *out, uint64_t out_cap, uint64_t *out_len) {
    return zguard([&] {
        ZfpShape z;
        zfp_shape(dtype, rank, dims, (int)std::min<uint32_t>(rate, 1u << 20), z);
        *out_len = z.total;
        if (!out || out_cap < z.total)
            throw Error{HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(z.total), -1};
        CUDA_CHECK(cudaSetDevice(ctx->device));
        const int isz = dtype == 0 ? 4 : 8;
        const uint64_t n = (uint64_t)z.G.n[0] * z.G.n[1] * z.G.n[2];
        const uint64_t plane_bytes = (uint64_t)z.G.n[1] * z.G.n[2] * isz;
        const bool in_dev = classify(in) == MemKind::Device;
        const MemKind ok = classify(out);
        const bool out_dev = ok == MemKind::Device;
        cudaStream_t s = ctx->stream;
        // header (zfp.py:306-308)
        uint8_t head[kZHeader + 24];
        head[0] = (uint8_t)rank;
        head[1] = (uint8_t)dtype;
        head[2] = (uint8_t)rate;
        memcpy(head + kZHeader, dims, 8ull * rank);
        const uint64_t hl = kZHeader + 8ull * rank;
        uint8_t *o = (uint8_t *)out;
        if (out_dev) CUDA_CHECK(cudaMemcpyAsync(o, head, hl, cudaMemcpyHostToDevice, s));
        else memcpy(o, head, hl);
        uint32_t *pay = (uint32_t *)ctx->dbuf("zfp_pay", z.payload + 8);
        unsigned *bad = (unsigned *)ctx->dbuf("zfp_bad", 16);
        unsigned *bad_h = (unsigned *)ctx->hbuf("zfp_bad_h", 16);
        CUDA_CHECK(cudaMemsetAsync(bad, 0, 4, s));
        const void *din = in;
        const std::vector<int64_t> cut = zfp_slabs(z, in_dev ? 1 : zfp_slab_count(z, n * isz));
        const int K = (int)cut.size() - 1;
        if (!in_dev) din = ctx->dbuf("zfp_in", n * isz);
        // pageable destinations are written through a pinned staging copy
        uint8_t *stage = (!out_dev && ok == MemKind::Host) ? (uint8_t *)ctx->hbuf("zfp_stage", z.payload) : nullptr;
        uint64_t in_done = 0;   // planes resident
        for (int k = 0; k < K; k++) {
            const int64_t lo = cut[k], hi = cut[k + 1];
            if (!in_dev) {
                // planes needed by blocks [lo, hi): through the last block row, edge rows included
                const int64_t last_row = (hi - 1) / z.blocks_per_plane;
                const uint64_t need = std::min<uint64_t>((uint64_t)z.G.n[0], (uint64_t)(last_row + 1) * 4);
                if (need > in_done) {
                    CUDA_CHECK(cudaMemcpyAsync((uint8_t *)din + in_done * plane_bytes,
                                               (const uint8_t *)in + in_done * plane_bytes,
                                               (need - in_done) * plane_bytes, cudaMemcpyHostToDevice, ctx->h2d));
                    in_done = need;
                }
                CUDA_CHECK(cudaEventRecord(ctx->event(400 + k), ctx->h2d));
                CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(400 + k), 0));
            }
            encode_range(z, din, lo, hi, pay + (uint64_t)lo * z.w / 32, bad, s);
            // stream bytes [lo*w/8, hi*w/8) are final (lo, hi multiples of 32 blocks, or the end)
            const uint64_t a = (uint64_t)lo * z.w / 8;
            const uint64_t e = k == K - 1 ? z.payload : (uint64_t)hi * z.w / 8;
            CUDA_CHECK(cudaEventRecord(ctx->event(420 + k), s));
            CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(420 + k), 0));
            if (out_dev)
                CUDA_CHECK(cudaMemcpyAsync(o + hl + a, (uint8_t *)pay + a, e - a, cudaMemcpyDeviceToDevice, ctx->d2h));
            else
                CUDA_CHECK(cudaMemcpyAsync((stage ? stage : o + hl) + a, (uint8_t *)pay + a, e - a,
                                           cudaMemcpyDeviceToHost, ctx->d2h));
        }
        CUDA_CHECK(cudaMemcpyAsync(bad_h, bad, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
        if (*bad_h) throw Error{HPDR_ERR_VALIDATION, "non-finite values cannot be aligned", -1};
        if (stage) memcpy(o + hl, stage, z.payload);
    });
}

int hpdr_zfp_decompress(hpdr_ctx *ctx, const void *stream, uint64_t len, void *out, uint64_t out_bytes) {
    return zguard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        const bool in_dev = classify(stream) == MemKind::Device;
        uint8_t head[kZHeader + 24];
        const uint8_t *hp = (const uint8_t *)stream;
        if (in_dev) {
            CUDA_CHECK(cudaMemcpy(head, stream, std::min<uint64_t>(len, sizeof(head)), cudaMemcpyDeviceToHost));
            hp = head;
        }
        ZfpShape z;
        zfp_parse(hp, len, z);
        const int isz = z.dtype == 0 ? 4 : 8;
        const uint64_t plane_elems = (uint64_t)z.G.n[1] * z.G.n[2];
        const uint64_t n = (uint64_t)z.G.n[0] * plane_elems;
        if (out_bytes < n * isz) throw Error{HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(n * isz), -1};
        const uint64_t hl = kZHeader + 8ull * z.rank;
        const MemKind ok = classify(out);
        const bool out_dev = ok == MemKind::Device;
        cudaStream_t s = ctx->stream;
        uint32_t *pay = (uint32_t *)ctx->dbuf("zfp_dpay", z.payload + 8);
        void *dout = out_dev ? out : ctx->dbuf("zfp_out", n * isz);
        const std::vector<int64_t> cut = zfp_slabs(z, (in_dev && out_dev) ? 1 : zfp_slab_count(z, n * isz));
        const int K = (int)cut.size() - 1;
        uint64_t rows_out = 0;   // output planes copied out
        uint64_t pay_in = 0;     // payload bytes resident
        for (int k = 0; k < K; k++) {
            const int64_t lo = cut[k], hi = cut[k + 1];
            const uint64_t need = k == K - 1 ? z.payload : ((uint64_t)hi * z.w + 7) / 8;
            if (need > pay_in) {
                CUDA_CHECK(cudaMemcpyAsync((uint8_t *)pay + pay_in, (const uint8_t *)stream + hl + pay_in, need - pay_in,
                                           in_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->h2d));
                pay_in = need;
            }
            CUDA_CHECK(cudaEventRecord(ctx->event(440 + k), ctx->h2d));
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(440 + k), 0));
            decode_range(z, pay + (uint64_t)lo * z.w / 32, lo, hi, dout, s);
            if (out_dev) continue;
            // output planes whose block rows are complete
            const uint64_t rows = k == K - 1 ? (uint64_t)z.G.n[0]
                                             : std::min<uint64_t>((uint64_t)z.G.n[0], (uint64_t)(hi / z.blocks_per_plane) * 4);
            if (rows > rows_out) {
                CUDA_CHECK(cudaEventRecord(ctx->event(460 + k), s));
                CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(460 + k), 0));
                CUDA_CHECK(cudaMemcpyAsync((uint8_t *)out + rows_out * plane_elems * isz,
                                           (uint8_t *)dout + rows_out * plane_elems * isz,
                                           (rows - rows_out) * plane_elems * isz, cudaMemcpyDeviceToHost, ctx->d2h));
                rows_out = rows;
            }
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
    });
}

}  // extern "C"
