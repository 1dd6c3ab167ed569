// zfp.cu -- the fixed-rate block coder (reference: hpdr/zfp.py) on sm_100a.
//
// Every 4^d block becomes exactly w = 1 + e_bits + rate*4^d bits (zfp.py:64-65), so block b's
// bits start at b*w and the whole stream is a pure function of (dims, dtype, rate).  That makes
// the coder embarrassingly parallel: one thread owns one block end to end (gather with edge
// replication, common exponent, fixed point, reversible lifting, negabinary, bit planes), and a
// CTA of 128 threads owns 128 consecutive blocks = 16*w whole bytes of stream, assembled in
// shared memory and stored with coalesced 16-byte vector stores.  The roofline is HBM (4 or 8
// B/value in, rate/8 B/value out); measured at 0.4-0.5 of it, issue-bound -- DESIGN.md section 10.
//
// The host side streams: the input is copied in dim-0 slabs on the h2d stream, each slab's
// blocks are coded as soon as their planes are resident, and the finished stream bytes go out
// on the d2h stream while the next slab is coded (decompress mirrors it).
#include <algorithm>
#include <array>
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
// thread's first and last words can be shared with its neighbours (atomicOr); the words between
// are its own (plain stores).
struct BitWriter {
    uint32_t *s;
    uint32_t idx, first;
    uint64_t acc;
    int n;
    __device__ BitWriter(uint32_t *sm, uint32_t pos) : s(sm), idx(pos >> 5), first(pos >> 5), acc(0), n(pos & 31) {}
    __device__ __forceinline__ void put(uint32_t v, int nb) {   // 1 <= nb <= 32, v < 2^nb
        acc = (acc << nb) | v;   // n + nb <= 63 meaningful bits
        n += nb;
        if (n >= 32) {
            n -= 32;
            const uint32_t word = (uint32_t)(acc >> n);
            if (idx == first) atomicOr(&s[idx], word);
            else s[idx] = word;
            idx++;
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

// In-register 32x32 bit-matrix transpose, MSB-first: A[OFF+i] bit (31-j) <-> A[OFF+j] bit (31-i).
// Turns 32 coefficients into 32 bit planes (and back).  The 16- and 8-bit stages are byte
// permutes; the 4/2/1-bit stages are two shift+LOP3 pairs (the masks satisfy m << j == ~m).
//
// With `need` < 32 only output rows [0, need) are completed (the encoder's truncated planes):
// after the 16-row stage, row t depends only on the rows of its own aligned group, so groups
// starting at or beyond `need` are skipped.
template <int OFF, int N>
__device__ __forceinline__ void transpose32(uint32_t (&A)[N], int need = 32) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
        const uint32_t a = A[OFF + i], b = A[OFF + i + 16];
        A[OFF + i] = __byte_perm(a, b, 0x3276);        // a.hi16 : b.hi16
        A[OFF + i + 16] = __byte_perm(a, b, 0x1054);   // a.lo16 : b.lo16
    }
#pragma unroll
    for (int base = 0; base < 32; base += 16)
        if (base < need) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const uint32_t a = A[OFF + base + i], b = A[OFF + base + i + 8];
                A[OFF + base + i] = __byte_perm(a, b, 0x3715);
                A[OFF + base + i + 8] = __byte_perm(a, b, 0x2604);
            }
        }
#pragma unroll
    for (int lj = 2; lj >= 0; lj--) {
        const int j = 1 << lj;
        const uint32_t m = lj == 2 ? 0x0F0F0F0Fu : lj == 1 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int base = 0; base < 32; base += 2 * j)
            if (base < need) {
#pragma unroll
                for (int i = 0; i < j; i++) {
                    const uint32_t a = A[OFF + base + i], b = A[OFF + base + i + j];
                    A[OFF + base + i] = (a & ~m) | ((b >> j) & m);
                    A[OFF + base + i + j] = (b & m) | ((a << j) & ~m);
                }
            }
    }
}

// 2^e, exact: doubles for -1022 <= e <= 1023, floats for -126 <= e <= 127.
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ float pow2f(int e) { return __uint_as_float((uint32_t)(e + 127) << 23); }

// exp_align (zfp.py:125-150) for one block: e_max = floor(log2(max|v|)) clamped to -bias, then
// fixed = rint(ldexp(v, q-2-e_max)).  The reference works in float64; these are exact restatements:
//  * F32: |v| ordering, the exponent and v * 2^shift are all exact in fp32 (the scaled value keeps
//    v's 24-bit significand, |v * 2^shift| < 2^31), so the fp32 multiply + round-to-nearest-even
//    convert equals rint of the float64 product.  Products that underflow round to 0 either way.
//  * F64: one multiply by 2^shift is exact unless the product is subnormal (< 0.5, so rint gives 0
//    either way); shift > 1023 only for e_max < -961, where v * 2^(shift-64) is exact and normal.
template <class T, int M>
__device__ __forceinline__ void align_block(const T (&v)[M], typename ZSpec<T>::U (&fx)[M], int &emax, bool &zero,
                                            bool &finite) {
    using U = typename ZSpec<T>::U;
    if constexpr (sizeof(T) == 4) {
        float m = 0.f;
        finite = true;
#pragma unroll
        for (int f = 0; f < M; f++) {
            const float a = fabsf(v[f]);
            finite &= a <= 3.40282346638528859812e38f;
            m = fmaxf(m, a);
        }
        zero = m == 0.f;
        emax = max((int)(__float_as_uint(m) >> 23) - 127, -127);   // subnormal maxima clamp to -127
        const int shift = 30 - emax;                                  // in [-98, 157]
        // 2^shift as two exact factors (2^shift * 1, or 2^(shift-64) * 2^64 above 2^127)
        const bool big = shift > 127;
        const float s1 = pow2f(big ? shift - 64 : shift), s2 = big ? pow2f(64) : 1.0f;
#pragma unroll
        for (int f = 0; f < M; f++) fx[f] = (U)__float2int_rn(__fmul_rn(__fmul_rn(v[f], s1), s2));
    } else {
        double m = 0.0;
        finite = true;
#pragma unroll
        for (int f = 0; f < M; f++) {
            const double a = fabs(v[f]);
            finite &= a <= 1.79769313486231570815e308;
            m = fmax(m, a);
        }
        zero = m == 0.0;
        emax = (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;   // subnormal maxima: -1023
        const int shift = 62 - emax;                                      // in [-962, 1085]
        const bool big = shift > 1023;
        const double s1 = pow2(big ? shift - 64 : shift), s2 = big ? pow2(64) : 1.0;
#pragma unroll
        for (int f = 0; f < M; f++) fx[f] = (U)__double2ll_rn(__dmul_rn(__dmul_rn(v[f], s1), s2));
    }
}

// exp_restore (zfp.py:153-157): ldexp(float64(fixed), e_max-(q-2)), then the F32 cast -- one
// rounding of the exact value.  F32 with every nonzero result normal (sc >= -126): int->fp32
// rounding followed by an exact power-of-two scale is that same single rounding; otherwise the
// float64 product is exact (sc >= -157) and the cast rounds once.  F64: one multiply is correctly
// rounded for sc >= -1022; below, x * 2^(sc+64) is exact and the * 2^-64 rounds once.
template <class T, int M>
__device__ __forceinline__ void restore_block(const typename ZSpec<T>::U (&fx)[M], int sc, T (&r)[M]) {
    using S = typename ZSpec<T>::S;
    if constexpr (sizeof(T) == 4) {
        if (sc >= -126) {
            const float s = pow2f(sc);
#pragma unroll
            for (int f = 0; f < M; f++) r[f] = __fmul_rn(__int2float_rn((S)fx[f]), s);
        } else {
            const double s = pow2(sc);
#pragma unroll
            for (int f = 0; f < M; f++) r[f] = __double2float_rn(__dmul_rn((double)(S)fx[f], s));
        }
    } else {
        const bool low = sc < -1022;
        const double s1 = pow2(low ? sc + 64 : sc), s2 = low ? pow2(-64) : 1.0;
#pragma unroll
        for (int f = 0; f < M; f++) r[f] = __dmul_rn(__dmul_rn(__ll2double_rn((S)fx[f]), s1), s2);
    }
}

struct ZGrid {
    int64_t n[3];   // extents padded to rank 3 with leading 1s
    int64_t g[3];   // blocks per axis
};

// A block's element offsets: origin + row[r] + col, edge-replicated (np.pad mode="edge",
// zfp.py:98-100).  O is int32_t when 3*(n1*n2 + n2) fits, else int64_t.
template <int D, class O>
struct BlockAt {
    int64_t origin;
    O row[16];     // D=3: row[a*4+c] for in-block (i0=a, i1=c); D=2: row[a*4] for i1=a
    int col[4];    // clamped axis-2 offsets
    uint32_t rvalid;   // bit r: row r lies inside the field (not padding)
};

template <int D, class O>
__device__ __forceinline__ void block_at(const ZGrid &G, int64_t b, BlockAt<D, O> &B) {
    const int64_t b2 = b % G.g[2], r = b / G.g[2];
    const int64_t b1 = r % G.g[1], b0 = r / G.g[1];
    const int64_t x0 = b0 * 4, x1 = b1 * 4, x2 = b2 * 4;
    B.origin = (x0 * G.n[1] + x1) * G.n[2] + x2;
#pragma unroll
    for (int i = 0; i < 4; i++) B.col[i] = (int)(min64(x2 + i, G.n[2] - 1) - x2);
    B.rvalid = 0;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int64_t da = D == 3 ? min64(x0 + a, G.n[0] - 1) - x0 : 0;
            const int64_t dc = D == 3 ? min64(x1 + c, G.n[1] - 1) - x1 : D == 2 ? min64(x1 + a, G.n[1] - 1) - x1 : 0;
            B.row[a * 4 + c] = (O)((da * G.n[1] + dc) * G.n[2]);
            const bool ok = D == 3 ? (x0 + a < G.n[0] && x1 + c < G.n[1]) : D == 2 ? x1 + a < G.n[1] : a == 0;
            B.rvalid |= (ok ? 1u : 0u) << (a * 4 + c);
        }
}

template <int D>
__device__ __forceinline__ constexpr int row_of(int f) {   // f = flat in-block position
    return D == 3 ? (f >> 4) * 4 + ((f >> 2) & 3) : D == 2 ? (f >> 2) * 4 : 0;
}

// zfp_compress per block (zfp.py:291-303): exp_align :125-150, forward_transform :194-196,
// bitplane_encode :217-241.  Stream words go to out32 (MSB-first bits, byte-swapped on store so
// memory holds the np.packbits byte order).
template <class T, int D, class O>
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
    for (uint32_t i = threadIdx.x; i < (words + 3) / 4; i += kZThreads) reinterpret_cast<uint4 *>(zs)[i] = uint4{0, 0, 0, 0};
    __syncthreads();
    if ((int)threadIdx.x < nblk) {
        BlockAt<D, O> B;
        block_at<D, O>(G, cta0 + threadIdx.x, B);
        const T *p = in + B.origin;
        T v[M];   // np.asarray(blocks, float64): widening is exact, see align_block
        // in-range columns are loaded; padded ones repeat the last in-range column (edge mode)
        const int c2 = B.col[3];   // last in-range column of this block (0..3)
#pragma unroll
        for (int f = 0; f < M; f++) {
            const int i = f & 3;
            if (i == 0 || i <= c2) v[f] = __ldg(p + B.row[row_of<D>(f)] + i);
            else v[f] = v[f - 1];
        }
        U fx[M];
        int emax;
        bool zero, finite;
        align_block<T, M>(v, fx, emax, zero, finite);
        if (!finite) atomicOr(bad, 1u);
        transform<D, U, S, true>(fx);
        U c[M];
        gather_perm<D, U>(fx, c, std::make_integer_sequence<int, M>{});
        // zfp.py:204-208 negabinary (c + nb) ^ nb; a zero block is all zeros already (fixed = 0).
        // For D = 3 the ^ nb is applied to the plane words instead: nb's bit (q-1-t) is set for
        // even t, so even planes are complemented.
#pragma unroll
        for (int k = 0; k < M; k++) c[k] = D == 3 ? (U)(c[k] + Z::nb) : (U)((c[k] + Z::nb) ^ Z::nb);
        const uint32_t pos0 = (uint32_t)threadIdx.x * w;
        if constexpr (D == 3) {
            // planes MSB first: transpose the 64 coefficients' top halves into 32 plane pairs, then
            // emit whole words at the thread's fixed bit phase (funnel shifts).  The header and the
            // first word can share a word with the previous block (atomicOr); the last partial word
            // with the next one; every word between belongs to this thread alone (plain stores).
            const uint32_t head = ((zero ? 1u : 0u) << Z::ebits) | (zero ? 0u : (uint32_t)(emax + Z::bias));
            const uint32_t p1 = pos0 + 1 + Z::ebits;      // first plane bit
            const uint32_t ph = p1 & 31;                  // bit phase of every plane word
            uint32_t wi = p1 >> 5;
            // prev: this block's bits of word wi that precede p1 (the header's tail), in place
            uint32_t prev;
            {
                const uint32_t hb = 1 + Z::ebits, end = (pos0 & 31) + hb;
                if (end < 32) {
                    prev = head << (32 - end);                               // header inside word wi
                } else {
                    atomicOr(&zs[pos0 >> 5], head >> (end - 32));            // completes the word before
                    prev = end == 32 ? 0u : head << (64 - end);
                }
            }
            auto word_of = [&](uint32_t x) {
                const uint32_t word = ph ? (prev | (x >> ph)) : x;
                prev = ph ? x << (32 - ph) : 0u;
                return word;
            };
            uint32_t hi[64];
#pragma unroll
            for (int k = 0; k < 64; k++) hi[k] = (uint32_t)(c[k] >> (Z::q - 32));
            transpose32<0>(hi, rate);
            transpose32<32>(hi, rate);
            atomicOr(&zs[wi++], word_of(~hi[0]));   // may hold the previous block's tail (rate >= 1)
            zs[wi++] = word_of(~hi[32]);
#pragma unroll
            for (int t = 1; t < 32; t++)
                if (t < rate) {
                    zs[wi++] = word_of(t % 2 ? hi[t] : ~hi[t]);
                    zs[wi++] = word_of(t % 2 ? hi[32 + t] : ~hi[32 + t]);
                }
            if constexpr (Z::q == 64) {
                if (rate > 32) {
                    uint32_t lo[64];
#pragma unroll
                    for (int k = 0; k < 64; k++) lo[k] = (uint32_t)c[k];
                    transpose32<0>(lo, rate - 32);
                    transpose32<32>(lo, rate - 32);
#pragma unroll
                    for (int t = 0; t < 32; t++)
                        if (32 + t < rate) {
                            zs[wi++] = word_of(t % 2 ? lo[t] : ~lo[t]);
                            zs[wi++] = word_of(t % 2 ? lo[32 + t] : ~lo[32 + t]);
                        }
                }
            }
            if (ph) atomicOr(&zs[wi], prev);   // trailing partial word, shared with the next block
        } else {
            BitWriter bw(zs, pos0);
            bw.put(zero ? 1u : 0u, 1);
            bw.put(zero ? 0u : (uint32_t)(emax + Z::bias), Z::ebits);
            for (int t = 0; t < rate; t++) {
                const int sh = Z::q - 1 - t;
                uint32_t pl = 0;
#pragma unroll
                for (int k = 0; k < M; k++) pl |= (uint32_t)((c[k] >> sh) & 1) << (M - 1 - k);
                bw.put(pl, M);
            }
            bw.flush();
        }
    }
    __syncthreads();
    // 128 blocks = 4*w words, so every CTA's slice of the stream starts 16-byte aligned
    uint32_t *dst = out32 + (uint64_t)(cta0 - b_lo) * w / 32;
    for (uint32_t i = threadIdx.x; i < words / 4; i += kZThreads) {
        const uint4 x = reinterpret_cast<const uint4 *>(zs)[i];
        reinterpret_cast<uint4 *>(dst)[i] = uint4{__byte_perm(x.x, 0, 0x0123), __byte_perm(x.y, 0, 0x0123),
                                                  __byte_perm(x.z, 0, 0x0123), __byte_perm(x.w, 0, 0x0123)};
    }
    for (uint32_t i = words / 4 * 4 + threadIdx.x; i < words; i += kZThreads) dst[i] = __byte_perm(zs[i], 0, 0x0123);
}

// zfp_decompress per block (zfp.py:338-347): bitplane_decode :244-264, inverse_transform,
// exp_restore :153-157, zero blocks -> 0.0, padding discarded.
template <class T, int D, class O>
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
    for (uint32_t i = threadIdx.x; i < words / 4; i += kZThreads) {
        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(src) + i);
        reinterpret_cast<uint4 *>(zs)[i] = uint4{__byte_perm(x.x, 0, 0x0123), __byte_perm(x.y, 0, 0x0123),
                                                 __byte_perm(x.z, 0, 0x0123), __byte_perm(x.w, 0, 0x0123)};
    }
    for (uint32_t i = words / 4 * 4 + threadIdx.x; i <= words; i += kZThreads)
        zs[i] = i < words ? __byte_perm(__ldg(src + i), 0, 0x0123) : 0u;
    __syncthreads();
    if ((int)threadIdx.x >= nblk) return;
    BitReader br{zs, (uint32_t)threadIdx.x * w};
    const bool zero = br.get(1) != 0;
    const int biased = (int)br.get(Z::ebits);
    const int emax = zero ? -Z::bias : biased - Z::bias;
    const int reff = zero ? 0 : rate;   // a zero block's planes are ignored (zfp.py:263, :346)
    U c[M];
    if constexpr (D == 3) {
        // 32-bit plane halves at a fixed bit phase: one shared load + funnel shift each
        uint32_t wi = br.pos >> 5;
        const uint32_t o = br.pos & 31;
        uint32_t cur = zs[wi];
        auto next32 = [&]() {
            const uint32_t nxt = zs[++wi];
            const uint32_t r = __funnelshift_l(nxt, cur, o);
            cur = nxt;
            return r;
        };
        uint32_t hi[64];
#pragma unroll
        for (int t = 0; t < 32; t++) {
            hi[t] = t < reff ? next32() : 0u;
            hi[32 + t] = t < reff ? next32() : 0u;
        }
        transpose32<0>(hi);
        transpose32<32>(hi);
        if constexpr (Z::q == 64) {
            uint32_t lo[64];
#pragma unroll
            for (int t = 0; t < 32; t++) {
                lo[t] = 32 + t < reff ? next32() : 0u;
                lo[32 + t] = 32 + t < reff ? next32() : 0u;
            }
            if (reff > 32) {
                transpose32<0>(lo);
                transpose32<32>(lo);
            }
#pragma unroll
            for (int k = 0; k < 64; k++) c[k] = ((U)hi[k] << 32) | lo[k];
        } else {
#pragma unroll
            for (int k = 0; k < 64; k++) c[k] = hi[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < M; k++) c[k] = 0;
        for (int t = 0; t < reff; t++) {
            const int sh = Z::q - 1 - t;
            const uint32_t pl = br.get(M);
#pragma unroll
            for (int k = 0; k < M; k++) c[k] |= (U)((pl >> (M - 1 - k)) & 1) << sh;
        }
    }
#pragma unroll
    for (int k = 0; k < M; k++) c[k] = (U)((c[k] ^ Z::nb) - Z::nb);   // zfp.py:211-214
    U fx[M];
    scatter_perm<D, U>(c, fx, std::make_integer_sequence<int, M>{});
    transform<D, U, S, false>(fx);
    BlockAt<D, O> B;
    block_at<D, O>(G, cta0 + threadIdx.x, B);
    T *q = out + B.origin;
    T r[M];
    restore_block<T, M>(fx, emax - (Z::q - 2), r);
    const int c2 = B.col[3];
#pragma unroll
    for (int f = 0; f < M; f++)   // padding positions are discarded (unpartition_blocks :122)
        if (((B.rvalid >> row_of<D>(f)) & 1) && (f & 3) <= c2) q[B.row[row_of<D>(f)] + (f & 3)] = r[f];
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

// int32 in-block offsets unless a block spans more than 2^31 elements
// (HPDR_ZFP_WIDE=1 forces the int64 variant, for its parity test)
bool zfp_wide(const ZfpShape &z) {
    static const bool force = getenv("HPDR_ZFP_WIDE") != nullptr;
    return force || 3 * (z.G.n[1] * z.G.n[2] + z.G.n[2]) + 3 >= (1LL << 31);
}

template <class T, int D, class O>
void launch_encode(const ZfpShape &z, const void *in, int64_t lo, int64_t hi, uint32_t *out32, unsigned *bad,
                   cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_zfp_encode<T, D, O>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
    }
    const unsigned grid = (unsigned)((hi - lo + kZThreads - 1) / kZThreads);
    KPROF("k_zfp_encode", (double)(hi - lo) * ((double)(1 << (2 * D)) * sizeof(T) + z.w / 8.0), s);
    k_zfp_encode<T, D, O><<<grid, kZThreads, zfp_smem(z), s>>>((const T *)in, z.G, lo, hi, z.rate, out32, bad);
    LAUNCH_CHECK();
}

template <class T, int D, class O>
void launch_decode(const ZfpShape &z, const uint32_t *in32, int64_t lo, int64_t hi, void *out, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_zfp_decode<T, D, O>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
    }
    const unsigned grid = (unsigned)((hi - lo + kZThreads - 1) / kZThreads);
    KPROF("k_zfp_decode", (double)(hi - lo) * ((double)(1 << (2 * D)) * sizeof(T) + z.w / 8.0), s);
    k_zfp_decode<T, D, O><<<grid, kZThreads, zfp_smem(z) + 4, s>>>(in32, z.G, lo, hi, z.rate, (T *)out);
    LAUNCH_CHECK();
}

template <class T, class O>
void encode_t(const ZfpShape &z, const void *in, int64_t lo, int64_t hi, uint32_t *out32, unsigned *bad,
              cudaStream_t s) {
    if (z.rank == 1) launch_encode<T, 1, O>(z, in, lo, hi, out32, bad, s);
    else if (z.rank == 2) launch_encode<T, 2, O>(z, in, lo, hi, out32, bad, s);
    else launch_encode<T, 3, O>(z, in, lo, hi, out32, bad, s);
}

template <class T, class O>
void decode_t(const ZfpShape &z, const uint32_t *in32, int64_t lo, int64_t hi, void *out, cudaStream_t s) {
    if (z.rank == 1) launch_decode<T, 1, O>(z, in32, lo, hi, out, s);
    else if (z.rank == 2) launch_decode<T, 2, O>(z, in32, lo, hi, out, s);
    else launch_decode<T, 3, O>(z, in32, lo, hi, out, s);
}

void encode_range(const ZfpShape &z, const void *in, int64_t lo, int64_t hi, uint32_t *out32, unsigned *bad,
                  cudaStream_t s) {
    if (hi <= lo) return;
    const bool wide = zfp_wide(z);
    if (z.dtype == 0) wide ? encode_t<float, int64_t>(z, in, lo, hi, out32, bad, s) : encode_t<float, int32_t>(z, in, lo, hi, out32, bad, s);
    else wide ? encode_t<double, int64_t>(z, in, lo, hi, out32, bad, s) : encode_t<double, int32_t>(z, in, lo, hi, out32, bad, s);
}

void decode_range(const ZfpShape &z, const uint32_t *in32, int64_t lo, int64_t hi, void *out, cudaStream_t s) {
    if (hi <= lo) return;
    const bool wide = zfp_wide(z);
    if (z.dtype == 0) wide ? decode_t<float, int64_t>(z, in32, lo, hi, out, s) : decode_t<float, int32_t>(z, in32, lo, hi, out, s);
    else wide ? decode_t<double, int64_t>(z, in32, lo, hi, out, s) : decode_t<double, int32_t>(z, in32, lo, hi, out, s);
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
    if (!d) throw Error{HPDR_ERR_VALIDATION, "null stream pointer", -1};
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


// ---- HPDR container with fixed-rate chunks (pipeline id 1, params: rate u8) ----
uint32_t zcrc32(const uint8_t *p, size_t n) {   // zlib polynomial (container.py uses zlib.crc32)
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; i++) {
        c ^= p[i];
        for (int k = 0; k < 8; k++) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return c ^ 0xFFFFFFFFu;
}

struct ZChunk {
    uint64_t raw_off, raw_size, pay_off, pay_size;
};

template <class X>
void zput(std::vector<uint8_t> &v, X x) {
    const size_t o = v.size();
    v.resize(o + sizeof(X));
    memcpy(v.data() + o, &x, sizeof(X));
}

std::vector<uint8_t> zfp_container_header(int dtype, int rank, const uint64_t *dims, int rate,
                                          const std::vector<ZChunk> &ch) {
    std::vector<uint8_t> h = {'H', 'P', 'D', 'R'};
    zput<uint16_t>(h, 1);
    zput<uint8_t>(h, 1);   // ZFP
    zput<uint8_t>(h, (uint8_t)dtype);
    zput<uint8_t>(h, (uint8_t)rank);
    for (int d = 0; d < rank; d++) zput<uint64_t>(h, dims[d]);
    zput<uint8_t>(h, (uint8_t)rate);
    zput<uint32_t>(h, (uint32_t)ch.size());
    for (const ZChunk &c : ch) {
        zput<uint64_t>(h, c.raw_off);
        zput<uint64_t>(h, c.raw_size);
        zput<uint64_t>(h, c.pay_off);
        zput<uint64_t>(h, c.pay_size);
    }
    zput<uint32_t>(h, zcrc32(h.data(), h.size()));
    return h;
}

// Per-chunk copy/compute timestamps (ms from the first event): H2D start/end, compute start/end,
// D2H start/end -- the trace layout of hpdr_pipeline_compress.
struct ZTimer {
    std::vector<cudaEvent_t> ev;
    cudaEvent_t t0 = nullptr;
    explicit ZTimer(size_t n) {
        CUDA_CHECK(cudaEventCreate(&t0));
        ev.resize(n);
        for (auto &e : ev) CUDA_CHECK(cudaEventCreate(&e));
    }
    ~ZTimer() {
        if (t0) cudaEventDestroy(t0);
        for (auto e : ev) cudaEventDestroy(e);
    }
};

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
        if (!ctx || !dims || !out_len) throw Error{HPDR_ERR_VALIDATION, "null argument", -1};
        ZfpShape z;
        zfp_shape(dtype, rank, dims, (int)std::min<uint32_t>(rate, 1u << 20), z);
        *out_len = z.total;
        if (!out || out_cap < z.total)
            throw Error{HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(z.total), -1};
        if (!in) throw Error{HPDR_ERR_VALIDATION, "null input pointer", -1};
        CUDA_CHECK(cudaSetDevice(ctx->device));
        const int isz = dtype == 0 ? 4 : 8;
        const uint64_t n = (uint64_t)z.G.n[0] * z.G.n[1] * z.G.n[2];
        const uint64_t plane_bytes = (uint64_t)z.G.n[1] * z.G.n[2] * isz;
        const MemKind ik = classify(in);
        const bool in_dev = ik == MemKind::Device, in_pageable = ik == MemKind::Host;
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
        zero_async(bad, 4, s);
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
                    if (in_pageable)   // staged while the previous slab is coded
                        stage_h2d(ctx, (uint8_t *)din + in_done * plane_bytes, (const uint8_t *)in + in_done * plane_bytes,
                                  (need - in_done) * plane_bytes, ctx->h2d);
                    else
                        CUDA_CHECK(cudaMemcpyAsync((uint8_t *)din + in_done * plane_bytes,
                                                   (const uint8_t *)in + in_done * plane_bytes,
                                                   (need - in_done) * plane_bytes, cudaMemcpyHostToDevice, ctx->h2d));
                    in_done = need;
                }
                CUDA_CHECK(cudaEventRecord(ctx->event(EvZfpIn, k), ctx->h2d));
                CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(EvZfpIn, k), 0));
            }
            encode_range(z, din, lo, hi, pay + (uint64_t)lo * z.w / 32, bad, s);
            // stream bytes [lo*w/8, hi*w/8) are final (lo, hi multiples of 32 blocks, or the end)
            const uint64_t a = (uint64_t)lo * z.w / 8;
            const uint64_t e = k == K - 1 ? z.payload : (uint64_t)hi * z.w / 8;
            CUDA_CHECK(cudaEventRecord(ctx->event(EvZfpOut, k), s));
            CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(EvZfpOut, k), 0));
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
        if (stage) parallel_memcpy(o + hl, stage, z.payload);
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
        zero_async((uint8_t *)pay + z.payload, 8, s);   // the staged tail word past the payload reads zeros
        void *dout = out_dev ? out : ctx->dbuf("zfp_out", n * isz);
        const std::vector<int64_t> cut = zfp_slabs(z, (in_dev && out_dev) ? 1 : zfp_slab_count(z, n * isz));
        const int K = (int)cut.size() - 1;
        uint64_t rows_out = 0;   // output planes copied out
        uint64_t pay_in = 0;     // payload bytes resident
        const bool in_pageable = !in_dev && classify(stream) == MemKind::Host;
        const bool out_pageable = ok == MemKind::Host;
        std::vector<std::array<uint64_t, 3>> outs;
        for (int k = 0; k < K; k++) {
            const int64_t lo = cut[k], hi = cut[k + 1];
            const uint64_t need = k == K - 1 ? z.payload : ((uint64_t)hi * z.w + 7) / 8;
            if (need > pay_in) {
                if (in_pageable)
                    stage_h2d(ctx, (uint8_t *)pay + pay_in, (const uint8_t *)stream + hl + pay_in, need - pay_in, ctx->h2d);
                else
                    CUDA_CHECK(cudaMemcpyAsync((uint8_t *)pay + pay_in, (const uint8_t *)stream + hl + pay_in,
                                               need - pay_in, in_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                               ctx->h2d));
                pay_in = need;
            }
            CUDA_CHECK(cudaEventRecord(ctx->event(EvZfpDecIn, k), ctx->h2d));
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(EvZfpDecIn, k), 0));
            decode_range(z, pay + (uint64_t)lo * z.w / 32, lo, hi, dout, s);
            if (out_dev) continue;
            // output planes whose block rows are complete
            const uint64_t rows = k == K - 1 ? (uint64_t)z.G.n[0]
                                             : std::min<uint64_t>((uint64_t)z.G.n[0], (uint64_t)(hi / z.blocks_per_plane) * 4);
            if (rows > rows_out) {
                CUDA_CHECK(cudaEventRecord(ctx->event(EvZfpDecOut, k), s));
                if (out_pageable) {
                    outs.push_back({rows_out, rows, (uint64_t)k});   // copied out below, after every slab is queued
                } else {
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(EvZfpDecOut, k), 0));
                    CUDA_CHECK(cudaMemcpyAsync((uint8_t *)out + rows_out * plane_elems * isz,
                                               (uint8_t *)dout + rows_out * plane_elems * isz,
                                               (rows - rows_out) * plane_elems * isz, cudaMemcpyDeviceToHost, ctx->d2h));
                }
                rows_out = rows;
            }
        }
        for (const auto &r : outs) {   // pageable output: pinned staging ring, host-blocking
            CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(EvZfpDecOut, (size_t)r[2]), 0));
            stage_d2h(ctx, (uint8_t *)out + r[0] * plane_elems * isz, (uint8_t *)dout + r[0] * plane_elems * isz,
                      (r[1] - r[0]) * plane_elems * isz, ctx->d2h);
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
    });
}


// Streams pipeline with fixed-rate chunks (the reducer slot of run_pipeline):
// dim-0 slabs, each an independent zfp_compress(slab, rate) stream, in an HPDR container with
// pipeline id 1.  Stream sizes are a function of the slab shape, so the whole container layout is
// known before any work starts: chunk k's H2D, encode and D2H are issued without host syncs, with
// two input and two output device buffers (Fig. 7 reuse edges as events: the H2D of chunk k+2
// waits for chunk k's encode, the encode of chunk k+2 for chunk k's D2H).
int hpdr_pipeline_zfp_compress(hpdr_ctx *ctx, const void *host_in, int dtype, int rank, const uint64_t *dims,
                               uint32_t rate, uint64_t chunk_planes, const uint64_t *chunk_list, uint64_t n_list,
                               void *out, uint64_t out_cap, uint64_t *out_len, double *trace) {
    return zguard([&] {
        ZfpShape whole;
        zfp_shape(dtype, rank, dims, (int)std::min<uint32_t>(rate, 1u << 20), whole);
        CUDA_CHECK(cudaSetDevice(ctx->device));
        const int isz = dtype == 0 ? 4 : 8;
        uint64_t plane = 1;   // elements per dim-0 index (the chunking axis is the caller's dims[0])
        for (int d = 1; d < rank; d++) plane *= dims[d];
        const uint64_t n0 = dims[0];
        std::vector<uint64_t> planes;
        if (chunk_list && n_list) {
            uint64_t sum = 0;
            for (uint64_t i = 0; i < n_list; i++) {
                if (!chunk_list[i]) throw Error{HPDR_ERR_VALIDATION, "chunk of 0 planes", -1};
                planes.push_back(chunk_list[i]);
                sum += chunk_list[i];
            }
            if (sum != n0) throw Error{HPDR_ERR_VALIDATION, "chunk plane counts do not sum to dims[0]", -1};
        } else {
            // default ~64 MB of input per chunk, whole 4-plane block rows
            uint64_t cp = chunk_planes ? chunk_planes : std::max<uint64_t>(4, ((64ull << 20) / (plane * isz)) / 4 * 4);
            for (uint64_t a = 0; a < n0; a += cp) planes.push_back(std::min(cp, n0 - a));
        }
        const size_t K = planes.size();
        std::vector<ZChunk> ch(K);
        std::vector<ZfpShape> zs(K);
        uint64_t off = 0, raw = 0, max_in = 0, max_pay = 0;
        for (size_t k = 0; k < K; k++) {
            uint64_t cd[3] = {planes[k], rank > 1 ? dims[1] : 0, rank > 2 ? dims[2] : 0};
            zfp_shape(dtype, rank, cd, whole.rate, zs[k]);
            ch[k] = ZChunk{raw, planes[k] * plane, off, zs[k].total};
            raw += planes[k] * plane;
            off += zs[k].total;
            max_in = std::max(max_in, planes[k] * plane * isz);
            max_pay = std::max(max_pay, zs[k].payload);
        }
        const std::vector<uint8_t> head = zfp_container_header(dtype, rank, dims, whole.rate, ch);
        *out_len = head.size() + off;
        if (!out || out_cap < *out_len)
            throw Error{HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(*out_len), -1};
        const bool out_dev = classify(out) == MemKind::Device;
        const bool in_dev = classify(host_in) == MemKind::Device;
        uint8_t *o = (uint8_t *)out;
        cudaStream_t s = ctx->stream;
        // container header and the per-chunk stream headers (zfp.py:306-308) are host bytes
        std::vector<uint8_t> hdrs(head);
        for (size_t k = 0; k < K; k++) {
            uint8_t zh[kZHeader + 24];
            zh[0] = (uint8_t)rank;
            zh[1] = (uint8_t)dtype;
            zh[2] = (uint8_t)whole.rate;
            memcpy(zh + kZHeader, zs[k].dims, 8ull * rank);
            const uint64_t at = head.size() + ch[k].pay_off;
            if (out_dev) CUDA_CHECK(cudaMemcpyAsync(o + at, zh, kZHeader + 8ull * rank, cudaMemcpyHostToDevice, s));
            else memcpy(o + at, zh, kZHeader + 8ull * rank);
        }
        if (out_dev) CUDA_CHECK(cudaMemcpyAsync(o, head.data(), head.size(), cudaMemcpyHostToDevice, s));
        else memcpy(o, head.data(), head.size());
        unsigned *bad = (unsigned *)ctx->dbuf("zfp_bad", 16);
        unsigned *bad_h = (unsigned *)ctx->hbuf("zfp_bad_h", 16);
        zero_async(bad, 4, s);
        void *din[2] = {in_dev ? nullptr : ctx->dbuf("zfp_pin0", max_in), in_dev ? nullptr : ctx->dbuf("zfp_pin1", max_in)};
        uint32_t *dp[2] = {(uint32_t *)ctx->dbuf("zfp_ppay0", max_pay + 8), (uint32_t *)ctx->dbuf("zfp_ppay1", max_pay + 8)};
        std::unique_ptr<ZTimer> tm(trace ? new ZTimer(6 * K) : nullptr);
        CUDA_CHECK(cudaEventRecord(ctx->event(480), s));   // everything after the setup above
        CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(480), 0));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(480), 0));
        if (tm) CUDA_CHECK(cudaEventRecord(tm->t0, s));
        for (size_t k = 0; k < K; k++) {
            const int b = (int)(k & 1);
            const void *src;
            if (in_dev) {
                src = (const uint8_t *)host_in + ch[k].raw_off * isz;
            } else {
                if (k >= 2) CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(482 + b), 0));   // encode k-2 read din[b]
                if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k], ctx->h2d));
                CUDA_CHECK(cudaMemcpyAsync(din[b], (const uint8_t *)host_in + ch[k].raw_off * isz, ch[k].raw_size * isz,
                                           cudaMemcpyHostToDevice, ctx->h2d));
                if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 1], ctx->h2d));
                CUDA_CHECK(cudaEventRecord(ctx->event(486 + b), ctx->h2d));
                CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(486 + b), 0));
                src = din[b];
            }
            if (k >= 2) CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(484 + b), 0));   // D2H k-2 read dp[b]
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 2], s));
            encode_range(zs[k], src, 0, zs[k].nblk, dp[b], bad, s);
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 3], s));
            CUDA_CHECK(cudaEventRecord(ctx->event(482 + b), s));
            CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(482 + b), 0));
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 4], ctx->d2h));
            CUDA_CHECK(cudaMemcpyAsync(o + head.size() + ch[k].pay_off + kZHeader + 8ull * rank, dp[b], zs[k].payload,
                                       out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->d2h));
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 5], ctx->d2h));
            CUDA_CHECK(cudaEventRecord(ctx->event(484 + b), ctx->d2h));
        }
        CUDA_CHECK(cudaMemcpyAsync(bad_h, bad, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
        CUDA_CHECK(cudaStreamSynchronize(ctx->h2d));
        if (*bad_h) throw Error{HPDR_ERR_VALIDATION, "non-finite values cannot be aligned", -1};
        if (tm)
            for (size_t i = 0; i < 6 * K; i++) {
                float ms = 0.f;
                if (in_dev && (i % 6) < 2) {   // no H2D: report the compute start
                    CUDA_CHECK(cudaEventElapsedTime(&ms, tm->t0, tm->ev[6 * (i / 6) + 2]));
                } else {
                    CUDA_CHECK(cudaEventElapsedTime(&ms, tm->t0, tm->ev[i]));
                }
                trace[i] = ms;
            }
    });
}

}  // extern "C"

namespace hpdr {

// Container decompress for pipeline id 1 (called by hpdr_pipeline_decompress after the common
// magic / version checks).  Mirrors the compress runner: chunk k's stream H2D, decode into a slab
// buffer (or straight into a device output), D2H of the slab, two buffer sets.
int zfp_container_decompress(hpdr_ctx *ctx, const uint8_t *c, uint64_t len, void *out, uint64_t out_bytes,
                             double *trace) {
    return zguard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        auto need = [&](uint64_t p, uint64_t n) {
            if (p > len || n > len - p) throw Error{HPDR_ERR_FORMAT, "container truncated", -1};
        };
        need(0, 9);
        const int dtype = c[7], rank = c[8];
        if (rank < 1 || rank > 3) throw Error{HPDR_ERR_FORMAT, "bad rank for a fixed-rate container", -1};
        if (dtype != 0 && dtype != 1) throw Error{HPDR_ERR_FORMAT, "fixed-rate container needs F32/F64", -1};
        uint64_t pos = 9;
        need(pos, 8ull * rank + 1 + 4);
        uint64_t dims[3] = {1, 1, 1};
        memcpy(dims, c + pos, 8ull * rank);
        pos += 8ull * rank;
        const int rate = c[pos++];
        uint32_t K;
        memcpy(&K, c + pos, 4);
        pos += 4;
        need(pos, 32ull * K + 4);
        std::vector<ZChunk> ch(K);
        memcpy(ch.data(), c + pos, 32ull * K);
        pos += 32ull * K;
        uint32_t crc;
        memcpy(&crc, c + pos, 4);
        if (zcrc32(c, pos) != crc) throw Error{HPDR_ERR_FORMAT, "header checksum mismatch", -1};
        pos += 4;
        const uint64_t base = pos;
        ZfpShape whole;
        zfp_shape(dtype, rank, dims, rate, whole);
        const int isz = dtype == 0 ? 4 : 8;
        uint64_t plane = 1;
        for (int d = 1; d < rank; d++) plane *= dims[d];
        const uint64_t N = dims[0] * plane;
        if (out_bytes < N * isz) throw Error{HPDR_ERR_BUFFER, "output buffer too small", -1};
        std::vector<ZfpShape> zs(K);
        uint64_t max_pay = 1, max_raw = 1;
        for (uint32_t k = 0; k < K; k++) {
            need(base + ch[k].pay_off, ch[k].pay_size);
            if (ch[k].raw_off + ch[k].raw_size > N || ch[k].raw_off % plane || ch[k].raw_size % plane)
                throw Error{HPDR_ERR_FORMAT, "chunk outside the field or not whole planes", -1};
            zfp_parse(c + base + ch[k].pay_off, ch[k].pay_size, zs[k]);   // zfp_decompress's checks per chunk
            if (zs[k].dtype != dtype || zs[k].rank != rank || zs[k].rate != rate || zs[k].dims[0] * plane != ch[k].raw_size ||
                (rank > 1 && zs[k].dims[1] != dims[1]) || (rank > 2 && zs[k].dims[2] != dims[2]))
                throw Error{HPDR_ERR_FORMAT, "chunk stream does not match the container", -1};
            max_pay = std::max(max_pay, zs[k].payload);
            max_raw = std::max(max_raw, ch[k].raw_size);
        }
        const bool out_dev = classify(out) == MemKind::Device;
        cudaStream_t s = ctx->stream;
        uint32_t *dp[2] = {(uint32_t *)ctx->dbuf("zfp_dpay0", max_pay + 8), (uint32_t *)ctx->dbuf("zfp_dpay1", max_pay + 8)};
        void *dout[2] = {out_dev ? nullptr : ctx->dbuf("zfp_dout0", max_raw * isz),
                         out_dev ? nullptr : ctx->dbuf("zfp_dout1", max_raw * isz)};
        std::unique_ptr<ZTimer> tm(trace ? new ZTimer(6 * (size_t)K) : nullptr);
        CUDA_CHECK(cudaEventRecord(ctx->event(480), s));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(480), 0));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(480), 0));
        if (tm) CUDA_CHECK(cudaEventRecord(tm->t0, s));
        for (uint32_t k = 0; k < K; k++) {
            const int b = (int)(k & 1);
            const uint64_t hl = kZHeader + 8ull * rank;
            if (k >= 2) CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(482 + b), 0));   // decode k-2 read dp[b]
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k], ctx->h2d));
            CUDA_CHECK(cudaMemcpyAsync(dp[b], c + base + ch[k].pay_off + hl, zs[k].payload, cudaMemcpyHostToDevice,
                                       ctx->h2d));
            zero_async((uint8_t *)dp[b] + zs[k].payload, 8, ctx->h2d);   // tail word past the payload
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 1], ctx->h2d));
            CUDA_CHECK(cudaEventRecord(ctx->event(486 + b), ctx->h2d));
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(486 + b), 0));
            if (!out_dev && k >= 2) CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(484 + b), 0));   // D2H k-2 read dout[b]
            void *dst = out_dev ? (void *)((uint8_t *)out + ch[k].raw_off * isz) : dout[b];
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 2], s));
            decode_range(zs[k], dp[b], 0, zs[k].nblk, dst, s);
            if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 3], s));
            CUDA_CHECK(cudaEventRecord(ctx->event(482 + b), s));
            if (!out_dev) {
                CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(482 + b), 0));
                if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 4], ctx->d2h));
                CUDA_CHECK(cudaMemcpyAsync((uint8_t *)out + ch[k].raw_off * isz, dout[b], ch[k].raw_size * isz,
                                           cudaMemcpyDeviceToHost, ctx->d2h));
                if (tm) CUDA_CHECK(cudaEventRecord(tm->ev[6 * k + 5], ctx->d2h));
                CUDA_CHECK(cudaEventRecord(ctx->event(484 + b), ctx->d2h));
            }
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
        if (tm)
            for (size_t i = 0; i < 6 * (size_t)K; i++) {
                float ms = 0.f;
                const size_t j = (out_dev && (i % 6) >= 4) ? 6 * (i / 6) + 3 : i;   // no D2H: compute end
                CUDA_CHECK(cudaEventElapsedTime(&ms, tm->t0, tm->ev[j]));
                trace[i] = ms;
            }
    });
}

}  // namespace hpdr
