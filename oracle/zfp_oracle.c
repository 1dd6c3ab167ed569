/*
 * zfp_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never shipped).
 *
 * Scalar C restatement of the reference fixed-rate block coder
 * (/root/reference/pkg/src/hpdr/zfp.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg load it.  Pinned against blobs produced by the
 * reference itself (tests/golden/gen_zfp_golden.py -> tests/golden/zfp.npz).
 *
 * Integer arithmetic is carried in uint64_t and reduced modulo 2^q after every
 * step (q = 32 for F32, 64 for F64), which is what numpy's wrapping int32/int64
 * in-place operators do (zfp.py:186 errstate over="ignore").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mgard_oracle.h"

#define SIDE 4            /* zfp.py:30 BLOCK_SIDE */
#define MAX_RANK 3        /* zfp.py:31 */
#define HDR 3             /* zfp.py:267 "<BBB" rank, dtype code, rate */

typedef struct {
    int q, ebits, bias;
    uint64_t mask, nb;
} Spec;

/* zfp.py:47-52 */
static Spec spec_of(int dtype) {
    Spec s;
    if (dtype == ORC_F32) {
        s.q = 32; s.ebits = 8; s.bias = 127; s.mask = 0xFFFFFFFFull; s.nb = 0xAAAAAAAAull;
    } else {
        s.q = 64; s.ebits = 11; s.bias = 1023; s.mask = ~0ull; s.nb = 0xAAAAAAAAAAAAAAAAull;
    }
    return s;
}

static int64_t sx(const Spec *s, uint64_t v) { return s->q == 64 ? (int64_t)v : (int64_t)(int32_t)(uint32_t)v; }
static uint64_t asr1(const Spec *s, uint64_t v) { return (uint64_t)(sx(s, v) >> 1) & s->mask; }
static uint64_t add(const Spec *s, uint64_t a, uint64_t b) { return (a + b) & s->mask; }
static uint64_t sub(const Spec *s, uint64_t a, uint64_t b) { return (a - b) & s->mask; }

/* zfp.py:68-80: positions ordered by total per-axis frequency, ties by flat index. */
static void sequency_perm(int d, int *perm) {
    static const int freq[4] = {0, 3, 1, 2};
    int m = 1, key[64];
    for (int i = 0; i < d; i++) m *= SIDE;
    for (int f = 0; f < m; f++) {
        int k = 0, r = f;
        for (int i = 0; i < d; i++) { k += freq[r % SIDE]; r /= SIDE; }
        key[f] = k;
        perm[f] = f;
    }
    for (int i = 1; i < m; i++)  /* stable insertion sort on (key, flat) */
        for (int j = i; j > 0 && key[perm[j - 1]] > key[perm[j]]; j--) {
            int t = perm[j]; perm[j] = perm[j - 1]; perm[j - 1] = t;
        }
}

/* zfp.py:160-180 on one 4-vector (x, y, z, w) = v[0..3] at stride st. */
static void lift(const Spec *s, uint64_t *v, int st, int forward) {
    uint64_t x = v[0], y = v[st], z = v[2 * st], w = v[3 * st];
    if (forward) {
        w = sub(s, w, x); x = add(s, x, asr1(s, w));
        y = sub(s, y, z); z = add(s, z, asr1(s, y));
        z = sub(s, z, x); x = add(s, x, asr1(s, z));
        y = sub(s, y, w); w = add(s, w, asr1(s, y));
        w = add(s, w, asr1(s, y)); y = sub(s, y, asr1(s, w));
    } else {
        y = add(s, y, asr1(s, w)); w = sub(s, w, asr1(s, y));
        w = sub(s, w, asr1(s, y)); y = add(s, y, w);
        x = sub(s, x, asr1(s, z)); z = add(s, z, x);
        z = sub(s, z, asr1(s, y)); y = add(s, y, z);
        x = sub(s, x, asr1(s, w)); w = add(s, w, x);
    }
    v[0] = x; v[st] = y; v[2 * st] = z; v[3 * st] = w;
}

/* zfp.py:183-201: forward over in-block axes slowest first, inverse in reverse order. */
static void transform(const Spec *s, uint64_t *blk, int d, int forward) {
    int m = 1;
    for (int i = 0; i < d; i++) m *= SIDE;
    for (int t = 0; t < d; t++) {
        const int ax = forward ? t : d - 1 - t;      /* 0 = slowest in-block axis */
        int st = 1;
        for (int i = ax + 1; i < d; i++) st *= SIDE;
        for (int f = 0; f < m; f++)
            if ((f / st) % SIDE == 0) lift(s, blk + f, st, forward);
    }
}

static uint64_t block_bits(const Spec *s, int d, int rate) {   /* zfp.py:64-65 */
    uint64_t m = 1;
    for (int i = 0; i < d; i++) m *= SIDE;
    return 1 + (uint64_t)s->ebits + (uint64_t)rate * m;
}

int orz_compressed_size(int dtype, int rank, const uint64_t *dims, int rate, uint64_t *size) {
    if (dtype != ORC_F32 && dtype != ORC_F64) return ORC_VALIDATION;
    const Spec s = spec_of(dtype);
    if (rate < 1 || rate > s.q || rank < 1 || rank > MAX_RANK) return ORC_VALIDATION;
    uint64_t nb = 1;
    for (int i = 0; i < rank; i++) nb *= (dims[i] + SIDE - 1) / SIDE;
    *size = HDR + 8ull * rank + (nb * block_bits(&s, rank, rate) + 7) / 8;   /* zfp.py:270-278 */
    return ORC_OK;
}

static void put_bit(uint8_t *p, uint64_t pos, int b) {
    if (b) p[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
}
static int get_bit(const uint8_t *p, uint64_t pos) { return (p[pos >> 3] >> (7 - (pos & 7))) & 1; }

/* zfp.py:281-308 (partition_blocks :87-109, exp_align :125-150, forward_transform,
 * bitplane_encode :217-241, np.packbits MSB first). */
int orz_compress(const void *in, int dtype, int rank, const uint64_t *dims, int rate, uint8_t *out, uint64_t cap,
                 uint64_t *len) {
    uint64_t total;
    int rc = orz_compressed_size(dtype, rank, dims, rate, &total);
    if (rc) return rc;
    *len = total;
    if (cap < total) return ORC_ALLOC;
    const Spec s = spec_of(dtype);
    const int d = rank, m = d == 1 ? 4 : d == 2 ? 16 : 64;
    uint64_t n[3] = {1, 1, 1}, g[3] = {1, 1, 1};
    for (int i = 0; i < d; i++) { n[3 - d + i] = dims[i]; g[3 - d + i] = (dims[i] + 3) / 4; }
    const uint64_t nblk = g[0] * g[1] * g[2], w = block_bits(&s, d, rate);
    int perm[64];
    sequency_perm(d, perm);
    memset(out, 0, total);
    out[0] = (uint8_t)d; out[1] = (uint8_t)dtype; out[2] = (uint8_t)rate;
    memcpy(out + HDR, dims, 8ull * d);
    uint8_t *pay = out + HDR + 8 * d;
    const float *f32 = (const float *)in;
    const double *f64 = (const double *)in;
    int bad = 0;
    /* groups of 8 blocks are byte-aligned (zfp.py:32-34), so they can be written in parallel */
#pragma omp parallel for schedule(static) reduction(| : bad) num_threads(orc_get_threads())
    for (int64_t grp = 0; grp < (int64_t)((nblk + 7) / 8); grp++) {
        for (uint64_t b = (uint64_t)grp * 8; b < nblk && b < (uint64_t)grp * 8 + 8; b++) {
            const uint64_t b2 = b % g[2], b1 = (b / g[2]) % g[1], b0 = b / (g[2] * g[1]);
            double v[64];
            double maxabs = 0.0;
            for (int f = 0; f < m; f++) {
                /* in-block position (row-major over the block's d axes), edge-replicated padding */
                int p[3] = {0, 0, 0};
                int r = f;
                for (int i = 2; i >= 3 - d; i--) { p[i] = r % 4; r /= 4; }
                uint64_t i0 = b0 * 4 + p[0], i1 = b1 * 4 + p[1], i2 = b2 * 4 + p[2];
                if (i0 >= n[0]) i0 = n[0] - 1;
                if (i1 >= n[1]) i1 = n[1] - 1;
                if (i2 >= n[2]) i2 = n[2] - 1;
                const uint64_t e = (i0 * n[1] + i1) * n[2] + i2;
                v[f] = dtype == ORC_F32 ? (double)f32[e] : f64[e];
                if (!isfinite(v[f])) bad = 1;
                const double a = fabs(v[f]);
                if (a > maxabs) maxabs = a;
            }
            uint64_t fx[64];
            const int zero = maxabs == 0.0;
            int emax = 0;
            if (!zero) {
                int e;
                frexp(maxabs, &e);
                emax = e - 1;                      /* floor(log2(maxabs)) after the :141-144 guards */
            }
            if (emax < -s.bias) emax = -s.bias;   /* :145 */
            const int shift = s.q - 2 - emax;
            for (int f = 0; f < m; f++)
                fx[f] = zero ? 0 : ((uint64_t)(int64_t)rint(ldexp(v[f], shift))) & s.mask;
            transform(&s, fx, d, 1);
            uint64_t pos = b * w;
            put_bit(pay, pos++, zero);
            const uint64_t biased = zero ? 0 : (uint64_t)(emax + s.bias);
            for (int i = 0; i < s.ebits; i++) put_bit(pay, pos++, (int)((biased >> (s.ebits - 1 - i)) & 1));
            uint64_t nbv[64];
            for (int k = 0; k < m; k++) nbv[k] = zero ? 0 : ((fx[perm[k]] + s.nb) & s.mask) ^ s.nb;   /* :204-208 */
            for (int t = 0; t < rate; t++)
                for (int k = 0; k < m; k++) put_bit(pay, pos++, (int)((nbv[k] >> (s.q - 1 - t)) & 1));
        }
    }
    return bad ? ORC_VALIDATION : ORC_OK;
}

/* Header of a fixed-rate stream (zfp.py:314-334). */
int orz_peek(const uint8_t *in, uint64_t len, int *dtype, int *rank, uint64_t *dims, int *rate) {
    if (len < HDR) return ORC_CORRUPT;
    const int d = in[0], dt = in[1];
    if (d < 1 || d > MAX_RANK || dt > 6) return ORC_CORRUPT;
    if (dt != ORC_F32 && dt != ORC_F64) return ORC_CORRUPT;
    const Spec s = spec_of(dt);
    if (in[2] < 1 || in[2] > s.q) return ORC_VALIDATION;          /* RateSpec.__post_init__ */
    if (len < HDR + 8ull * d) return ORC_CORRUPT;
    memcpy(dims, in + HDR, 8ull * d);
    uint64_t total;
    int rc = orz_compressed_size(dt, d, dims, in[2], &total);
    if (rc) return rc;
    if (len < total) return ORC_CORRUPT;                          /* :333-334 */
    *dtype = dt; *rank = d; *rate = in[2];
    return ORC_OK;
}

/* zfp.py:311-353 (bitplane_decode :244-264, inverse_transform, exp_restore :153-157). */
int orz_decompress(const uint8_t *in, uint64_t len, void *out, uint64_t out_cap) {
    int dtype, d, rate;
    uint64_t dims[3];
    int rc = orz_peek(in, len, &dtype, &d, dims, &rate);
    if (rc) return rc;
    const Spec s = spec_of(dtype);
    const int m = d == 1 ? 4 : d == 2 ? 16 : 64;
    uint64_t n[3] = {1, 1, 1}, g[3] = {1, 1, 1};
    for (int i = 0; i < d; i++) { n[3 - d + i] = dims[i]; g[3 - d + i] = (dims[i] + 3) / 4; }
    if (out_cap < n[0] * n[1] * n[2] * (dtype == ORC_F32 ? 4 : 8)) return ORC_ALLOC;
    const uint64_t nblk = g[0] * g[1] * g[2], w = block_bits(&s, d, rate);
    int perm[64];
    sequency_perm(d, perm);
    const uint8_t *pay = in + HDR + 8 * d;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
    for (int64_t bb = 0; bb < (int64_t)nblk; bb++) {
        const uint64_t b = (uint64_t)bb;
        uint64_t pos = b * w;
        const int zero = get_bit(pay, pos++);
        int64_t biased = 0;
        for (int i = 0; i < s.ebits; i++) biased = (biased << 1) | get_bit(pay, pos++);
        const int emax = zero ? -s.bias : (int)(biased - s.bias);
        uint64_t nbv[64] = {0}, fx[64];
        for (int t = 0; t < rate; t++)
            for (int k = 0; k < m; k++) nbv[k] |= (uint64_t)get_bit(pay, pos++) << (s.q - 1 - t);
        for (int k = 0; k < m; k++) fx[perm[k]] = zero ? 0 : ((nbv[k] ^ s.nb) - s.nb) & s.mask;
        transform(&s, fx, d, 0);
        const uint64_t b2 = b % g[2], b1 = (b / g[2]) % g[1], b0 = b / (g[2] * g[1]);
        for (int f = 0; f < m; f++) {
            int p[3] = {0, 0, 0};
            int r = f;
            for (int i = 2; i >= 3 - d; i--) { p[i] = r % 4; r /= 4; }
            const uint64_t i0 = b0 * 4 + p[0], i1 = b1 * 4 + p[1], i2 = b2 * 4 + p[2];
            if (i0 >= n[0] || i1 >= n[1] || i2 >= n[2]) continue;   /* padding discarded */
            const uint64_t e = (i0 * n[1] + i1) * n[2] + i2;
            const double val = zero ? 0.0 : ldexp((double)sx(&s, fx[f]), emax - (s.q - 2));
            if (dtype == ORC_F32) ((float *)out)[e] = (float)val;
            else ((double *)out)[e] = val;
        }
    }
    return ORC_OK;
}
