// codec.cu -- the MGARD blob path (codec.py:25-113) and the C ABI of include/hpdr_b200.h.
//
// Blob layout (little-endian, no padding; codec.py:43-55, huffman.py:361-396):
//   rank u8 | dims u64*rank | dtype u8 eb_rel f64 dict u32 u_min f64 u_max f64 eb_abs f64
//   bin_width f64 levels u32 | n_out u64 | idx u64*n_out | bins i64*n_out | n_coarse u64 |
//   coarse f64*n_coarse | dict u16 | n_sym u64 | lengths u8*dict | n_units u32 |
//   offsets u64*n_units | total_bits u64 | packed bits (MSB first)
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <memory>
#include <new>

#include "stages.cuh"
#include "transform.cuh"
#include "fused.cuh"

namespace hpdr {

namespace {

template <class F>
int guard(F &&f) {
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

[[noreturn]] void fail(int code, const std::string &msg, int64_t bit = -1) { throw Error{code, msg, bit}; }

std::string fmt_double(double v) {
    char b[64];
    snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

int itemsize(int dtype) {
    static const int sz[7] = {4, 8, 4, 8, 4, 8, 1};
    return (dtype >= 0 && dtype < 7) ? sz[dtype] : 0;
}

template <class T>
void put(std::vector<uint8_t> &v, T x) {
    size_t o = v.size();
    v.resize(o + sizeof(T));
    memcpy(v.data() + o, &x, sizeof(T));
}

// Bounds-checked little-endian reader over the blob.
struct Reader {
    const uint8_t *p;
    uint64_t len, pos = 0;
    bool has(uint64_t n) const { return pos <= len && n <= len - pos; }
    template <class T>
    bool get(T &out) {
        if (!has(sizeof(T))) return false;
        memcpy(&out, p + pos, sizeof(T));
        pos += sizeof(T);
        return true;
    }
};

// Device -> host copy of a result: pageable destinations through the pinned staging ring.
void result_to_host(hpdr_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t s) {
    if (n >= (1u << 20) && classify(dst) == MemKind::Host) stage_d2h(ctx, dst, src, n, s);
    else CUDA_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s));
}

// Device-resident input: copy host data to a context buffer when needed.
const void *device_input(hpdr_ctx *ctx, const void *in, size_t bytes, const char *name, cudaStream_t s) {
    const MemKind k = classify(in);
    if (k == MemKind::Device) return in;
    void *d = ctx->dbuf(name, bytes);
    if (k == MemKind::Host) stage_h2d(ctx, d, in, bytes, s);   // pageable: pinned staging ring
    else CUDA_CHECK(cudaMemcpyAsync(d, in, bytes, cudaMemcpyDefault, s));
    return d;
}

// Number of levels for arbitrary dims (hierarchy.py:63-74), for the stored-level check.
int levels_of(const std::vector<uint64_t> &dims) {
    int nco = 0;
    for (uint64_t n : dims) {
        int st = 0;
        while (n > 2) { n = n / 2 + 1; st++; }
        nco = std::max(nco, st);
    }
    return nco + 1;
}

// Encode keys (device) into the pending Huffman layout.  Returns false for single-key streams.
void huffman_stage(hpdr_ctx *ctx, const uint16_t *d_keys, int64_t n, uint32_t dict, const std::vector<uint64_t> &hist,
                   std::vector<uint8_t> &mid, EncodeResult &enc, bool &single, cudaStream_t s,
                   const EncodeHooks *hooks = nullptr) {
    // huffman_compress (huffman.py:366-396)
    put<uint16_t>(mid, (uint16_t)dict);
    put<uint64_t>(mid, (uint64_t)n);
    single = false;
    enc = EncodeResult();
    if (n == 0) {
        mid.insert(mid.end(), dict, 0);
        put<uint32_t>(mid, 0);
        single = true;
        return;
    }
    std::vector<uint8_t> lens(dict);
    std::vector<uint32_t> codes(dict);
    std::string err;
    static const bool tcb = getenv("HPDR_PHASES") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = build_codebook(hist.data(), dict, lens.data(), codes.data(), err);
    if (tcb)
        fprintf(stderr, "[codebook] %.1f us\n",
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    if (rc == HPDR_ERR_OVERFLOW) fail(rc, "Python integer out of bounds for uint32");
    if (rc) fail(rc, err);
    mid.insert(mid.end(), lens.begin(), lens.end());
    uint32_t present = 0;
    for (uint32_t k = 0; k < dict; k++) present += hist[k] != 0;
    if (present == 1) {
        put<uint32_t>(mid, 0);
        single = true;
        return;
    }
    put<uint32_t>(mid, (uint32_t)((n + kBlockSymbols - 1) / kBlockSymbols));
    encode_device(ctx, d_keys, n, dict, lens.data(), codes.data(), enc, s, hooks, hist.data());
}

// Write the pending stream (head | outliers | mid | offsets | total_bits | packed) to out; with
// payload = false everything but the packed bytes.  Returns the offset of the packed bytes.
uint64_t fetch_pending(hpdr_ctx *ctx, const hpdr_ctx::Pending &P, void *out, uint64_t cap, cudaStream_t s, bool sync,
                       bool payload) {
    if (!P.valid) fail(HPDR_ERR_VALIDATION, "no pending compressed stream in this context");
    if (cap < P.total_len) fail(HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(P.total_len));
    const MemKind ok = classify(out);
    const bool dev = ok == MemKind::Device;
    uint8_t *o = (uint8_t *)out;
    uint64_t pos = 0;
    auto host_bytes = [&](const void *src, size_t n) {
        if (!n) return;
        if (dev) CUDA_CHECK(cudaMemcpyAsync(o + pos, src, n, cudaMemcpyHostToDevice, s));
        else memcpy(o + pos, src, n);
        pos += n;
    };
    auto dev_bytes = [&](const void *src, size_t n) {
        if (!n) return;
        if (ok == MemKind::Host && n >= (1u << 20)) stage_d2h(ctx, o + pos, src, n, s);   // pageable (Python bytes)
        else CUDA_CHECK(cudaMemcpyAsync(o + pos, src, n, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        pos += n;
    };
    if (!P.huffman_only) {
        host_bytes(P.head.data(), P.head.size());
        dev_bytes(ctx->dbuf(ctx->oname("oidx", P.slot), P.n_out * 8), P.n_out * 8);
        dev_bytes(ctx->dbuf(ctx->oname("obins", P.slot), P.n_out * 8), P.n_out * 8);
    }
    host_bytes(P.mid.data(), P.mid.size());
    uint64_t pay = pos;
    if (!P.single_key) {
        dev_bytes(ctx->dbuf(ctx->oname("enc_uoff", P.slot), (P.n_units + 1) * 8), P.n_units * 8);
        uint64_t tb = P.total_bits;
        host_bytes(&tb, 8);
        pay = pos;
        if (payload)
            dev_bytes(ctx->dbuf(ctx->oname("enc_words", P.slot), (P.total_bits + 31) / 32 * 4 + 8), (P.total_bits + 7) / 8);
    } else {
        uint64_t z = 0;
        host_bytes(&z, 8);
        pay = pos;
    }
    if (sync) CUDA_CHECK(cudaStreamSynchronize(s));
    return pay;
}

void fetch_pending(hpdr_ctx *ctx, void *out, uint64_t cap) { fetch_pending(ctx, ctx->pending, out, cap, ctx->stream, true, true); }

struct HuffHeader {
    uint32_t dict = 0;
    uint64_t n_sym = 0;
    const uint8_t *lengths = nullptr;
    uint32_t n_units = 0;
    const uint8_t *offsets = nullptr;
    uint64_t total_bits = 0;
    const uint8_t *packed = nullptr;
    const uint8_t *packed_dev = nullptr;   // device copy of the packed bits, when available
    uint32_t n_present = 0, first_present = 0;
    bool single = false;
};

// huffman_decompress header checks, in the reference's order (huffman.py:399-433).
// Returns false when n_sym == 0 (empty key array).
bool parse_huffman(const uint8_t *d, uint64_t len, HuffHeader &h) {
    Reader r{d, len};
    uint16_t dict;
    if (len < 10) fail(HPDR_ERR_CORRUPT, "stream shorter than fixed header");
    r.get(dict);
    r.get(h.n_sym);
    h.dict = dict;
    if (!r.has((uint64_t)dict + 4)) fail(HPDR_ERR_CORRUPT, "stream truncated in length array");
    h.lengths = d + r.pos;
    r.pos += dict;
    r.get(h.n_units);
    if (!r.has(8ULL * h.n_units + 8)) fail(HPDR_ERR_CORRUPT, "stream truncated in decode-unit index");
    h.offsets = d + r.pos;
    r.pos += 8ULL * h.n_units;
    r.get(h.total_bits);
    if (h.n_sym == 0) return false;
    for (uint32_t k = 0; k < dict; k++)
        if (h.lengths[k]) {
            if (!h.n_present) h.first_present = k;
            h.n_present++;
        }
    if (!h.n_present) fail(HPDR_ERR_CORRUPT, "no codewords in stored length array");
    if (h.n_units == 0 && h.total_bits == 0) {
        if (h.n_present != 1) fail(HPDR_ERR_CORRUPT, "empty payload with multi-key codebook");
        h.single = true;
        return true;
    }
    const uint64_t pbytes = h.total_bits / 8 + (h.total_bits % 8 != 0);
    if (!r.has(pbytes))
        fail(HPDR_ERR_CORRUPT, "stream truncated in packed bits", (int64_t)((len - r.pos) * 8));
    h.packed = d + r.pos;
    std::vector<uint32_t> codes(dict ? dict : 1);
    if (canonical_codes(h.lengths, dict, codes.data()) != HPDR_OK)
        fail(HPDR_ERR_OVERFLOW, "Python integer out of bounds for uint32");
    const uint64_t need = (h.n_sym + kBlockSymbols - 1) / kBlockSymbols;
    if (h.n_units < need)
        fail(HPDR_ERR_CORRUPT, "stream has " + std::to_string(h.n_units) + " decode units, need " + std::to_string(need));
    return true;
}

// Decode (and optionally dequantize) the parsed stream.  keys / coef may be null (check-only).
DecodeResult run_decode(hpdr_ctx *ctx, const HuffHeader &h, uint32_t *keys, double *coef, double bin,
                        uint32_t key_limit, cudaStream_t s) {
    DecodeResult res;
    if (h.single) {
        if (keys || coef) fill_single(keys, coef, (int64_t)h.n_sym, h.first_present, bin, s);
        res.max_key = h.first_present;
        res.key_out_of_range = h.first_present >= key_limit;
        return res;
    }
    DecodeJob job;
    job.dict_size = h.dict;
    job.lengths = h.lengths;
    job.n_symbols = h.n_sym;
    job.n_units = (h.n_sym + kBlockSymbols - 1) / kBlockSymbols;
    job.offsets = h.offsets;
    job.total_bits = h.total_bits;
    job.packed = h.packed_dev ? h.packed_dev : h.packed;
    job.packed_on_device = h.packed_dev != nullptr;
    job.keys = keys;
    job.coef = coef;
    job.bin_width = bin;
    job.key_limit = key_limit;
    decode_device(ctx, job, res, s);
    if (res.bad_bit >= 0)
        fail(HPDR_ERR_CORRUPT, "invalid or truncated codeword at bit " + std::to_string(res.bad_bit), res.bad_bit);
    return res;
}

__global__ void k_outliers(double *coef, int64_t n, const uint64_t *idx, const int64_t *bins, uint64_t m, double bw,
                           int *flags) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)m; k += (int64_t)gridDim.x * blockDim.x) {
        long long i = (long long)idx[k];
        if (i < 0) i += n;                                   // numpy negative indices
        if (i < 0 || i >= n) { atomicOr(flags, 1); continue; }
        if (k > 0 && idx[k] <= idx[k - 1]) atomicOr(flags, 2);   // not strictly ascending
        coef[i] = __dmul_rn((double)bins[k], bw);
    }
}

__global__ void k_outliers_serial(double *coef, int64_t n, const uint64_t *idx, const int64_t *bins, uint64_t m, double bw) {
    for (uint64_t k = 0; k < m; k++) {
        long long i = (long long)idx[k];
        if (i < 0) i += n;
        coef[i] = __dmul_rn((double)bins[k], bw);
    }
}

__global__ void k_set_coarse(double *coef, const long long *idx, const double *vals, int n, int broadcast) {
    int k = threadIdx.x;
    if (k < n) coef[idx[k]] = broadcast ? vals[0] : vals[k];
}

// values = unzigzag(keys) * bin (quantize.py:110-111), tracking the largest key
__global__ void k_dequant(const uint32_t *__restrict__ keys, int64_t n, double bw, double *__restrict__ coef,
                          unsigned *__restrict__ kmax_g) {
    unsigned kmax = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        kmax = k > kmax ? k : kmax;
        const long long b = (long long)(k >> 1) ^ -(long long)(k & 1u);
        coef[i] = __dmul_rn((double)b, bw);
    }
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    if ((threadIdx.x & 31) == 0 && kmax) atomicMax(kmax_g, kmax);
}

// Coarse restore of quantize.py:116-117 (values[coarse_idx] = coarse_values, numpy broadcast rules).
void restore_coarse(hpdr_ctx *ctx, double *coef, const DevPlan &p, const double *coarse, uint64_t n_co, cudaStream_t s) {
    const size_t nci = p.host.coarsest.size();
    if (n_co != nci && n_co != 1)
        fail(HPDR_ERR_VALUE, "shape mismatch: value array of shape (" + std::to_string(n_co) +
                                 ",) could not be broadcast to indexing result of shape (" + std::to_string(nci) + ",)");
    long long *di = (long long *)ctx->dbuf("co_idx", 16 * 8);
    double *dv = (double *)ctx->dbuf("co_val", 16 * 8);
    long long *hs = (long long *)ctx->hbuf("co_stage", 32 * 8);
    for (size_t k = 0; k < nci; k++) hs[k] = p.host.coarsest[k];
    memcpy(hs + 16, coarse, std::min<size_t>(n_co, 16) * 8);
    small_copy(di, hs, 16 * 8, s);
    small_copy(dv, hs + 16, 16 * 8, s);
    k_set_coarse<<<1, 32, 0, s>>>(coef, di, dv, (int)nci, n_co == 1 && nci != 1);
    LAUNCH_CHECK();
}

}  // namespace

int scatter_outliers(hpdr_ctx *ctx, double *coef, int64_t n, const uint64_t *h_idx, const int64_t *h_bins,
                     uint64_t n_out, double bin_width, cudaStream_t s) {
    if (!n_out) return HPDR_OK;
    uint64_t *di = (uint64_t *)ctx->dbuf("dq_oidx", n_out * 8);
    int64_t *db = (int64_t *)ctx->dbuf("dq_obins", n_out * 8);
    int *fl = (int *)ctx->dbuf("dq_flags", 16);
    small_copy(di, h_idx, n_out * 8, s);
    small_copy(db, h_bins, n_out * 8, s);
    zero_async(fl, 16, s);
    {
        KPROF("k_outliers", 24.0 * n_out, s);
        k_outliers<<<grid_for(n_out, 256, 148 * 8), 256, 0, s>>>(coef, n, di, db, n_out, bin_width, fl);
        LAUNCH_CHECK();
    }
    int *h = (int *)ctx->hbuf("dq_flags_h", 16);
    small_copy(h, fl, 4, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (h[0] & 1) return HPDR_ERR_INDEX;
    if (h[0] & 2) {   // duplicates / unordered (never produced by the encoder): numpy's last-wins order
        k_outliers_serial<<<1, 1, 0, s>>>(coef, n, di, db, n_out, bin_width);
        LAUNCH_CHECK();
    }
    return HPDR_OK;
}

}  // namespace hpdr

using namespace hpdr;

extern "C" {

}  // extern "C"

namespace hpdr {
void fetch_pending_on(hpdr_ctx *ctx, const hpdr_ctx::Pending &P, void *out, uint64_t cap, cudaStream_t s, bool sync) {
    fetch_pending(ctx, P, out, cap, s, sync, true);
}

__global__ void k_widen_keys(const uint16_t *__restrict__ a, uint32_t *__restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_narrow_keys(const uint32_t *__restrict__ a, uint16_t *__restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (uint16_t)a[i];
}

__global__ void k_gather_vals(const double *__restrict__ src, const long long *__restrict__ idx, int n,
                              double *__restrict__ dst) {
    const int k = threadIdx.x;
    if (k < n) dst[k] = src[idx[k]];
}

// codec.py:43-56 from quantized keys on: coarse values (d_coarse: dense coarsest level, or
// coef_for_coarse: the CoefficientSet whose coarsest slots hold them), head, Huffman stage, and
// the optional streamed fetch into fetch_out.
void finish_blob(hpdr_ctx *ctx, DevPlan &p, int dtype, int rank, const uint64_t *dims, double eb_rel,
                 uint32_t dict_size, double u_min, double u_max, double eb_abs, double bin, const QuantResult &q,
                 uint16_t *keys, const double *d_coarse, const double *coef_for_coarse, void *fetch_out,
                 uint64_t fetch_cap, bool coarse_ready = false, const OutAlloc *alloc = nullptr) {
    {
        const int64_t N = p.n_total;
        const int L = p.host.L;
        cudaStream_t s = ctx->stream;
        if (q.flags & 1) fail(HPDR_ERR_VALIDATION, "coefficients contain non-finite values");
        if (q.flags & 2) fail(HPDR_ERR_VALIDATION, "coefficient exceeds representable bin range");
        const size_t nco = p.host.coarsest.size();
        std::vector<double> coarse(nco);
        // one copy into pinned staging (the coarsest set is <= 16 values; gathered on the device
        // from the coefficient set when there is no dense coarsest level)
        double *hco = (double *)ctx->hbuf("coarse_rb", 16 * 8);
        if (coarse_ready) {
            // read back with the histogram (quantize_finish's round trip)
        } else if (d_coarse) {
            small_copy(hco, d_coarse, nco * 8, s);
        } else if (nco) {
            double *dco = (double *)ctx->dbuf("coarse_gather", 16 * 8);
            k_gather_vals<<<1, 32, 0, s>>>(coef_for_coarse, p.coarsest, (int)nco, dco);
            LAUNCH_CHECK();
            small_copy(hco, dco, nco * 8, s);
        }
        if (!coarse_ready) CUDA_CHECK(cudaStreamSynchronize(s));
        if (nco) memcpy(coarse.data(), hco, nco * 8);
        auto &P = ctx->pending;
        P = hpdr_ctx::Pending();
        put<uint8_t>(P.head, (uint8_t)rank);
        for (int d = 0; d < rank; d++) put<uint64_t>(P.head, dims[d]);
        put<uint8_t>(P.head, (uint8_t)dtype);
        put<double>(P.head, eb_rel);
        put<uint32_t>(P.head, dict_size);
        put<double>(P.head, u_min);
        put<double>(P.head, u_max);
        put<double>(P.head, eb_abs);
        put<double>(P.head, bin);
        put<uint32_t>(P.head, (uint32_t)L);
        put<uint64_t>(P.head, q.n_outliers);
        P.n_out = q.n_outliers;
        put<uint64_t>(P.mid, (uint64_t)nco);
        for (double v : coarse) put<double>(P.mid, v);
        EncodeResult enc;
        bool single;
        phase_mark("coarse_read", s);
        // Streamed fetch (pinned / device output): as soon as the stream layout is known the blob
        // head, outliers and unit offsets go out on the D2H stream, and the packed payload follows
        // unit group by unit group behind the encode launches.
        EncodeHooks hooks;
        bool streamed_fetch = false;
        uint64_t pay_pos = 0;
        MemKind ok = fetch_out ? classify(fetch_out) : MemKind::Host;
        // pageable destinations (the drop-in's Python bytes, allocated through `alloc` once the size is
        // known): the head and each payload group go out through the pinned staging ring after the
        // encode launches are all enqueued (host-blocking copies must not hold up the launches)
        std::vector<std::pair<uint64_t, uint64_t>> pg_ranges;
        std::vector<int> pg_groups;
        hpdr_ctx::Pending PQ;
        const char *words_dev = nullptr;   // the packed payload (EncodeResult::d_words)
        if ((fetch_out && ok != MemKind::Host) || (!fetch_out && alloc)) {
            hooks.groups = N >= (16LL << 20) ? 8 : 1;   // small streams: one launch, no group read-back
            hooks.ready = [&](const EncodeResult &e) {
                const uint64_t total = P.head.size() + 16 * P.n_out + P.mid.size() + 8 * e.n_units + 8 + (e.total_bits + 7) / 8;
                if (!fetch_out) {
                    fetch_out = alloc->fn(alloc->user, total);
                    if (!fetch_out) fail(HPDR_ERR_ALLOCATION, "output allocation failed");
                    fetch_cap = total;
                    ok = classify(fetch_out);
                }
                if (fetch_cap < total) return;
                streamed_fetch = true;
                words_dev = (const char *)e.d_words;
                hpdr_ctx::Pending Q = P;
                Q.n_units = e.n_units;
                Q.total_bits = e.total_bits;
                Q.total_len = total;
                Q.slot = ctx->out_slot;
                Q.valid = true;
                CUDA_CHECK(cudaEventRecord(ctx->event(0), s));
                CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(0), 0));
                if (ok == MemKind::Host) PQ = Q;   // pageable: after the launches
                else pay_pos = fetch_pending(ctx, Q, fetch_out, fetch_cap, ctx->d2h, false, /*payload=*/false);
            };
            hooks.group_done = [&](int g, uint64_t lo, uint64_t hi) {
                if (!streamed_fetch || hi <= lo) return;
                CUDA_CHECK(cudaEventRecord(ctx->event(EvEncGroup, g), s));
                if (ok == MemKind::Host) {
                    pg_ranges.emplace_back(lo, hi);
                    pg_groups.push_back(g);
                    return;
                }
                CUDA_CHECK(cudaStreamWaitEvent(ctx->d2h, ctx->event(EvEncGroup, g), 0));
                const bool dev = ok == MemKind::Device;
                CUDA_CHECK(cudaMemcpyAsync((char *)fetch_out + pay_pos + lo, words_dev + lo, hi - lo,
                                           dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->d2h));
            };
        }
        huffman_stage(ctx, keys, N, dict_size, q.hist, P.mid, enc, single, s,
                      (fetch_out || alloc) ? &hooks : nullptr);
        if (streamed_fetch && ok == MemKind::Host) {
            pay_pos = fetch_pending(ctx, PQ, fetch_out, fetch_cap, ctx->d2h, false, /*payload=*/false);
            const char *words = words_dev;
            std::vector<StageRange> rs;
            for (size_t g = 0; g < pg_ranges.size(); g++)
                rs.push_back({pg_ranges[g].first, pg_ranges[g].second, ctx->event(EvEncGroup, pg_groups[g])});
            stage_d2h_ranges(ctx, (char *)fetch_out + pay_pos, words, rs, ctx->d2h);
        }
        phase_mark("encoded", s);
        P.single_key = single;
        P.n_units = enc.n_units;
        P.total_bits = enc.total_bits;
        P.total_len = P.head.size() + 16 * P.n_out + P.mid.size() + 8 * P.n_units + 8 + (P.total_bits + 7) / 8;
        P.slot = ctx->out_slot;
        P.valid = true;
        P.fetched = streamed_fetch;
        if (streamed_fetch) CUDA_CHECK(cudaStreamSynchronize(ctx->d2h));
    }
}

// mgard_compress (codec.py:25-56) up to a pending blob in ctx->pending (device parts in output
// slot ctx->out_slot).  allow_stream: a host input may be streamed in dim-0 chunks.
void compress_core(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                   uint32_t dict_size, int has_range, double range_min, double range_max, bool allow_stream,
                   void *fetch_out, uint64_t fetch_cap, const OutAlloc *alloc) {
    {
        ctx->pending.valid = false;
        if (dtype != 0 && dtype != 1) fail(HPDR_ERR_VALIDATION, "lossy compression needs F32/F64");
        DevPlan &p = ctx->plan(rank, dims);
        const int64_t N = p.n_total;
        const int L = p.host.L;
        cudaStream_t s = ctx->stream;
        // quantize.py:58-62 (the reference checks these after decompose; nothing before can fail)
        if (!(0.0 < eb_rel && eb_rel < 1.0)) fail(HPDR_ERR_VALIDATION, "eb_rel must be in (0, 1), got " + fmt_double(eb_rel));
        if (dict_size < 2 || dict_size > 65535)
            fail(HPDR_ERR_VALIDATION, "dict_size must be in [2, 65535], got " + std::to_string(dict_size));
        const bool host_in = classify(in) != MemKind::Device;
        const bool fused = L > 1 && use_fused(p);
        static const bool no_stream = getenv("HPDR_NO_STREAM") != nullptr;
        const bool streamed = host_in && fused && !no_stream && allow_stream;
        phase_mark("start", s);
        const void *d_in = streamed ? nullptr : device_input(ctx, in, (size_t)N * itemsize(dtype), "input", s);
        double u_min = range_min, u_max = range_max;
        if (!has_range && !streamed) {
            minmax_device(ctx, d_in, dtype, N, &u_min, &u_max, s);
            apply_range_hook(ctx, &u_min, &u_max);
        }
        phase_mark("minmax", s);
        uint16_t *keys = (uint16_t *)ctx->dbuf("keys16", N * 2 + 64);
        QuantResult q;
        const double *d_coarse;
        double eb_abs = 0.0, bin = 1.0;
        bool coarse_ready = false;
        if (fused) {
            // quantize-on-write: keys, outlier mask and histogram come out of the level kernels
            QuantOut qo;
            qo.half = dict_size / 2;
            qo.dict = dict_size;
            qo.keys = keys;
            const int64_t words = (N + 31) / 32;
            qo.omask = (uint32_t *)ctx->dbuf("omask", words * 4);
            qo.obins = (long long *)ctx->dbuf("obins_sparse", N * 8);
            qo.hist = (unsigned long long *)ctx->dbuf("hist", (size_t)dict_size * 8);
            qo.flags = (int *)ctx->dbuf("qflags", 16);
            zero_async(qo.omask, words * 4, s);
            zero_async(qo.hist, (size_t)dict_size * 8, s);
            zero_async(qo.flags, 16, s);
            if (streamed) {
                // the range (relative mode) is complete only after the last chunk; q.bin set inside
                d_coarse = decompose_quantize_streamed(ctx, p, in, dtype, has_range, range_min, range_max, eb_rel,
                                                       qo, &u_min, &u_max, s);
            } else {
                qo.bin = bin = 0.0;
            }
            eb_abs = eb_rel * (u_max - u_min);
            bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)L : 1.0;
            if (!streamed) {
                qo.bin = bin;
                d_coarse = decompose_quantize(ctx, p, d_in, dtype, qo, s);
            }
            phase_mark("decomposed", s);
            if (d_coarse && !p.host.coarsest.empty()) {   // the coarsest values ride the next host round trip
                small_copy(ctx->hbuf("coarse_rb", 16 * 8), d_coarse, p.host.coarsest.size() * 8, s);
                coarse_ready = true;
            }
            quantize_finish(ctx, N, dict_size, bin, nullptr, qo.obins, q, s);
            phase_mark("outliers", s);
        } else {
            eb_abs = eb_rel * (u_max - u_min);
            bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)L : 1.0;
            double *coef = (double *)ctx->dbuf("coef", N * 8);
            d_coarse = decompose_device(ctx, p, d_in, dtype, coef, s);
            quantize_device(ctx, coef, N, p.host.coarsest, bin, dict_size, keys, q, s);
        }
        finish_blob(ctx, p, dtype, rank, dims, eb_rel, dict_size, u_min, u_max, eb_abs, bin, q, keys, d_coarse, nullptr,
                    fetch_out, fetch_cap, coarse_ready, alloc);
    }
}

// Phase B of the relative-mode streams pipeline: a chunk already decomposed into coef (device,
// the full CoefficientSet in finest order) is quantized with the global range, now known, and
// entropy coded into a pending blob (quantize.py:50-98 then codec.py:43-56).
void compress_from_coef(hpdr_ctx *ctx, const double *coef, int dtype, int rank, const uint64_t *dims, double eb_rel,
                        uint32_t dict_size, double u_min, double u_max) {
    ctx->pending.valid = false;
    DevPlan &p = ctx->plan(rank, dims);
    if (!(0.0 < eb_rel && eb_rel < 1.0)) fail(HPDR_ERR_VALIDATION, "eb_rel must be in (0, 1), got " + fmt_double(eb_rel));
    if (dict_size < 2 || dict_size > 65535)
        fail(HPDR_ERR_VALIDATION, "dict_size must be in [2, 65535], got " + std::to_string(dict_size));
    const int64_t N = p.n_total;
    const int L = p.host.L;
    uint16_t *keys = (uint16_t *)ctx->dbuf("keys16", N * 2 + 64);
    const double eb_abs = eb_rel * (u_max - u_min);
    const double bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)L : 1.0;
    QuantResult q;
    static const bool tph = getenv("HPDR_PHASES") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    quantize_device(ctx, coef, N, p.host.coarsest, bin, dict_size, keys, q, ctx->stream);
    const auto t1 = std::chrono::steady_clock::now();
    finish_blob(ctx, p, dtype, rank, dims, eb_rel, dict_size, u_min, u_max, eb_abs, bin, q, keys, nullptr, coef, nullptr, 0);
    if (tph) {
        const auto t2 = std::chrono::steady_clock::now();
        fprintf(stderr, "[phaseB] quantize %.0f us, blob %.0f us\n",
                std::chrono::duration<double, std::micro>(t1 - t0).count(),
                std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
}

// Phase A of the relative-mode streams pipeline: decompose a device-resident chunk into coef
// (range-independent, transform.py:287-323) and fold its min/max into mm (k_minmax order keys).
void decompose_chunk(hpdr_ctx *ctx, const void *d_in, int dtype, int rank, const uint64_t *dims, double *coef,
                     unsigned long long *mm) {
    DevPlan &p = ctx->plan(rank, dims);
    if (mm) minmax_accumulate(d_in, dtype, p.n_total, mm, ctx->stream);
    decompose_device(ctx, p, d_in, dtype, coef, ctx->stream);
}
}  // namespace hpdr

extern "C" {

int hpdr_mgard_compress(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                        uint32_t dict_size, int has_range, double range_min, double range_max, void *out,
                        uint64_t out_cap, uint64_t *blob_len) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->out_slot = 0;
        compress_core(ctx, in, dtype, rank, dims, eb_rel, dict_size, has_range, range_min, range_max, true, out, out_cap,
                      nullptr);
        *blob_len = ctx->pending.total_len;
        if (ctx->pending.fetched) CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        else if (out && out_cap >= ctx->pending.total_len) fetch_pending(ctx, out, out_cap);
        else CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        phase_mark("fetched", ctx->stream);
        phase_dump("mgard_compress");
    });
}

int hpdr_mgard_compress_alloc(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                              uint32_t dict_size, int has_range, double range_min, double range_max,
                              hpdr_alloc_fn alloc, void *user, uint64_t *blob_len) {
    return guard([&] {
        if (!alloc) fail(HPDR_ERR_VALIDATION, "alloc callback is required");
        CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->out_slot = 0;
        const OutAlloc oa{alloc, user};
        compress_core(ctx, in, dtype, rank, dims, eb_rel, dict_size, has_range, range_min, range_max, true, nullptr, 0,
                      &oa);
        *blob_len = ctx->pending.total_len;
        if (ctx->pending.fetched) {
            CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } else {   // not streamed (single-key / generic paths): allocate now and copy out
            void *dst = alloc(user, ctx->pending.total_len);
            if (!dst && ctx->pending.total_len) fail(HPDR_ERR_ALLOCATION, "output allocation failed");
            if (ctx->pending.total_len) fetch_pending(ctx, dst, ctx->pending.total_len);
            else CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        }
        phase_mark("fetched", ctx->stream);
        phase_dump("mgard_compress");
    });
}

int hpdr_mgard_fetch(hpdr_ctx *ctx, void *out, uint64_t out_cap) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        fetch_pending(ctx, out, out_cap);
    });
}

int hpdr_mgard_peek(const void *blob, uint64_t len, int *dtype, int *rank, uint64_t *dims) {
    return guard([&] {
        Reader r{(const uint8_t *)blob, len};
        uint8_t rk, dt;
        if (!r.get(rk)) fail(HPDR_ERR_CORRUPT, "truncated stream header");
        for (int d = 0; d < rk; d++) {
            uint64_t v;
            if (!r.get(v)) fail(HPDR_ERR_CORRUPT, "truncated stream header");
            if (d < 4) dims[d] = v;
        }
        if (!r.get(dt)) fail(HPDR_ERR_CORRUPT, "truncated stream header");
        *rank = rk;
        *dtype = dt;
    });
}

}  // extern "C"

namespace hpdr {
// mgard_decompress (codec.py:59-113).  The header is parsed from the host copy of the blob;
// when dev_blob (a device copy of the same bytes) is given, the bulk parts (outliers, packed
// bits) are read from it instead of being copied from the host.
void decompress_core(hpdr_ctx *ctx, const void *blob_in, uint64_t len, const uint8_t *dev_blob, void *out,
                     uint64_t out_bytes, bool sync) {
    {
        cudaStream_t s = ctx->stream;
        const uint8_t *blob = (const uint8_t *)blob_in;
        // A device-resident blob stays on the device: only the parts the host parses (fixed header,
        // coarse values, Huffman header and unit offsets) are copied into a sparse host mirror at
        // their own offsets; outliers and the packed payload are read in place.
        std::unique_ptr<uint8_t[]> mirror;
        if (!dev_blob && classify(blob_in) == MemKind::Device) {
            mirror.reset(new uint8_t[len ? len : 1]);
            const uint8_t *d = (const uint8_t *)blob_in;
            auto pull = [&](uint64_t a, uint64_t b) {
                b = std::min(b, len);
                if (b > a) CUDA_CHECK(cudaMemcpy(mirror.get() + a, d + a, b - a, cudaMemcpyDeviceToHost));
            };
            auto u64_at = [&](uint64_t p) -> uint64_t {
                uint64_t v = 0;
                if (p + 8 <= len) memcpy(&v, mirror.get() + p, 8);
                return v;
            };
            pull(0, 1);
            const uint64_t rk = len ? mirror[0] : 0;
            uint64_t p = 1 + 8 * rk + 49;                         // codec.py:44-49
            pull(1, p + 8);
            const uint64_t no = std::min<uint64_t>(u64_at(p), len / 16);
            p += 8 + 16 * no;                                     // outlier arrays stay on the device
            pull(p, p + 8);
            const uint64_t nco = std::min<uint64_t>(u64_at(p), len / 8);
            const uint64_t h0 = p + 8 + 8 * nco;                  // Huffman stream
            pull(p, h0 + 10);
            uint16_t dict = 0;
            if (h0 + 2 <= len) memcpy(&dict, mirror.get() + h0, 2);
            const uint64_t q = h0 + 10 + dict;
            pull(h0 + 10, q + 4);
            uint32_t nu = 0;
            if (q + 4 <= len) memcpy(&nu, mirror.get() + q, 4);
            pull(q + 4, q + 4 + 8ull * nu + 8);
            blob = mirror.get();
            dev_blob = d;
        }
        // codec.py:62-81 header parse; any truncation is a CorruptStreamError
        Reader r{blob, len};
        const char *trunc = "truncated stream header";
        uint8_t rank;
        if (!r.get(rank)) fail(HPDR_ERR_CORRUPT, trunc);
        std::vector<uint64_t> dims(rank);
        for (int d = 0; d < rank; d++)
            if (!r.get(dims[d])) fail(HPDR_ERR_CORRUPT, trunc);
        uint8_t dtype;
        double eb_rel, u_min, u_max, eb_abs, bin;
        uint32_t dict, levels;
        if (!(r.get(dtype) && r.get(eb_rel) && r.get(dict) && r.get(u_min) && r.get(u_max) && r.get(eb_abs) &&
              r.get(bin) && r.get(levels)))
            fail(HPDR_ERR_CORRUPT, trunc);
        uint64_t n_out, n_co;
        if (!r.get(n_out)) fail(HPDR_ERR_CORRUPT, trunc);
        if (n_out > (len - r.pos) / 8) fail(HPDR_ERR_CORRUPT, trunc);
        const uint64_t oidx_off = r.pos;
        r.pos += 8 * n_out;
        if (n_out > (len - r.pos) / 8) fail(HPDR_ERR_CORRUPT, trunc);
        const uint64_t obins_off = r.pos;
        r.pos += 8 * n_out;
        if (!r.get(n_co)) fail(HPDR_ERR_CORRUPT, trunc);
        if (n_co > (len - r.pos) / 8) fail(HPDR_ERR_CORRUPT, trunc);
        std::vector<double> coarse(n_co);
        if (n_co) memcpy(coarse.data(), blob + r.pos, 8 * n_co);
        r.pos += 8 * n_co;
        if (dtype > 6) fail(HPDR_ERR_CORRUPT, "unknown dtype code " + std::to_string(dtype));
        // huffman_decompress(data[pos:])
        HuffHeader hh;
        const bool has_syms = parse_huffman(blob + r.pos, len - r.pos, hh);
        if (dev_blob && hh.packed) hh.packed_dev = dev_blob + (hh.packed - blob);
        const uint64_t n_sym = has_syms ? hh.n_sym : 0;
        // build_hierarchy(dims) (hierarchy.py:63-66) and the level check (codec.py:95-96)
        bool dims_ok = true;
        uint64_t N = 1;
        for (uint64_t d : dims) {
            if (d < 1) dims_ok = false;
            N *= d;
        }
        const bool plan_ok = dims_ok && rank >= 1 && rank <= 4;
        auto bad_dims = [&] { fail(HPDR_ERR_VALIDATION, "extents must be >= 1"); };
        double *coef = nullptr;
        DevPlan *pp = nullptr;
        if (plan_ok && n_sym == N && levels_of(dims) == (int)levels) {
            pp = &ctx->plan(rank, dims.data());
            coef = (double *)ctx->dbuf("coef", N * 8);
        }
        DecodeResult dr;
        phase_mark("start", s);
        // Streamed decompress (host blob): the payload arrives in unit groups, each decoded as its
        // bytes land, and the finest transition's correction -- which depends only on the finest
        // coefficients (transform.py:342-345) -- follows slab by slab on the side stream.
        const double *T0_pre = nullptr, *T1_pre = nullptr;
        cudaEvent_t ev_pre = nullptr, ev1_pre = nullptr;
        bool t0_split = false;
        static const bool no_stream_dec = getenv("HPDR_NO_STREAM_DECODE") != nullptr;
        static const uint64_t min_stream_bits = getenv("HPDR_STREAM_DECODE_MIN_BITS")
                                                    ? strtoull(getenv("HPDR_STREAM_DECODE_MIN_BITS"), nullptr, 10)
                                                    : (4ull << 20);   // C1 129^3 (4 MB blob): 0.85 -> 0.75 ms
        bool streamed = !no_stream_dec && !dev_blob && has_syms && !hh.single && coef && pp && n_sym == N &&
                        levels_of(dims) == (int)levels && (dtype == 0 || dtype == 1) && pp->host.L > 2 &&
                        use_fused(*pp) && classify(blob_in) != MemKind::Device && hh.n_units >= 64 &&
                        hh.total_bits >= (uint64_t)min_stream_bits && n_out <= N / 64;
        // payload groups of >= 12 MB, 4..16 (decode launches of fewer units lose more than the
        // earlier start gains): 513^3 (106 MB) 8 groups 12.57 vs 12.97 ms with 16; 1024^3 16
        static const int G_env = getenv("HPDR_DEC_GROUPS") ? std::max(1, std::min(32, atoi(getenv("HPDR_DEC_GROUPS")))) : 0;
        const int G = G_env ? G_env
                            : (int)std::max<uint64_t>(4, std::min<uint64_t>(16, ((hh.total_bits + 7) / 8) / (12ull << 20)));
        // Pinned blob: the first payload group goes out before the host-side checks below (~1 ms at
        // 1024^3), into the buffer decode_begin will hand out (same name and size); it stops short
        // of the zero-padded tail decode_begin clears on the compute stream.
        size_t early = 0;
        if (streamed && classify(hh.packed) == MemKind::Pinned) {
            const uint64_t units0 = (hh.n_sym + kBlockSymbols - 1) / kBlockSymbols;
            const uint64_t ub0 = units0 / G;
            const size_t pbytes = (size_t)((hh.total_bits + 7) / 8);
            if (ub0 > 0 && ub0 < units0 && ub0 < hh.n_units) {
                uint64_t off;
                memcpy(&off, hh.offsets + 8 * ub0, 8);   // (byte pointer into the blob)
                const size_t want = std::min<size_t>(pbytes, ((size_t)(off / 8) + 64) & ~size_t(3));
                if (off <= hh.total_bits && want <= (pbytes & ~size_t(3))) {
                    const size_t pwords = ((pbytes / 4 + 12) & ~size_t(3));
                    void *dw = ctx->dbuf("dec_words", pwords * 4);
                    CUDA_CHECK(cudaEventRecord(ctx->event(194), s));
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(194), 0));
                    CUDA_CHECK(cudaMemcpyAsync(dw, hh.packed, want, cudaMemcpyHostToDevice, ctx->h2d));
                    early = want;
                }
            }
        }
        std::vector<uint64_t> uoffs;
        const uint64_t *oidx_h = (const uint64_t *)(blob + oidx_off);   // unaligned-safe reads below
        if (streamed) {
            int max_len = 0;
            for (uint32_t k = 0; k < dict; k++) max_len = std::max<int>(max_len, hh.lengths[k]);
            uoffs.resize(hh.n_units);
            memcpy(uoffs.data(), hh.offsets, 8ull * hh.n_units);
            streamed = max_len <= 32 && (uint64_t)hh.n_units * kBlockSymbols >= N;
            for (uint64_t u = 0; u < hh.n_units && streamed; u++)
                if (uoffs[u] > hh.total_bits || (u && uoffs[u] < uoffs[u - 1])) streamed = false;
            uint64_t prev = 0;
            for (uint64_t k = 0; k < n_out && streamed; k++) {
                uint64_t i;
                memcpy(&i, oidx_h + k, 8);
                if (i >= N || (k && i <= prev)) streamed = false;
                prev = i;
            }
        }
        if (early && !streamed) {   // the one-shot path rewrites the payload buffer on the compute stream
            CUDA_CHECK(cudaEventRecord(ctx->event(195), ctx->h2d));
            CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(195), 0));
        }
        if (streamed) {
            DevPlan &p = *pp;
            const DevStep &st0 = p.steps[0];
            DecodeJob job;
            job.dict_size = hh.dict;
            job.lengths = hh.lengths;
            job.n_symbols = hh.n_sym;
            job.n_units = (hh.n_sym + kBlockSymbols - 1) / kBlockSymbols;
            job.offsets = hh.offsets;
            job.total_bits = hh.total_bits;
            job.packed = hh.packed;
            job.coef = coef;
            job.bin_width = bin;
            job.key_limit = dict;
            DecodeSession S;
            decode_begin(ctx, job, S, s, false);
            uint64_t *di = (uint64_t *)ctx->dbuf("dq_oidx", n_out * 8);
            int64_t *db = (int64_t *)ctx->dbuf("dq_obins", n_out * 8);
            int *fl = (int *)ctx->dbuf("dq_flags", 16);
            // (the outlier lists follow the payload group by group on the copy stream, below)
            zero_async(fl, 16, s);
            phase_mark("dec_begin", s);
            const int64_t units = S.units;
            const int64_t plane = st0.fsh.n[2] * st0.fsh.n[3];
            const int n0 = (int)st0.fsh.n[1];
            const int m0 = fused_out_planes(p, 0);
            const AxisTables &ax0 = p.host.steps[0].ax[1];
            auto ready = [&](int arrived) -> int {
                if (arrived >= n0) return m0;
                if (!ax0.active) return arrived;
                int c = 0;
                while (c < m0 && ax0.r0[c] + 2 < arrived) c++;
                return c;
            };
            double *Z0f = (double *)ctx->dbuf("z0f", z0_elems(p, 0) * 8);
            double *T0f = (double *)ctx->dbuf("t0f", st0.csh.size() * 8);
            // Transition 1's correction streams too: its coefficients arrive with the finest ones,
            // so its pass 1 / pass 2 follow the decode like the finest's and only its Thomas solve
            // is left after the last group (the coarse chain of the recompose waits on it).
            static const bool no_l1 = getenv("HPDR_NO_STREAM_L1") != nullptr;
            const bool lvl1 = !no_l1 && p.host.L > 2 && tiny_start(p, 1) != 1;
            double *Z1f = lvl1 ? (double *)ctx->dbuf("z1f", z0_elems(p, 1) * 8) : nullptr;
            double *T1f = lvl1 ? (double *)ctx->dbuf("t1f", p.steps[1].csh.size() * 8) : nullptr;
            const AxisTables &ax01 = p.host.steps[1].ax[1];
            const std::vector<int32_t> &map01 = p.host.map[1][1];   // level-1 plane -> finest plane
            const int n01 = (int)p.steps[1].fsh.n[1];
            const int m1 = lvl1 ? fused_out_planes(p, 1) : 0;
            auto ready1 = [&](int finest_planes) -> int {   // transition-1 outputs whose stencil has landed
                if (finest_planes >= n0) return m1;
                int arrived = 0;
                while (arrived < n01 && map01[arrived] < finest_planes) arrived++;
                if (!ax01.active) return arrived;
                int c = 0;
                while (c < m1 && ax01.r0[c] + 2 < arrived) c++;
                return c;
            };
            int c1_done = 0;
            const bool fwd1 = lvl1 && thomas_fwd_stream(p, 1);
            int f1 = 0;   // coarse planes of T1f whose forward elimination is done
            auto oidx_at = [&](uint64_t k) {
                uint64_t i;
                memcpy(&i, oidx_h + k, 8);
                return i;
            };
            auto lower = [&](uint64_t key) {   // first outlier index >= key (the list is ascending)
                uint64_t lo = 0, hi = n_out;
                while (lo < hi) {
                    const uint64_t mid = (lo + hi) / 2;
                    if (oidx_at(mid) < key) lo = mid + 1;
                    else hi = mid;
                }
                return lo;
            };
            CUDA_CHECK(cudaEventRecord(ctx->event(0), s));
            CUDA_CHECK(cudaStreamWaitEvent(ctx->h2d, ctx->event(0), 0));   // tables / buffers ready
            const bool pageable_blob = classify(hh.packed) == MemKind::Host;
            size_t copied = early;
            int c_done = 0;
            const bool fwd0 = thomas_fwd_stream(p, 0);
            int f0 = 0;   // coarse planes of T0f whose forward elimination is done
            for (int g = 0; g < G; g++) {
                const int64_t ua = units * g / G, ub = units * (g + 1) / G;
                if (ub <= ua) continue;
                const size_t want = ub < units ? std::min<size_t>(S.pbytes, ((size_t)(uoffs[ub] / 8) + 64) & ~size_t(3))
                                               : S.pbytes;
                if (want > copied) {
                    if (pageable_blob)   // Python bytes: staged while the previous group decodes
                        stage_h2d(ctx, (char *)S.d_words + copied, hh.packed + copied, want - copied, ctx->h2d);
                    else
                        CUDA_CHECK(cudaMemcpyAsync((char *)S.d_words + copied, hh.packed + copied, want - copied,
                                                   cudaMemcpyHostToDevice, ctx->h2d));
                    copied = want;
                }
                const uint64_t o_lo = lower((uint64_t)ua * kBlockSymbols);
                const uint64_t o_hi = ub == units ? n_out : lower((uint64_t)ub * kBlockSymbols);
                if (o_hi > o_lo) {   // this group's outliers (ascending indices: one contiguous range)
                    const size_t ob = 8 * (o_hi - o_lo);
                    const uint8_t *si = blob + oidx_off + 8 * o_lo, *sb = blob + obins_off + 8 * o_lo;
                    if (pageable_blob && ob >= (1u << 20)) {
                        stage_h2d(ctx, di + o_lo, si, ob, ctx->h2d);
                        stage_h2d(ctx, db + o_lo, sb, ob, ctx->h2d);
                    } else {
                        CUDA_CHECK(cudaMemcpyAsync(di + o_lo, si, ob, cudaMemcpyDefault, ctx->h2d));
                        CUDA_CHECK(cudaMemcpyAsync(db + o_lo, sb, ob, cudaMemcpyDefault, ctx->h2d));
                    }
                }
                CUDA_CHECK(cudaEventRecord(ctx->event(EvDecIn, g), ctx->h2d));
                phase_mark("h2d", ctx->h2d);
                CUDA_CHECK(cudaStreamWaitEvent(s, ctx->event(EvDecIn, g), 0));
                decode_units(S, ua, ub, true, s);
                phase_mark("dec", s);
                if (o_hi > o_lo) {
                    k_outliers<<<grid_for(o_hi - o_lo, 256, 148 * 8), 256, 0, s>>>(coef, (int64_t)N, di + o_lo, db + o_lo,
                                                                                 o_hi - o_lo, bin, fl);
                    LAUNCH_CHECK();
                }
                const int planes_done = ub == units ? n0 : (int)std::min<int64_t>(n0, (ub * kBlockSymbols) / plane);
                const int c_ready = ready(planes_done);
                if (c_ready > c_done) {
                    CUDA_CHECK(cudaEventRecord(ctx->event(EvDecCorr, g), s));
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->aux_hi, ctx->event(EvDecCorr, g), 0));
                    fused_pass1_recompose(p, 0, coef, Z0f, ctx->aux_hi, c_done, c_ready);
                    fused_pass2(p, 0, Z0f, T0f, ctx->aux_hi, c_done, c_ready);
                    if (fwd0) {   // the plane-axis solve follows its right-hand side
                        thomas_plane_fwd(p, 0, T0f, c_done, c_ready, ctx->aux_hi);
                        f0 = c_ready;
                    }
                    phase_mark("corr", ctx->aux_hi);
                    c_done = c_ready;
                }
                if (lvl1) {
                    const int c1_ready = ready1(planes_done);
                    if (c1_ready > c1_done) {
                        CUDA_CHECK(cudaEventRecord(ctx->event(EvDecCorr, g), s));
                        CUDA_CHECK(cudaStreamWaitEvent(ctx->side[0], ctx->event(EvDecCorr, g), 0));
                        fused_pass1_recompose(p, 1, coef, Z1f, ctx->side[0], c1_done, c1_ready);
                        fused_pass2(p, 1, Z1f, T1f, ctx->side[0], c1_done, c1_ready);
                        if (fwd1) {   // transition 1's plane-axis solve follows too
                            thomas_plane_fwd(p, 1, T1f, c1_done, c1_ready, ctx->side[0]);
                            f1 = c1_ready;
                        }
                        c1_done = c1_ready;
                    }
                }
            }
            decode_end(ctx, S, dr, s, true);
            if (dr.bad_bit >= 0)
                fail(HPDR_ERR_CORRUPT, "invalid or truncated codeword at bit " + std::to_string(dr.bad_bit), dr.bad_bit);
            if (dr.deferred) {   // redone units were dequantized again: re-apply outliers, redo the correction
                if (n_out) {
                    k_outliers<<<grid_for(n_out, 256, 148 * 8), 256, 0, s>>>(coef, (int64_t)N, di, db, n_out, bin, fl);
                    LAUNCH_CHECK();
                }
                CUDA_CHECK(cudaEventRecord(ctx->event(190), s));
                CUDA_CHECK(cudaStreamWaitEvent(ctx->aux_hi, ctx->event(190), 0));
                fused_pass1_recompose(p, 0, coef, Z0f, ctx->aux_hi);
                fused_pass2(p, 0, Z0f, T0f, ctx->aux_hi);
                f0 = 0;
                if (lvl1) {
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->side[0], ctx->event(190), 0));
                    fused_pass1_recompose(p, 1, coef, Z1f, ctx->side[0]);
                    fused_pass2(p, 1, Z1f, T1f, ctx->side[0]);
                    c1_done = m1;
                    f1 = 0;
                }
            }
            phase_mark("dec_end", s);
            // host output: only the plane-axis sweep here; the in-plane sweeps run per output slab
            t0_split = classify(out) != MemKind::Device && thomas_plane_split(p, 0);
            if (fwd0) thomas_finish_fwd(p, 0, T0f, f0, !t0_split, ctx->aux_hi);
            else if (t0_split) thomas_plane_axis(p, 0, T0f, ctx->aux_hi);
            else thomas_all(p, 0, T0f, ctx->aux_hi);
            phase_mark("thomas0", ctx->aux_hi);
            ev_pre = ctx->event(191);
            CUDA_CHECK(cudaEventRecord(ev_pre, ctx->aux_hi));
            T0_pre = T0f;
            if (lvl1) {
                if (c1_done < m1) {   // outputs whose stencil reached the end of the field
                    CUDA_CHECK(cudaEventRecord(ctx->event(192), s));
                    CUDA_CHECK(cudaStreamWaitEvent(ctx->side[0], ctx->event(192), 0));
                    fused_pass1_recompose(p, 1, coef, Z1f, ctx->side[0], c1_done, m1);
                    fused_pass2(p, 1, Z1f, T1f, ctx->side[0], c1_done, m1);
                }
                if (fwd1) thomas_finish_fwd(p, 1, T1f, f1, true, ctx->side[0]);
                else thomas_all(p, 1, T1f, ctx->side[0]);
                ev1_pre = ctx->event(193);
                CUDA_CHECK(cudaEventRecord(ev1_pre, ctx->side[0]));
                T1_pre = T1f;
            }
        } else if (has_syms) {
            dr = run_decode(ctx, hh, nullptr, coef, bin, dict, s);
        }
        phase_mark("decoded", s);
        if (!dims_ok) bad_dims();
        if (levels_of(dims) != (int)levels) fail(HPDR_ERR_CORRUPT, "stored level count does not match dims");
        // dequantize (quantize.py:101-125)
        if (n_sym != N) fail(HPDR_ERR_VALIDATION, "key count does not match dims");
        if (n_sym && dr.max_key >= dict)
            fail(HPDR_ERR_VALIDATION, "key " + std::to_string(dr.max_key) + " out of range for dict_size " + std::to_string(dict));
        if (!coef) {
            // rank outside 1..4: the reference fails building TensorData after reconstruction
            fail(HPDR_ERR_VALIDATION, rank == 0 ? "dims must be non-empty" : "rank exceeds maximum 4");
        }
        DevPlan &p = *pp;
        if (!streamed) {
            const uint8_t *bulk = dev_blob ? dev_blob : blob;
            int rc = scatter_outliers(ctx, coef, (int64_t)N, (const uint64_t *)(bulk + oidx_off),
                                      (const int64_t *)(bulk + obins_off), n_out, bin, s);
            if (rc == HPDR_ERR_INDEX) fail(rc, "outlier index out of bounds for axis 0 with size " + std::to_string(N));
        }
        restore_coarse(ctx, coef, p, coarse.data(), n_co, s);
        phase_mark("dequantized", s);
        // codec.py:112-113 recompose, then TensorData(dims, dtype, values.astype(dtype))
        const size_t ob = (size_t)N * itemsize(dtype);
        if (out_bytes < ob) fail(HPDR_ERR_BUFFER, "output buffer too small: need " + std::to_string(ob));
        if (classify(out) == MemKind::Device) {
            recompose_into(ctx, p, coef, out, dtype, s, nullptr, T0_pre, ev_pre, false, T1_pre, ev1_pre);
        } else {
            void *stage = ctx->dbuf("out_stage", ob);
            recompose_into(ctx, p, coef, stage, dtype, s, out, T0_pre, ev_pre, t0_split, T1_pre, ev1_pre);
        }
        if (sync) CUDA_CHECK(cudaStreamSynchronize(s));
    }
}
}  // namespace hpdr

extern "C" {

int hpdr_mgard_decompress(hpdr_ctx *ctx, const void *blob_in, uint64_t len, void *out, uint64_t out_bytes) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        decompress_core(ctx, blob_in, len, nullptr, out, out_bytes, true);
        phase_mark("done", ctx->stream);
        phase_dump("mgard_decompress");
    });
}

int hpdr_minmax(hpdr_ctx *ctx, const void *in, int dtype, uint64_t n, double *vmin, double *vmax) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        if (dtype != 0 && dtype != 1) fail(HPDR_ERR_VALIDATION, "min/max needs F32/F64");
        cudaStream_t s = ctx->stream;
        const void *d_in = device_input(ctx, in, (size_t)n * itemsize(dtype), "input", s);
        minmax_device(ctx, d_in, dtype, (int64_t)n, vmin, vmax, s);
    });
}

// ------------------------------------------------------------------ stage entry points
int hpdr_decompose(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, double *coef_out,
                   double *u_min, double *u_max) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        if (dtype != 0 && dtype != 1) fail(HPDR_ERR_VALIDATION, "decomposition requires F32 or F64 input");
        DevPlan &p = ctx->plan(rank, dims);
        cudaStream_t s = ctx->stream;
        const int64_t N = p.n_total;
        const void *d_in = device_input(ctx, in, (size_t)N * itemsize(dtype), "input", s);
        minmax_device(ctx, d_in, dtype, N, u_min, u_max, s);
        double *coef = classify(coef_out) == MemKind::Device ? coef_out : (double *)ctx->dbuf("coef", N * 8);
        decompose_device(ctx, p, d_in, dtype, coef, s);
        if (coef != coef_out) result_to_host(ctx, coef_out, coef, N * 8, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int hpdr_recompose(hpdr_ctx *ctx, const double *coef_in, int rank, const uint64_t *dims, double *out) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        DevPlan &p = ctx->plan(rank, dims);
        cudaStream_t s = ctx->stream;
        const int64_t N = p.n_total;
        const double *coef = (const double *)device_input(ctx, coef_in, N * 8, "coef", s);
        double *rec = classify(out) == MemKind::Device ? out : (double *)ctx->dbuf("out_stage", N * 8);
        recompose_into(ctx, p, coef, rec, 1, s);
        if (rec != out) result_to_host(ctx, out, rec, N * 8, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int hpdr_quantize(hpdr_ctx *ctx, const double *coef_in, int rank, const uint64_t *dims, double u_min, double u_max,
                  double eb_rel, uint32_t dict_size, int has_range, double range_min, double range_max, uint32_t *keys_out,
                  uint64_t *outlier_idx, int64_t *outlier_bins, uint64_t *n_outliers, double *coarse_out,
                  uint64_t *n_coarse, double *eb_abs_out, double *bin_out, uint32_t *levels) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        if (!(0.0 < eb_rel && eb_rel < 1.0)) fail(HPDR_ERR_VALIDATION, "eb_rel must be in (0, 1), got " + fmt_double(eb_rel));
        if (dict_size < 2 || dict_size > 65535)
            fail(HPDR_ERR_VALIDATION, "dict_size must be in [2, 65535], got " + std::to_string(dict_size));
        DevPlan &p = ctx->plan(rank, dims);
        cudaStream_t s = ctx->stream;
        const int64_t N = p.n_total;
        const double *coef = (const double *)device_input(ctx, coef_in, N * 8, "coef", s);
        const double vmin = has_range ? range_min : u_min, vmax = has_range ? range_max : u_max;
        const double eb_abs = eb_rel * (vmax - vmin);
        const double bin = eb_abs > 0 ? (2.0 * eb_abs) / (double)p.host.L : 1.0;
        uint16_t *keys = (uint16_t *)ctx->dbuf("keys16", N * 2 + 64);
        QuantResult q;
        quantize_device(ctx, coef, N, p.host.coarsest, bin, dict_size, keys, q, s);
        if (q.flags & 1) fail(HPDR_ERR_VALIDATION, "coefficients contain non-finite values");
        if (q.flags & 2) fail(HPDR_ERR_VALIDATION, "coefficient exceeds representable bin range");
        // the stage API hands out the reference's uint32 keys (quantize.py:84)
        uint32_t *keys32 = (uint32_t *)ctx->dbuf("keys32", N * 4 + 64);
        if (N) {
            k_widen_keys<<<grid_for(N, 256, 148 * 16), 256, 0, s>>>(keys, keys32, N);
            LAUNCH_CHECK();
        }
        CUDA_CHECK(cudaMemcpyAsync(keys_out, keys32, N * 4, cudaMemcpyDefault, s));
        CUDA_CHECK(cudaMemcpyAsync(outlier_idx, q.d_outlier_idx, q.n_outliers * 8, cudaMemcpyDefault, s));
        CUDA_CHECK(cudaMemcpyAsync(outlier_bins, q.d_outlier_bins, q.n_outliers * 8, cudaMemcpyDefault, s));
        std::vector<double> cv(p.host.coarsest.size());
        for (size_t k = 0; k < cv.size(); k++)
            CUDA_CHECK(cudaMemcpyAsync(&coarse_out[k], coef + p.host.coarsest[k], 8, cudaMemcpyDefault, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        *n_outliers = q.n_outliers;
        *n_coarse = cv.size();
        *eb_abs_out = eb_abs;
        *bin_out = bin;
        *levels = (uint32_t)p.host.L;
    });
}

int hpdr_dequantize(hpdr_ctx *ctx, const uint32_t *keys_in, uint64_t n_keys, int rank, const uint64_t *dims,
                    uint32_t dict_size, double bin_width, const uint64_t *outlier_idx, const int64_t *outlier_bins,
                    uint64_t n_outliers, const double *coarse, uint64_t n_coarse, double *coef_out) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        DevPlan &p = ctx->plan(rank, dims);
        cudaStream_t s = ctx->stream;
        const int64_t N = p.n_total;
        if ((int64_t)n_keys != N) fail(HPDR_ERR_VALIDATION, "key count does not match dims");
        const uint32_t *keys = (const uint32_t *)device_input(ctx, keys_in, N * 4, "hkeys", s);
        double *coef = classify(coef_out) == MemKind::Device ? coef_out : (double *)ctx->dbuf("coef", N * 8);
        unsigned *kmax = (unsigned *)ctx->dbuf("dq_kmax", 16);
        zero_async(kmax, 16, s);
        {
            KPROF("k_dequant", 12.0 * N, s);
            k_dequant<<<grid_for(N, 256, 148 * 16), 256, 0, s>>>(keys, N, bin_width, coef, kmax);
            LAUNCH_CHECK();
        }
        unsigned *hk = (unsigned *)ctx->hbuf("dq_kmax_h", 16);
        CUDA_CHECK(cudaMemcpyAsync(hk, kmax, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (N && hk[0] >= dict_size)
            fail(HPDR_ERR_VALIDATION, "key " + std::to_string(hk[0]) + " out of range for dict_size " + std::to_string(dict_size));
        int rc = scatter_outliers(ctx, coef, N, outlier_idx, outlier_bins, n_outliers, bin_width, s);
        if (rc == HPDR_ERR_INDEX) fail(rc, "outlier index out of bounds for axis 0 with size " + std::to_string(N));
        restore_coarse(ctx, coef, p, coarse, n_coarse, s);
        if (coef != coef_out) result_to_host(ctx, coef_out, coef, N * 8, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int hpdr_histogram(hpdr_ctx *ctx, const uint32_t *keys_in, uint64_t n, uint32_t dict_size, int64_t *counts) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        if (dict_size < 1 || dict_size > (uint32_t)kMaxDict)
            fail(HPDR_ERR_VALIDATION, "dict_size must be in [1, 65535]");
        cudaStream_t s = ctx->stream;
        const uint32_t *keys = n ? (const uint32_t *)device_input(ctx, keys_in, n * 4, "hkeys", s) : nullptr;
        std::vector<uint64_t> hist;
        bool bad = false;
        histogram_device(ctx, keys, (int64_t)n, dict_size, hist, &bad, s);
        if (bad) fail(HPDR_ERR_VALIDATION, "key out of range for dict_size " + std::to_string(dict_size));
        for (uint32_t k = 0; k < dict_size; k++) counts[k] = (int64_t)hist[k];
    });
}

int hpdr_build_codebook(const int64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes) {
    return guard([&] {
        std::vector<uint64_t> c(dict_size);
        for (uint32_t k = 0; k < dict_size; k++) c[k] = counts[k] > 0 ? (uint64_t)counts[k] : 0;
        std::string err;
        int rc = build_codebook(c.data(), dict_size, lengths, codes, err);
        if (rc == HPDR_ERR_OVERFLOW) fail(rc, "Python integer out of bounds for uint32");
        if (rc) fail(rc, err);
    });
}

int hpdr_huffman_compress(hpdr_ctx *ctx, const uint32_t *keys_in, uint64_t n, uint32_t dict_size, uint64_t *stream_len) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->pending.valid = false;
        if (dict_size < 1 || dict_size > (uint32_t)kMaxDict)
            fail(HPDR_ERR_VALIDATION, "dict_size must be in [1, 65535]");
        cudaStream_t s = ctx->stream;
        uint32_t *keys = (uint32_t *)ctx->dbuf("hkeys", n * 4 + 64);
        if (n) CUDA_CHECK(cudaMemcpyAsync(keys, keys_in, n * 4, cudaMemcpyDefault, s));
        std::vector<uint64_t> hist;
        bool bad = false;
        histogram_device(ctx, keys, (int64_t)n, dict_size, hist, &bad, s);
        if (bad) fail(HPDR_ERR_VALIDATION, "key out of range for dict_size " + std::to_string(dict_size));
        // validated keys are < dict_size <= 65535: the encoder reads them as 16 bits
        uint16_t *keys16 = (uint16_t *)ctx->dbuf("hkeys16", n * 2 + 64);
        if (n) {
            k_narrow_keys<<<grid_for((int64_t)n, 256, 148 * 16), 256, 0, s>>>(keys, keys16, (int64_t)n);
            LAUNCH_CHECK();
        }
        auto &P = ctx->pending;
        P = hpdr_ctx::Pending();
        P.huffman_only = true;
        EncodeResult enc;
        bool single;
        huffman_stage(ctx, keys16, (int64_t)n, dict_size, hist, P.mid, enc, single, s);
        P.single_key = single;
        P.n_units = enc.n_units;
        P.total_bits = enc.total_bits;
        P.total_len = P.mid.size() + 8 * P.n_units + 8 + (P.total_bits + 7) / 8;
        P.valid = true;
        *stream_len = P.total_len;
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int hpdr_huffman_fetch(hpdr_ctx *ctx, void *out, uint64_t out_cap) { return hpdr_mgard_fetch(ctx, out, out_cap); }

int hpdr_huffman_decompress(hpdr_ctx *ctx, const void *in, uint64_t len, uint32_t *keys_out, uint64_t cap, uint64_t *n) {
    return guard([&] {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        std::vector<uint8_t> hostcopy;
        const uint8_t *d = (const uint8_t *)in;
        if (classify(in) == MemKind::Device) {
            hostcopy.resize(len);
            CUDA_CHECK(cudaMemcpy(hostcopy.data(), in, len, cudaMemcpyDeviceToHost));
            d = hostcopy.data();
        }
        HuffHeader hh;
        const bool has = parse_huffman(d, len, hh);
        *n = has ? hh.n_sym : 0;
        if (!has) return;
        if (!keys_out || cap < hh.n_sym) fail(HPDR_ERR_BUFFER, "key buffer too small: need " + std::to_string(hh.n_sym));
        const bool dev = classify(keys_out) == MemKind::Device;
        uint32_t *keys = dev ? keys_out : (uint32_t *)ctx->dbuf("hkeys", hh.n_sym * 4 + 64);
        run_decode(ctx, hh, keys, nullptr, 1.0, 0xffffffffu, s);
        if (!dev) result_to_host(ctx, keys_out, keys, hh.n_sym * 4, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
