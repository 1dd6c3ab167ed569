// stages.cuh -- quantization and Huffman stages (device), plus the host codebook.
#pragma once

#include <functional>

#include <vector>

#include "context.cuh"

namespace hpdr {

// ---- quantize.py:50-98 -------------------------------------------------------------
struct QuantResult {
    uint64_t n_outliers = 0;
    int flags = 0;                           // bit0 non-finite coefficient, bit1 bin overflow
    std::vector<uint64_t> hist;              // dict_size counts
    uint64_t *d_outlier_idx = nullptr;       // ascending flat indices (device, n_outliers)
    int64_t *d_outlier_bins = nullptr;       // their signed bins (device, n_outliers)
};

// Quantize N coefficients (device) into keys (device) and the ordered outlier arrays
// (device, sized after counting).  hist is accumulated on the device and copied back.
void quantize_device(hpdr_ctx *ctx, const double *coef, int64_t n, const std::vector<int64_t> &coarsest,
                     double bin_width, uint32_t dict_size, uint16_t *keys, QuantResult &res, cudaStream_t s);

// Second half of quantization once keys, the outlier mask ("omask"), "hist" and "qflags" are
// populated: ordered outlier compaction and read-back.  Outlier bins come from the sparse
// per-element array when given, otherwise they are recomputed from coef.
void quantize_finish(hpdr_ctx *ctx, int64_t n, uint32_t dict_size, double bin_width, const double *coef,
                     const long long *obins_sparse, QuantResult &res, cudaStream_t s);

// Histogram of keys already on the device (huffman.py:74-104).  Sets *bad when a key >= dict.
void histogram_device(hpdr_ctx *ctx, const uint32_t *keys, int64_t n, uint32_t dict_size,
                      std::vector<uint64_t> &hist, bool *bad, cudaStream_t s);

// ---- huffman.py:107-204 (host) -----------------------------------------------------
// Returns HPDR_OK, HPDR_ERR_VALIDATION (empty table / code length > 32).
int build_codebook(const uint64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes, std::string &err);
// Returns HPDR_OK or HPDR_ERR_OVERFLOW (numpy uint32 assignment overflow).
int canonical_codes(const uint8_t *lengths, uint32_t dict_size, uint32_t *codes);

// ---- huffman.py:228-289 (device) ---------------------------------------------------
struct EncodeResult {
    uint64_t n_units = 0;
    uint64_t total_bits = 0;
    uint64_t *d_offsets = nullptr;    // n_units unit bit offsets (device)
    uint32_t *d_words = nullptr;      // packed stream, MSB-first bytes (device)
};
// Optional hooks: ready(res) once offsets / total_bits are known (before the packing kernels);
// group_done(g, lo, hi) after unit group g's packing launch, bytes [lo, hi) of the packed stream
// are then final in stream order.
// Caller-side allocation of a compressed stream's destination once its size is known.
struct OutAlloc {
    hpdr_alloc_fn fn;
    void *user;
};

struct EncodeHooks {
    int groups = 1;
    std::function<void(const EncodeResult &)> ready;
    std::function<void(int, uint64_t, uint64_t)> group_done;
};
void encode_device(hpdr_ctx *ctx, const uint16_t *keys, int64_t n, uint32_t dict_size, const uint8_t *lengths,
                   const uint32_t *codes, EncodeResult &res, cudaStream_t s, const EncodeHooks *hooks = nullptr,
                   const uint64_t *hist = nullptr);   // host histogram: total bits without a device read-back

// ---- huffman.py:207-358 (device) ---------------------------------------------------
struct DecodeJob {
    uint32_t dict_size = 0;
    const uint8_t *lengths = nullptr;  // host
    uint64_t n_symbols = 0;
    uint64_t n_units = 0;              // units to decode (ceil(n/4096))
    const uint8_t *offsets = nullptr;  // host, little-endian u64 x n_units (unaligned ok)
    uint64_t total_bits = 0;
    const uint8_t *packed = nullptr;   // host or device bytes
    bool packed_on_device = false;
    // outputs (device, nullable): keys and / or dequantized coefficients
    uint32_t *keys = nullptr;
    double *coef = nullptr;
    double bin_width = 1.0;
    uint32_t key_limit = 0xffffffffu;  // mgard dict_size for the dequantize range check
};
struct DecodeResult {
    int64_t bad_bit = -1;        // CorruptStreamError bit offset of the lowest failing unit
    bool key_out_of_range = false;
    uint32_t max_key = 0;
    uint64_t deferred = 0;       // units a streamed pass deferred to the final redo
};
void decode_device(hpdr_ctx *ctx, const DecodeJob &job, DecodeResult &res, cudaStream_t s);

// The decode as a session, for streaming the payload in: begin (tables, offsets; payload copy
// unless the caller streams it into d_words), launches over unit ranges (streamed: a unit whose
// canonical walk fails is deferred, not walked, as its bytes may not have landed), end (redo of
// deferred units with the whole payload present, error / max-key readback).
struct DecodeSession {
    DecodeJob job;
    int max_len = 0;
    const char *d_tab = nullptr;
    int64_t units = 0;
    uint64_t *d_off = nullptr;
    uint32_t *d_words = nullptr;
    size_t pbytes = 0, pwords = 0;
    long long *uerr = nullptr;
    unsigned long long *flag = nullptr;
    int *deferred = nullptr;
    unsigned long long *stats = nullptr;
    int window = 1024;                 // shared payload window (words per warp)
};
void decode_begin(hpdr_ctx *ctx, const DecodeJob &job, DecodeSession &S, cudaStream_t s, bool copy_payload);
void decode_units(const DecodeSession &S, int64_t u_lo, int64_t u_hi, bool streamed, cudaStream_t s, int redo = 0);
void decode_end(hpdr_ctx *ctx, const DecodeSession &S, DecodeResult &res, cudaStream_t s, bool streamed);

// Fill n keys / coefficients with one symbol (single-key stream, huffman.py:423-426).
void fill_single(uint32_t *keys, double *coef, int64_t n, uint32_t sym, double bin_width, cudaStream_t s);

// ---- quantize.py:110-117 -----------------------------------------------------------
// coef[idx] = bins * bin_width; returns HPDR_ERR_INDEX on out-of-range indices.
int scatter_outliers(hpdr_ctx *ctx, double *coef, int64_t n, const uint64_t *h_idx, const int64_t *h_bins,
                     uint64_t n_out, double bin_width, cudaStream_t s);

}  // namespace hpdr
