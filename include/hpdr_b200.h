/*
 * hpdr_b200.h -- C ABI of the B200-native MGARD reduction path.
 *
 * This is the drop-in boundary for the reference's codec-level entry points
 * (the reference is pure Python, so its "FFI" is the ctypes binding shown in
 * INTEGRATION.md).  Every entry point below names the reference function it
 * replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - dims are listed slowest-varying first (row-major), rank 1..4
 *     (hpdr/exec_core/tensor.py:63-106).
 *   - dtype codes are the reference's on-disk codes (tensor.py:51-60):
 *     0 = F32, 1 = F64, 2 = U32, 3 = U64, 4 = I32, 5 = I64, 6 = U8.
 *   - Host buffers may be pageable or pinned; device pointers (from any
 *     allocator on the context's device) are detected with
 *     cudaPointerGetAttributes and used in place.
 *   - Return codes map 1:1 onto the reference's exception classes
 *     (hpdr/errors.py:4-33); the message and CorruptStreamError.bit_offset
 *     come from hpdr_last_error() (thread-local).
 *   - A context is owned by one host thread at a time.
 */
#ifndef HPDR_B200_H
#define HPDR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPDR_OK              0
#define HPDR_ERR_VALIDATION  1  /* hpdr.errors.ValidationError (errors.py:8)   */
#define HPDR_ERR_CORRUPT     2  /* hpdr.errors.CorruptStreamError (errors.py:20) */
#define HPDR_ERR_ALLOCATION  3  /* hpdr.errors.AllocationError (errors.py:16)   */
#define HPDR_ERR_CUDA        4  /* CUDA runtime failure (no reference analogue) */
#define HPDR_ERR_INDEX       5  /* IndexError: outlier index out of range (quantize.py:113) */
#define HPDR_ERR_OVERFLOW    6  /* OverflowError: canonical code leaves uint32 (huffman.py:201) */
#define HPDR_ERR_VALUE       7  /* ValueError: coarse-value broadcast mismatch (quantize.py:117) */
#define HPDR_ERR_BUFFER      8  /* caller-supplied buffer too small            */
#define HPDR_ERR_FORMAT      9  /* hpdr.errors.FormatError: bad container (errors.py:32) */

typedef struct hpdr_ctx hpdr_ctx;

/* ---- persistent device context: the CMM analogue (hpdr/exec_core/context.py:22-146) ---- */
int      hpdr_ctx_create(int device, hpdr_ctx **out);
void     hpdr_ctx_destroy(hpdr_ctx *ctx);
/* Context.alloc_events (context.py:58): device/pinned allocations made so far. */
uint64_t hpdr_ctx_alloc_events(const hpdr_ctx *ctx);
int      hpdr_ctx_device(const hpdr_ctx *ctx);
/* Release cached device buffers (keeps the context usable). */
void     hpdr_ctx_trim(hpdr_ctx *ctx);

/* Job-wide value range for block-partitioned compression (the multi-GPU path
 * of SURVEY 8(e)).  In relative mode (has_range = 0) hpdr_mgard_compress calls hook(user, &vmin,
 * &vmax) on the calling host thread once this block's min / max are known -- after the
 * range-independent decomposition of a streamed host input has been issued, before anything is
 * quantized -- and compresses with the values the hook leaves there, exactly as
 * mgard_compress(block, eb_rel, value_range=(vmin, vmax)) (quantize.py:66, codec.py:47-48).  A
 * rank-per-GPU job puts its min/max all-reduce (16 bytes) here, so the exchange overlaps the
 * input transfer instead of costing an extra pass over the field.  A non-zero return fails the
 * call with HPDR_ERR_VALIDATION.  hook = NULL removes it. */
typedef int (*hpdr_range_hook)(void *user, double *vmin, double *vmax);
void     hpdr_ctx_set_range_hook(hpdr_ctx *ctx, hpdr_range_hook hook, void *user);

/* Thread-local error message of the last failing call; *bit_offset receives
 * CorruptStreamError.bit_offset (-1 when unknown), may be NULL. */
const char *hpdr_last_error(int64_t *bit_offset);

/* Pinned host memory (cudaHostAlloc) for zero-staging transfers. */
void    *hpdr_host_alloc(uint64_t bytes);
/* Host memcpy split across the library's copy threads (large results into Python-owned memory). */
void     hpdr_host_copy(void *dst, const void *src, uint64_t n);
void     hpdr_host_free(void *p);
/* First-touch a fresh pageable buffer on background threads (zero-filling it, huge pages where the
 * kernel allows); returns a handle for hpdr_host_prefault_wait, which must return before anything
 * else writes the buffer. */
void    *hpdr_host_prefault_begin(void *p, uint64_t bytes);
void     hpdr_host_prefault_wait(void *handle);
/* Page-lock an existing host range (cudaHostRegister, portable) so transfers DMA straight from /
 * to it; returns HPDR_ERR_ALLOCATION on failure.  A range that is already registered is OK. */
int      hpdr_host_register(void *p, uint64_t bytes);
void     hpdr_host_unregister(void *p);

/* ---- whole-path entry points: hpdr/mgard/codec.py ---- */

/* mgard_compress (codec.py:25-56).  Runs the full reduction and keeps the
 * result in the context; *blob_len receives the exact blob size.  Copy the
 * blob out with hpdr_mgard_fetch.  If out != NULL and out_cap >= blob size,
 * the blob is also written to out in the same call (one-shot path). */
int hpdr_mgard_compress(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims,
                        double eb_rel, uint32_t dict_size, int has_range, double range_min,
                        double range_max, void *out, uint64_t out_cap, uint64_t *blob_len);
/* Copy the last compressed blob into out (host or device pointer). */
int hpdr_mgard_fetch(hpdr_ctx *ctx, void *out, uint64_t out_cap);

/* Destination allocator: a writable buffer of `bytes` (pageable or pinned host, or device), or
 * NULL on failure. */
typedef void *(*hpdr_alloc_fn)(void *user, uint64_t bytes);
/* mgard_compress (codec.py:25-56) into a buffer the caller allocates through alloc(user, size)
 * as soon as the blob size is known (the codebook fixes it, before the payload is packed); the
 * blob then streams into it behind the encode launches.  alloc is called exactly once on
 * success.  Replaces the compress + fetch pair for callers that must own a fresh result object
 * (the reference returns a new `bytes`). */
int hpdr_mgard_compress_alloc(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims,
                              double eb_rel, uint32_t dict_size, int has_range, double range_min,
                              double range_max, hpdr_alloc_fn alloc, void *user, uint64_t *blob_len);

/* Parse the blob header: dtype code, rank and dims (codec.py:62-84). */
int hpdr_mgard_peek(const void *blob, uint64_t len, int *dtype, int *rank, uint64_t *dims);

/* mgard_decompress (codec.py:59-113).  out receives prod(dims) values of the
 * blob's dtype (host or device pointer). */
int hpdr_mgard_decompress(hpdr_ctx *ctx, const void *blob, uint64_t len, void *out, uint64_t out_bytes);

/* ---- overlapped host<->device pipeline ----
 * The field is split into dim-0 chunks of chunk_planes planes (0: ~64 MB), or into the explicit
 * plane counts chunk_list[0..n_list) (the adaptive schedule of Algorithm 4); each chunk becomes a
 * reference-identical MGARD blob compressed with the global value range (computed on the host
 * when has_range is 0), written into an HPDR container.  H2D of chunk k+1 and D2H of chunk k-1
 * overlap the reduction of chunk k (two input buffers, two output sets, Fig. 7 reuse edges).
 * trace (nullable) receives 6 doubles per chunk: H2D, compute, D2H start/end in ms. */
int hpdr_pipeline_compress(hpdr_ctx *ctx, const void *host_in, int dtype, int rank, const uint64_t *dims,
                           double eb_rel, uint32_t dict_size, int has_range, double range_min,
                           double range_max, uint64_t chunk_planes, const uint64_t *chunk_list,
                           uint64_t n_list, void *out, uint64_t out_cap, uint64_t *out_len,
                           double *trace);
int hpdr_pipeline_decompress(hpdr_ctx *ctx, const void *container, uint64_t len, void *out,
                             uint64_t out_bytes, double *trace);

/* Global min/max of a field (transform.py:304-305 u.values.min()/max(); NaN propagates).
 * Used to agree on one value_range across slabs / ranks before quantization. */
int hpdr_minmax(hpdr_ctx *ctx, const void *in, int dtype, uint64_t n, double *vmin, double *vmax);

/* ---- stage entry points (for parity tests; each mirrors one reference function) ---- */

/* decompose (transform.py:287-323): fp64 coefficients in finest-grid order. */
int hpdr_decompose(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims,
                   double *coef_out, double *u_min, double *u_max);
/* recompose (transform.py:326-348). */
int hpdr_recompose(hpdr_ctx *ctx, const double *coef, int rank, const uint64_t *dims, double *out);
/* quantize (quantize.py:50-98).  Buffers: keys[N], outlier_idx/bins[N] (worst
 * case), coarse[16].  Returns counts through the pointers. */
int hpdr_quantize(hpdr_ctx *ctx, const double *coef, int rank, const uint64_t *dims, double u_min,
                  double u_max, double eb_rel, uint32_t dict_size, int has_range, double range_min,
                  double range_max, uint32_t *keys, uint64_t *outlier_idx, int64_t *outlier_bins,
                  uint64_t *n_outliers, double *coarse, uint64_t *n_coarse, double *eb_abs,
                  double *bin_width, uint32_t *levels);
/* dequantize (quantize.py:101-125): keys + outliers + coarse values -> coefficients. */
int hpdr_dequantize(hpdr_ctx *ctx, const uint32_t *keys, uint64_t n_keys, int rank, const uint64_t *dims,
                    uint32_t dict_size, double bin_width, const uint64_t *outlier_idx,
                    const int64_t *outlier_bins, uint64_t n_outliers, const double *coarse,
                    uint64_t n_coarse, double *coef_out);
/* histogram (huffman.py:74-104). */
int hpdr_histogram(hpdr_ctx *ctx, const uint32_t *keys, uint64_t n, uint32_t dict_size, int64_t *counts);
/* build_codebook (huffman.py:160-185), host-side. */
int hpdr_build_codebook(const int64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes);
/* huffman_compress (huffman.py:366-396): two-phase like hpdr_mgard_compress. */
int hpdr_huffman_compress(hpdr_ctx *ctx, const uint32_t *keys, uint64_t n, uint32_t dict_size,
                          uint64_t *stream_len);
int hpdr_huffman_fetch(hpdr_ctx *ctx, void *out, uint64_t out_cap);
/* huffman_decompress (huffman.py:399-435).  *n receives the symbol count;
 * keys may be NULL to query it (returns HPDR_ERR_BUFFER when cap < n). */
int hpdr_huffman_decompress(hpdr_ctx *ctx, const void *in, uint64_t len, uint32_t *keys,
                            uint64_t cap, uint64_t *n);

/* ---- fixed-rate block coder: hpdr/zfp.py ---- */

/* compressed_size (zfp.py:270-278): exact stream bytes for (dtype, dims, rate). */
int hpdr_zfp_compressed_size(int dtype, int rank, const uint64_t *dims, uint32_t rate, uint64_t *size);
/* zfp_compress (zfp.py:281-308): rank 1..3 F32/F64 field -> "<BBB" rank, dtype, rate | dims u64 x rank |
 * packed blocks of 1 + e_bits + rate*4^rank bits.  *out_len receives the stream size; out_cap smaller
 * than that returns HPDR_ERR_BUFFER (so out = NULL queries the size). */
int hpdr_zfp_compress(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, uint32_t rate,
                      void *out, uint64_t out_cap, uint64_t *out_len);
/* Header of a fixed-rate stream with zfp_decompress's checks (zfp.py:314-334). */
int hpdr_zfp_peek(const void *stream, uint64_t len, int *dtype, int *rank, uint64_t *dims, uint32_t *rate);
/* zfp_decompress (zfp.py:311-353): out receives prod(dims) values of the stored dtype. */
int hpdr_zfp_decompress(hpdr_ctx *ctx, const void *stream, uint64_t len, void *out, uint64_t out_bytes);
/* run_pipeline with the fixed-rate reducer: dim-0 chunks (chunk_planes, default
 * ~64 MB in whole 4-plane rows, or the explicit chunk_list), each an independent zfp_compress stream of
 * its slab, in an HPDR container with pipeline id 1 (params: rate u8).  Decompress with
 * hpdr_pipeline_decompress (it dispatches on the pipeline id).  trace as hpdr_pipeline_compress. */
int hpdr_pipeline_zfp_compress(hpdr_ctx *ctx, const void *host_in, int dtype, int rank, const uint64_t *dims,
                               uint32_t rate, uint64_t chunk_planes, const uint64_t *chunk_list, uint64_t n_list,
                               void *out, uint64_t out_cap, uint64_t *out_len, double *trace);

/* Kernel launches issued by this thread since the last reset (bench accounting). */
uint64_t hpdr_launch_count(int reset);
/* Live per-kernel CUDA-event timing with algorithmic bytes (bench roofline).  on = 1: events on
 * the launching stream (kernels on side streams may overlap); on = 2: serialized, the device is
 * synchronized before and after every profiled launch (per-kernel times that add up).  Enabling
 * clears previous records; hpdr_prof_read writes {"kernel": [launches, total_ms,
 * total_bytes, max_ms], ...} as JSON and clears. */
void     hpdr_prof_enable(int on);
int      hpdr_prof_read(char *json, uint64_t cap);
/* The context's compute stream (cudaStream_t) for external event timing. */
void    *hpdr_ctx_stream(const hpdr_ctx *ctx);
/* Diagnostics: checks the Thomas sweeps' verified fast division against __ddiv_rn on n
 * pseudo-random operand pairs (device 0 / current device).  *mismatches must be 0. */
int      hpdr_selftest_div(uint64_t n, uint64_t seed, uint64_t *mismatches, uint64_t *fallbacks);

#ifdef __cplusplus
}
#endif
#endif /* HPDR_B200_H */
