/* mgard_oracle.h -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * HPDR MGARD path used as the parity checker.  See mgard_oracle.c. */
#ifndef MGARD_ORACLE_H
#define MGARD_ORACLE_H
#include <stdint.h>

enum { ORC_OK = 0, ORC_VALIDATION = 1, ORC_CORRUPT = 2, ORC_ALLOC = 3, ORC_INDEX = 5, ORC_OVERFLOW = 6 };
enum { ORC_F32 = 0, ORC_F64 = 1 };

void orc_set_threads(int n);
int orc_get_threads(void);
int orc_hierarchy(int rank, const uint64_t *dims, int *L, uint64_t *counts);
int orc_axis_tables(int rank, const uint64_t *dims, int step, int axis, uint64_t *n, uint64_t *nc, double *t,
                    double *ml, double *md, double *mu, double *tw, double *tb, double *tu);
int orc_coarsest_indices(int rank, const uint64_t *dims, uint64_t *out, uint64_t *n);
int orc_decompose(const void *in, int dtype, int rank, const uint64_t *dims, double *coef, double *vmin, double *vmax);
int orc_recompose(const double *coef, int rank, const uint64_t *dims, double *out);
int orc_quantize(const double *coef, int rank, const uint64_t *dims, double u_min, double u_max,
                 double eb_rel, uint32_t dict_size, int has_range, double r0, double r1,
                 uint32_t *keys, uint64_t *outlier_idx, int64_t *outlier_bins, uint64_t *n_out,
                 double *coarse_vals, uint64_t *n_coarse, double *eb_abs, double *bin, int *levels);
int orc_dequantize(const uint32_t *keys, uint64_t nkeys, int rank, const uint64_t *dims, uint32_t dict_size,
                   double bin, const uint64_t *oidx, const int64_t *obins, uint64_t n_out,
                   const double *coarse_vals, uint64_t n_coarse, double *coef);
int orc_histogram(const uint32_t *keys, uint64_t n, uint32_t dict_size, int64_t *counts);
int orc_canonical_codes(const uint8_t *lengths, uint32_t dict_size, uint32_t *codes);
int orc_build_codebook(const int64_t *counts, uint32_t dict_size, uint8_t *lengths, uint32_t *codes);
uint64_t orc_huffman_bound(uint64_t n, uint32_t dict_size);
int orc_huffman_compress(const uint32_t *keys, uint64_t n, uint32_t dict_size, uint8_t *out, uint64_t cap, uint64_t *len);
int orc_huffman_decompress(const uint8_t *in, uint64_t len, uint32_t *keys, uint64_t cap, uint64_t *n, int64_t *bit_off);
int orc_mgard_compress(const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel, uint32_t dict_size,
                       int has_range, double r0, double r1, uint8_t **blob, uint64_t *blob_len);
int orc_mgard_decompress(const uint8_t *blob, uint64_t len, void *out, uint64_t out_cap,
                         int *dtype, int *rank, uint64_t *dims, int64_t *bit_off);
void orc_free(void *p);
/* fixed-rate block coder (zfp_oracle.c; hpdr/zfp.py) */
int orz_compressed_size(int dtype, int rank, const uint64_t *dims, int rate, uint64_t *size);
int orz_compress(const void *in, int dtype, int rank, const uint64_t *dims, int rate, uint8_t *out, uint64_t cap,
                 uint64_t *len);
int orz_peek(const uint8_t *in, uint64_t len, int *dtype, int *rank, uint64_t *dims, int *rate);
int orz_decompress(const uint8_t *in, uint64_t len, void *out, uint64_t out_cap);
#endif
