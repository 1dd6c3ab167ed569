// common.cuh -- shared definitions for the B200 MGARD reduction library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "error.hpp"
#include "hpdr_b200.h"

namespace hpdr {

constexpr int kMaxRank = 4;
constexpr int kBlockSymbols = 4096;   // huffman.py:29 encode block = decode unit
constexpr int kMaxCodeLen = 32;       // huffman.py:30
constexpr int kMaxDict = 65535;       // huffman.py:31
constexpr int kLutBits = 12;          // decode fast-path table width
constexpr int kNumSMs = 148;

void set_error(int code, const std::string &msg, int64_t bit_offset = -1);
void count_launch();
void debug_sync(const char *where);
// HPDR_PHASES=1: CUDA-event phase marks on a stream, printed (ms since the first mark) by phase_dump.
void phase_mark(const char *name, cudaStream_t s);
bool prof_enabled();
void count_launches(uint64_t n);
void phase_dump(const char *title);   // HPDR_DEBUG_SYNC=1: device sync + check after every launch

// Live per-kernel timing for bench.py: when enabled (hpdr_prof_enable), each scope records a
// CUDA event pair on the launching stream plus the launch's algorithmic bytes.
struct ProfScope {
    ProfScope(const char *name, double bytes, cudaStream_t s);
    ~ProfScope();
    int slot;
    cudaStream_t stream;
};
#define KPROF(name, bytes, stream) ::hpdr::ProfScope prof_scope_(name, (double)(bytes), stream)

#define HPDR_THROW(code, msg) throw ::hpdr::Error{(code), (msg), -1}
#define CUDA_CHECK(x)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            throw ::hpdr::Error{HPDR_ERR_CUDA,                                             \
                                std::string(#x) + ": " + cudaGetErrorString(e_), -1};      \
        }                                                                                  \
    } while (0)
#define HPDR_STR2(x) #x
#define HPDR_STR(x) HPDR_STR2(x)
#define LAUNCH_CHECK()                                                                     \
    do {                                                                                   \
        ::hpdr::count_launch();                                                            \
        CUDA_CHECK(cudaGetLastError());                                                    \
        ::hpdr::debug_sync(__FILE__ ":" HPDR_STR(__LINE__));                               \
    } while (0)

// 4-D shape, slowest first; lower ranks are padded with leading 1s.
struct Shape4 {
    int64_t n[4];
    __host__ __device__ int64_t size() const { return n[0] * n[1] * n[2] * n[3]; }
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- cp.async (LDGSTS) helpers: asynchronous global -> shared copies for prefetch rings ----
template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}
// Same with a precomputed 32-bit shared-window address.
template <int BYTES>
__device__ __forceinline__ void cp_async_s(unsigned saddr, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(saddr), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

inline unsigned grid_for(int64_t work, int threads, int64_t cap = 148LL * 32) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

}  // namespace hpdr
