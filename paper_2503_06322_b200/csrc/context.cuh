// context.cuh -- persistent per-device context (the reference's CMM, context.py:22-146):
// device work buffers, pinned staging, streams, per-dims operator tables and an
// allocation counter.  Buffers grow but are never freed between calls, so repeated
// reductions of the same shape allocate nothing after warm-up.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "plan.hpp"

namespace hpdr {

// Device-side view of the tables of one (transition, axis).
struct DevAxis {
    int active;
    int32_t n, nc;
    const int32_t *pa, *pb;
    const double *pt;
    const int32_t *fa, *fb;
    const int32_t *r0, *rr, *rl;
    const double *wr, *wl;
    const double *ml, *md, *mu;
    const double *tw, *tb, *tu, *tr;
    const PlaneInfo *pi;
};

struct DevStep {
    Shape4 fsh, csh;
    DevAxis ax[4];
};

constexpr int kMaxLevels = 40;

struct DevPlan {
    HostPlan host;
    std::vector<DevStep> steps;
    const int32_t *map[4][kMaxLevels];   // device copies of the index maps
    const long long *coarsest = nullptr; // device copy of host.coarsest (<= 16 flat indices)
    void *dbuf = nullptr;
    size_t bytes = 0;
    Shape4 dims;
    int64_t n_total = 0;
    std::vector<int64_t> level_size;     // dense node count of level k (k = 0 finest)
    std::vector<int64_t> level_off;      // offset of level k >= 1 in the coarse-level arena
    int64_t coarse_arena = 0;            // sum of level sizes k >= 1
    // CUDA graphs of the coarse-level chain, keyed by the buffers / scalars baked into the launches
    struct Graph {
        std::vector<uintptr_t> key;
        cudaGraphExec_t exec = nullptr;
        size_t kernels = 0;
    };
    std::vector<Graph> graphs;
    bool graph_warm = false;             // one direct run first (static kernel attributes are set)
    ~DevPlan() {
        for (auto &g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
    }
};

struct Buffer {
    void *ptr = nullptr;
    size_t bytes = 0;
};

struct hpdr_ctx_impl;

// Event families: each purpose indexes its own pool, so a per-slab / per-chunk index can never
// alias another family's event (e.g. a 600-slab decompress vs the staging ring's slots).
enum EvNs : int {
    EvFixed = 0,    // single-purpose events, small fixed ids
    EvChunkIn,      // streamed decompose: H2D of input chunk k landed
    EvSlabOut,      // recompose: output slab k written (its D2H may start)
    EvStageIn,      // pinned H2D staging ring slot
    EvStageOut,     // pinned D2H staging ring slot
    EvEncGroup,     // Huffman encode unit group g packed
    EvDecIn,        // streamed decode: payload group g landed
    EvDecCorr,      // streamed decode: group g decoded (finest correction may proceed)
    EvLevel,        // recompose: correction of level l computed on a side stream
    EvPipeCoef,     // pipeline: chunk k's coefficients ready
    EvZfpIn,        // fixed-rate host path: input slab k landed
    EvZfpOut,       // fixed-rate host path: slab k coded
    EvZfpDecIn,     // fixed-rate decode host path: stream slab k landed
    EvZfpDecOut,    // fixed-rate decode host path: output slab k written
    EvNsCount
};

}  // namespace hpdr

struct hpdr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;    // compute
    cudaStream_t h2d = nullptr;       // copy engine 0
    cudaStream_t d2h = nullptr;       // copy engine 1
    cudaStream_t aux = nullptr;       // side compute off the critical path (low priority)
    cudaStream_t aux_hi = nullptr;    // side compute on the critical path (the finest correction of a decompress)
    cudaStream_t side[4] = {};        // more side streams (independent per-level corrections)
    uint64_t alloc_events = 0;
    hpdr_range_hook range_hook = nullptr;   // job-wide range exchange (hpdr_ctx_set_range_hook)
    void *range_user = nullptr;
    std::map<std::string, hpdr::Buffer> dev;      // named device buffers (grow-only)
    std::map<std::string, hpdr::Buffer> pinned;   // named pinned host buffers (grow-only)
    std::map<std::vector<uint64_t>, std::unique_ptr<hpdr::DevPlan>> plans;
    std::vector<std::vector<uint64_t>> plan_lru;

    // result of the last hpdr_mgard_compress / hpdr_huffman_compress, for fetch
    struct Pending {
        bool valid = false;
        std::vector<uint8_t> head;       // host bytes up to (excluding) the outlier arrays
        uint64_t n_out = 0;
        std::vector<uint8_t> mid;        // n_coarse + coarse values + huffman header up to offsets
        uint64_t n_units = 0;
        uint64_t total_bits = 0;
        uint64_t total_len = 0;
        bool single_key = false;
        bool huffman_only = false;
        int slot = 0;                    // which output buffer set holds the device parts
        bool fetched = false;            // already streamed to the caller's buffer by compress
    } pending;

    // Compress outputs (outliers, unit offsets, packed words) live in one of two buffer sets so
    // the pipeline can copy chunk k out while chunk k+1 is being reduced.
    int out_slot = 0;
    // CUDA-graph replays of the coarse levels; off while several host threads drive contexts of the
    // same device (a capture in one thread forbids device-wide synchronisation in the others)
    bool graphs_ok = true;
    unsigned stage_next = 0;   // next slot of the pinned H2D staging ring (stage_h2d)
    std::string oname(const char *base, int slot) const { return slot ? std::string(base) + "#1" : std::string(base); }
    std::string oname(const char *base) const { return oname(base, out_slot); }

    std::vector<cudaEvent_t> events[hpdr::EvNsCount];   // reusable sync events (no timing), per family
    // Extra queue contexts of the streams pipeline (paper Fig. 7's queues): each has its own
    // streams, buffers and plan cache, and is driven by its own host thread.  Owned.
    std::vector<hpdr_ctx *> queues;
    hpdr_ctx *queue(int q);   // q = 0: this context
    cudaEvent_t event(hpdr::EvNs ns, size_t i);
    cudaEvent_t event(size_t i) { return event(hpdr::EvFixed, i); }

    void *dbuf(const std::string &name, size_t bytes);
    void *hbuf(const std::string &name, size_t bytes);
    hpdr::DevPlan &plan(int rank, const uint64_t *dims);
    void sync();
    void sync_all();   // every stream of this context (buffer reuse / reallocation)
};

namespace hpdr {
// Pointer classification (cudaPointerGetAttributes).
enum class MemKind { Host, Pinned, Device };
MemKind classify(const void *p);
void copy_to_device(hpdr_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t s);
// Stream-ordered small copy (<= 1 MB) done by an SM instead of a copy engine, between device memory
// and/or pinned host memory (UVA): it does not queue behind bulk H2D / D2H transfers in flight on the
// copy engines (the pipeline's chunk copies), which would otherwise delay every host readback of a
// histogram or flag by up to a whole chunk transfer.  Pageable or large copies use cudaMemcpyAsync.
void small_copy(void *dst, const void *src, size_t bytes, cudaStream_t s);
// cudaMemsetAsync(dst, 0, bytes) as a kernel (same reason as small_copy; any size, 16-byte stores).
void zero_async(void *dst, size_t bytes, cudaStream_t s);
// Pageable host memory (plain numpy arrays, Python bytes) moves through pinned staging rings at
// full PCIe speed instead of the driver's slow pageable path: host-side copies are split across
// threads and overlap the DMA of the previous slot.
//   stage_h2d: returns once every DMA is issued on st (the last slots may still be in flight);
//   stage_d2h: DMA on st after its prior work, returns when dst holds the data.
void parallel_memcpy(void *dst, const void *src, size_t n);
void stage_h2d(hpdr_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t st);
void stage_d2h(hpdr_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t st);
// Byte ranges [lo, hi) of src -> dst (pageable), each released by its event, through one
// continuous pass of the pinned staging ring.
struct StageRange {
    size_t lo, hi;
    cudaEvent_t ready;
};
void stage_d2h_ranges(hpdr_ctx *ctx, char *dst, const char *src, const std::vector<StageRange> &ranges,
                      cudaStream_t st);
// Store one 8-byte value to device memory in stream order (a kernel parameter, no staging copy).
void store_u64(void *dst, uint64_t v, cudaStream_t s);
// Relative mode: pass this block's min / max through the context's range hook (if any).
void apply_range_hook(hpdr_ctx *ctx, double *vmin, double *vmax);
void copy_from_device(hpdr_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t s);
}  // namespace hpdr
