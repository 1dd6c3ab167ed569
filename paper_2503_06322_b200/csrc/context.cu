// context.cu -- device context, buffer pool, operator-table upload, error state.
#include <string.h>

#include <algorithm>
#include <atomic>
#include <sched.h>
#include <sys/mman.h>

#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "context.cuh"

namespace hpdr {

static thread_local std::string tl_msg;
static thread_local int64_t tl_bit = -1;
static std::atomic<uint64_t> g_launches{0};   // all threads (pipeline queue workers included)

void set_error(int code, const std::string &msg, int64_t bit_offset) {
    (void)code;
    tl_msg = msg;
    tl_bit = bit_offset;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void debug_sync(const char *where) {
    static const bool on = getenv("HPDR_DEBUG_SYNC") != nullptr;
    if (!on) return;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) throw Error{HPDR_ERR_CUDA, std::string("kernel at ") + where + ": " + cudaGetErrorString(e), -1};
}

// ---- phase marks ----
namespace {
std::mutex g_ph_mu;
std::vector<std::pair<const char *, cudaEvent_t>> g_ph;
bool phases_on() {
    static const bool on = getenv("HPDR_PHASES") != nullptr;
    return on;
}
}  // namespace

void phase_mark(const char *name, cudaStream_t s) {
    if (!phases_on()) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    std::lock_guard<std::mutex> g(g_ph_mu);
    g_ph.push_back({name, e});
}

void phase_dump(const char *title) {
    if (!phases_on()) return;
    std::lock_guard<std::mutex> g(g_ph_mu);
    if (g_ph.empty()) return;
    cudaDeviceSynchronize();
    fprintf(stderr, "[phases] %s:", title);
    for (auto &pe : g_ph) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_ph[0].second, pe.second);
        fprintf(stderr, " %s=%.3f", pe.first, ms);
    }
    fprintf(stderr, "\n");
    for (auto &pe : g_ph) cudaEventDestroy(pe.second);
    g_ph.clear();
}

// ---- live kernel profiling ----
namespace {
struct ProfRec {
    const char *name;
    double bytes;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
bool g_prof_serial = false;   // mode 2: the device is idle before and after every profiled launch
std::vector<ProfRec> g_prof;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_pool;
size_t g_prof_used = 0;
}  // namespace

bool prof_enabled() { return g_prof_on; }

ProfScope::ProfScope(const char *name, double bytes, cudaStream_t s) : slot(-1), stream(s) {
    if (!g_prof_on) return;
    if (g_prof_serial) cudaDeviceSynchronize();   // no other kernel overlaps this one
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (g_prof_used == g_prof_pool.size()) {
        cudaEvent_t a, b;
        if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) { cudaGetLastError(); return; }
        g_prof_pool.push_back({a, b});
    }
    auto ev = g_prof_pool[g_prof_used++];
    g_prof.push_back(ProfRec{name, bytes, ev.first, ev.second});
    slot = (int)g_prof.size() - 1;
    cudaEventRecord(ev.first, s);
}

ProfScope::~ProfScope() {
    if (slot < 0) return;
    {
        std::lock_guard<std::mutex> g(g_prof_mu);
        if (slot < (int)g_prof.size()) cudaEventRecord(g_prof[slot].b, stream);
    }
    if (g_prof_serial) cudaDeviceSynchronize();
}

MemKind classify(const void *p) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return MemKind::Host;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        // every entry point runs with the context's device current: a buffer of another GPU
        // would be read / written through the wrong device's kernels
        int cur = -1;
        if (a.type == cudaMemoryTypeDevice && cudaGetDevice(&cur) == cudaSuccess && a.device != cur)
            throw Error{HPDR_ERR_VALIDATION,
                        "device buffer is on GPU " + std::to_string(a.device) + " but the context is on GPU " +
                            std::to_string(cur), -1};
        return MemKind::Device;
    }
    if (a.type == cudaMemoryTypeHost) return MemKind::Pinned;
    return MemKind::Host;
}

namespace {
__global__ void k_small_copy(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src, size_t n) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)dst | (uintptr_t)src) & 7) == 0) {
        const size_t nw = n / 8;
        for (size_t i = tid; i < nw; i += nt) reinterpret_cast<uint64_t *>(dst)[i] = reinterpret_cast<const uint64_t *>(src)[i];
        for (size_t i = nw * 8 + tid; i < n; i += nt) dst[i] = src[i];
    } else {
        for (size_t i = tid; i < n; i += nt) dst[i] = src[i];
    }
}
__global__ void k_store_u64(uint64_t *dst, uint64_t v) { *dst = v; }
__global__ void k_zero(uint8_t *__restrict__ dst, size_t n) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    const size_t al = (16 - ((uintptr_t)dst & 15)) & 15, head = al < n ? al : n;
    for (size_t i = tid; i < head; i += nt) dst[i] = 0;
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
    const size_t n4 = (n - head) / 16;
    for (size_t i = tid; i < n4; i += nt) d4[i] = uint4{0, 0, 0, 0};
    for (size_t i = head + n4 * 16 + tid; i < n; i += nt) dst[i] = 0;
}
}  // namespace

void small_copy(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    // an SM copy beats a DMA launch for small pieces; across PCIe (pinned host memory) only up to
    // ~128 KB -- zero-copy reads by a few blocks are latency-bound beyond that
    const MemKind kd = classify(dst), ks = classify(src);
    const size_t cap = (kd == MemKind::Pinned || ks == MemKind::Pinned) ? (128u << 10) : (1u << 20);
    if (bytes > cap || kd == MemKind::Host || ks == MemKind::Host) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
        return;
    }
    const unsigned grid = (unsigned)std::min<size_t>(64, (bytes / 8 + 255) / 256 + 1);
    k_small_copy<<<grid, 256, 0, s>>>((uint8_t *)dst, (const uint8_t *)src, bytes);
    LAUNCH_CHECK();
}

void zero_async(void *dst, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    const unsigned grid = (unsigned)std::min<size_t>(148 * 8, (bytes / 16 + 255) / 256 + 1);
    k_zero<<<grid, 256, 0, s>>>((uint8_t *)dst, bytes);
    LAUNCH_CHECK();
}

namespace {
constexpr size_t kStageChunk = 32u << 20;   // 2 MB per copy thread
constexpr unsigned kStageSlots = 4;
// Host copy threads of this process: HPDR_COPY_THREADS, else the CPUs this process may run on
// (its affinity mask -- a rank bound to its GPU's NUMA node sees that node's CPUs) divided among
// the ranks sharing them (HPDR_RANKS_PER_NUMA, set by numa.bind_to_gpu), at most 16.
int host_threads() {
    static const int t = [] {
        if (const char *e = getenv("HPDR_COPY_THREADS")) return std::max(1, std::min(64, atoi(e)));
        int cpus = (int)std::thread::hardware_concurrency();
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) cpus = CPU_COUNT(&set);
        int share = 1;
        if (const char *e = getenv("HPDR_RANKS_PER_NUMA")) share = std::max(1, atoi(e));
        return std::max(1, std::min(16, cpus / share));
    }();
    return t;
}
}  // namespace

namespace {
// A persistent pool of memcpy workers (spawning threads per 16 MB slot costs more than the copy).
struct CopyPool {
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::vector<std::thread> th;
    char *dst = nullptr;
    const char *src = nullptr;
    size_t n = 0, per = 0, align = 4096;
    // slice boundary k (0..workers+1): on a page boundary of the destination, so every (huge) page
    // of a fresh destination is first touched -- and faulted in -- by exactly one thread
    size_t cut(int k) const {
        if (k >= workers + 1) return n;
        const uintptr_t b = (uintptr_t)dst, t = (b + (size_t)k * per + align - 1) & ~(uintptr_t)(align - 1);
        return std::min(n, (size_t)(t - b));
    }
    uint64_t gen = 0;
    int pending = 0, workers = 0;
    bool stop = false;
    explicit CopyPool(int w) : workers(w) {
        for (int i = 0; i < w; i++)
            th.emplace_back([this, i] {
                uint64_t seen = 0;
                for (;;) {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return stop || gen != seen; });
                    if (stop) return;
                    seen = gen;
                    char *d = dst;
                    const char *s = src;
                    const size_t a = cut(i + 1), e = cut(i + 2);
                    lk.unlock();
                    if (a < e) memcpy(d + a, s + a, e - a);
                    lk.lock();
                    if (--pending == 0) done_cv.notify_one();
                }
            });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto &t : th) t.join();
    }
    void copy(void *d, const void *s, size_t nn) {   // one caller at a time (guarded by call_mu)
        std::lock_guard<std::mutex> call(call_mu);
        const int T = workers + 1;
        {
            std::lock_guard<std::mutex> g(mu);
            dst = (char *)d;
            src = (const char *)s;
            n = nn;
            per = (nn + T - 1) / T;
            align = per >= (2u << 20) ? (2u << 20) : 4096;
            pending = workers;
            gen++;
        }
        cv.notify_all();
        memcpy(d, s, cut(1));   // slice 0 on the calling thread
        std::unique_lock<std::mutex> lk(mu);
        done_cv.wait(lk, [&] { return pending == 0; });
    }
    std::mutex call_mu;
};
}  // namespace

void parallel_memcpy(void *dst, const void *src, size_t n) {
    if (n < (4u << 20) || host_threads() == 1) {
        memcpy(dst, src, n);
        return;
    }
    static CopyPool *pool = new CopyPool(host_threads() - 1);   // intentionally leaked (process lifetime)
    pool->copy(dst, src, n);
}

void stage_h2d(hpdr_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t st) {
    char *ring = (char *)ctx->hbuf("stage_in", kStageChunk * kStageSlots);
    for (size_t off = 0; off < n; off += kStageChunk) {
        const unsigned slot = ctx->stage_next++ % kStageSlots;
        cudaEvent_t ev = ctx->event(EvStageIn, slot);
        CUDA_CHECK(cudaEventSynchronize(ev));   // the slot's previous DMA has read it
        const size_t m = std::min(kStageChunk, n - off);
        parallel_memcpy(ring + slot * kStageChunk, (const char *)src + off, m);
        CUDA_CHECK(cudaMemcpyAsync((char *)dst + off, ring + slot * kStageChunk, m, cudaMemcpyHostToDevice, st));
        CUDA_CHECK(cudaEventRecord(ev, st));
    }
}

void stage_d2h_ranges(hpdr_ctx *ctx, char *dst, const char *src, const std::vector<StageRange> &ranges,
                      cudaStream_t st) {
    // one continuous pass through the ring over every range (no drain between ranges); a range's
    // first chunk waits on the range's event, so the copies follow the producer range by range
    char *ring = (char *)ctx->hbuf("stage_out", kStageChunk * kStageSlots);
    struct Chunk {
        size_t off, len;
        cudaEvent_t wait;
    };
    std::vector<Chunk> ch;
    for (const StageRange &r : ranges) {
        if (r.hi > r.lo && r.hi - r.lo >= (8u << 20)) {
            const uintptr_t a = ((uintptr_t)(dst + r.lo) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
            const uintptr_t e = ((uintptr_t)(dst + r.hi)) & ~uintptr_t((2u << 20) - 1);
            if (e > a) madvise((void *)a, e - a, MADV_HUGEPAGE);
        }
        for (size_t o = r.lo; o < r.hi; o += kStageChunk)
            ch.push_back({o, std::min(kStageChunk, r.hi - o), o == r.lo ? r.ready : nullptr});
    }
    size_t issued = 0;
    for (size_t done = 0; done < ch.size(); done++) {
        for (; issued < ch.size() && issued < done + kStageSlots; issued++) {
            const unsigned slot = (unsigned)(issued % kStageSlots);
            if (ch[issued].wait) CUDA_CHECK(cudaStreamWaitEvent(st, ch[issued].wait, 0));
            CUDA_CHECK(cudaMemcpyAsync(ring + slot * kStageChunk, src + ch[issued].off, ch[issued].len,
                                       cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaEventRecord(ctx->event(EvStageOut, slot), st));
        }
        const unsigned slot = (unsigned)(done % kStageSlots);
        CUDA_CHECK(cudaEventSynchronize(ctx->event(EvStageOut, slot)));
        parallel_memcpy(dst + ch[done].off, ring + slot * kStageChunk, ch[done].len);
    }
}

void stage_d2h(hpdr_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t st) {
    char *ring = (char *)ctx->hbuf("stage_out", kStageChunk * kStageSlots);
    if (n >= (8u << 20)) {   // a fresh destination faults page by page: ask for huge pages (advisory)
        const uintptr_t a = ((uintptr_t)dst + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
        const uintptr_t e = ((uintptr_t)dst + n) & ~uintptr_t((2u << 20) - 1);
        if (e > a) madvise((void *)a, e - a, MADV_HUGEPAGE);
    }
    const size_t chunks = (n + kStageChunk - 1) / kStageChunk;
    size_t issued = 0;
    for (size_t done = 0; done < chunks; done++) {
        for (; issued < chunks && issued < done + kStageSlots; issued++) {
            const size_t off = issued * kStageChunk, m = std::min(kStageChunk, n - off);
            const unsigned slot = (unsigned)(issued % kStageSlots);
            CUDA_CHECK(cudaMemcpyAsync(ring + slot * kStageChunk, (const char *)src + off, m, cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaEventRecord(ctx->event(EvStageOut, slot), st));
        }
        const unsigned slot = (unsigned)(done % kStageSlots);
        CUDA_CHECK(cudaEventSynchronize(ctx->event(EvStageOut, slot)));
        const size_t off = done * kStageChunk;
        parallel_memcpy((char *)dst + off, ring + slot * kStageChunk, std::min(kStageChunk, n - off));
    }
}

void apply_range_hook(hpdr_ctx *ctx, double *vmin, double *vmax) {
    if (!ctx->range_hook) return;
    if (ctx->range_hook(ctx->range_user, vmin, vmax) != 0)
        throw Error{HPDR_ERR_VALIDATION, "range hook failed", -1};
}

void store_u64(void *dst, uint64_t v, cudaStream_t s) {
    k_store_u64<<<1, 1, 0, s>>>((uint64_t *)dst, v);
    LAUNCH_CHECK();
}

void copy_to_device(hpdr_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t s) {
    (void)ctx;
    if (!bytes) return;
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
}

void copy_from_device(hpdr_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t s) {
    (void)ctx;
    if (!bytes) return;
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
}

}  // namespace hpdr

using namespace hpdr;

void *hpdr_ctx::dbuf(const std::string &name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buffer &b = dev[name];
    if (b.bytes < bytes) {
        // work queued on any of the context's streams may still use the old buffer
        if (b.ptr) sync_all();
        if (b.ptr) CUDA_CHECK(cudaFree(b.ptr));
        b.ptr = nullptr;
        b.bytes = 0;
        size_t want = bytes + (bytes >> 4);   // slack so slightly larger shapes reuse the buffer
        cudaError_t e = cudaMalloc(&b.ptr, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            e = cudaMalloc(&b.ptr, bytes);
            want = bytes;
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw Error{HPDR_ERR_ALLOCATION, "allocating " + std::to_string(bytes) + " device bytes for '" + name + "'", -1};
        }
        b.bytes = want;
        alloc_events++;
    }
    return b.ptr;
}

void *hpdr_ctx::hbuf(const std::string &name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buffer &b = pinned[name];
    if (b.bytes < bytes) {
        if (b.ptr) sync_all();
        if (b.ptr) CUDA_CHECK(cudaFreeHost(b.ptr));
        b.ptr = nullptr;
        b.bytes = 0;
        cudaError_t e = cudaHostAlloc(&b.ptr, bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw Error{HPDR_ERR_ALLOCATION, "allocating " + std::to_string(bytes) + " pinned bytes for '" + name + "'", -1};
        }
        b.bytes = bytes;
        alloc_events++;
    }
    return b.ptr;
}

void hpdr_ctx::sync() { CUDA_CHECK(cudaStreamSynchronize(stream)); }

void hpdr_ctx::sync_all() {
    for (cudaStream_t x : {stream, h2d, d2h, aux, aux_hi}) CUDA_CHECK(cudaStreamSynchronize(x));
    for (cudaStream_t x : side) CUDA_CHECK(cudaStreamSynchronize(x));
}

hpdr_ctx *hpdr_ctx::queue(int q) {
    if (q == 0) return this;
    while ((int)queues.size() < q) {
        hpdr_ctx *c = nullptr;
        const int rc = hpdr_ctx_create(device, &c);
        if (rc != HPDR_OK) throw Error{rc, "creating a pipeline queue context", -1};
        queues.push_back(c);
    }
    return queues[q - 1];
}

cudaEvent_t hpdr_ctx::event(EvNs ns, size_t i) {
    std::vector<cudaEvent_t> &v = events[ns];
    while (v.size() <= i) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        v.push_back(e);
    }
    return v[i];
}

namespace {

struct Packer {
    std::vector<uint8_t> bytes;
    template <class T>
    size_t put(const std::vector<T> &v) {
        size_t off = (bytes.size() + 15) & ~size_t(15);
        bytes.resize(off + v.size() * sizeof(T));
        if (!v.empty()) memcpy(bytes.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

}  // namespace

DevPlan &hpdr_ctx::plan(int rank, const uint64_t *dims) {
    std::vector<uint64_t> key(dims, dims + rank);
    key.insert(key.begin(), (uint64_t)rank);
    auto it = plans.find(key);
    if (it != plans.end()) {
        plan_lru.erase(std::find(plan_lru.begin(), plan_lru.end(), key));
        plan_lru.push_back(key);
        return *it->second;
    }
    auto dp = std::make_unique<DevPlan>();
    build_host_plan(dp->host, rank, dims);
    HostPlan &h = dp->host;
    if (h.L > kMaxLevels) throw Error{HPDR_ERR_VALIDATION, "too many levels", -1};
    Packer pk;
    struct AxOff { size_t pa, pb, pt, fa, fb, r0, rr, rl, wr, wl, ml, md, mu, tw, tb, tu, tr, pi; };
    std::vector<std::vector<AxOff>> offs(h.steps.size(), std::vector<AxOff>(4));
    for (size_t s = 0; s < h.steps.size(); s++)
        for (int d = 0; d < 4; d++) {
            const AxisTables &a = h.steps[s].ax[d];
            if (!a.active) continue;
            AxOff &o = offs[s][d];
            o.pa = pk.put(a.pa); o.pb = pk.put(a.pb); o.pt = pk.put(a.pt);
            o.fa = pk.put(a.fa); o.fb = pk.put(a.fb);
            o.pi = pk.put(a.pinfo);
            o.r0 = pk.put(a.r0); o.rr = pk.put(a.rr); o.rl = pk.put(a.rl);
            o.wr = pk.put(a.wr); o.wl = pk.put(a.wl);
            o.ml = pk.put(a.ml); o.md = pk.put(a.md); o.mu = pk.put(a.mu);
            o.tw = pk.put(a.tw); o.tb = pk.put(a.tb); o.tu = pk.put(a.tu); o.tr = pk.put(a.tr);
        }
    std::vector<std::vector<size_t>> moff(4, std::vector<size_t>(h.L));
    for (int d = 0; d < 4; d++)
        for (int k = 0; k < h.L; k++) moff[d][k] = pk.put(h.map[d][k]);
    std::vector<long long> co(h.coarsest.begin(), h.coarsest.end());
    const size_t coff = pk.put(co);
    dp->bytes = pk.bytes.size();
    cudaError_t e = cudaMalloc(&dp->dbuf, dp->bytes ? dp->bytes : 16);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error{HPDR_ERR_ALLOCATION, "allocating operator tables", -1};
    }
    alloc_events++;
    // Stream-ordered upload: a plain cudaMemcpy from pageable memory may return before its DMA
    // lands (it is queued on the legacy stream, which the context's non-blocking streams do not
    // wait for), so kernels could read stale tables while a copy engine is busy with a pipeline
    // chunk.  Ordering on the compute stream plus a sync makes the tables visible to every stream.
    CUDA_CHECK(cudaMemcpyAsync(dp->dbuf, pk.bytes.data(), dp->bytes, cudaMemcpyHostToDevice, stream));
    CUDA_CHECK(cudaStreamSynchronize(stream));
    char *base = (char *)dp->dbuf;
    dp->steps.resize(h.steps.size());
    for (size_t s = 0; s < h.steps.size(); s++) {
        DevStep &ds = dp->steps[s];
        for (int d = 0; d < 4; d++) {
            ds.fsh.n[d] = h.steps[s].fsh[d];
            ds.csh.n[d] = h.steps[s].csh[d];
            const AxisTables &a = h.steps[s].ax[d];
            DevAxis &x = ds.ax[d];
            memset(&x, 0, sizeof(x));
            x.active = a.active;
            x.n = (int32_t)a.n;
            x.nc = (int32_t)a.nc;
            if (!a.active) continue;
            const AxOff &o = offs[s][d];
            x.pa = (const int32_t *)(base + o.pa); x.pb = (const int32_t *)(base + o.pb);
            x.pt = (const double *)(base + o.pt);
            x.fa = (const int32_t *)(base + o.fa); x.fb = (const int32_t *)(base + o.fb);
            x.pi = (const PlaneInfo *)(base + o.pi);
            x.r0 = (const int32_t *)(base + o.r0); x.rr = (const int32_t *)(base + o.rr);
            x.rl = (const int32_t *)(base + o.rl);
            x.wr = (const double *)(base + o.wr); x.wl = (const double *)(base + o.wl);
            x.ml = (const double *)(base + o.ml); x.md = (const double *)(base + o.md);
            x.mu = (const double *)(base + o.mu);
            x.tw = (const double *)(base + o.tw); x.tb = (const double *)(base + o.tb);
            x.tu = (const double *)(base + o.tu);
            x.tr = (const double *)(base + o.tr);
        }
    }
    for (int d = 0; d < 4; d++)
        for (int k = 0; k < kMaxLevels; k++) dp->map[d][k] = k < h.L ? (const int32_t *)(base + moff[d][k]) : nullptr;
    dp->coarsest = (const long long *)(base + coff);
    for (int d = 0; d < 4; d++) dp->dims.n[d] = h.dims[d];
    dp->n_total = h.total();
    dp->level_size.resize(h.L);
    dp->level_off.assign(h.L, 0);
    int64_t acc = 0;
    for (int k = 0; k < h.L; k++) {
        dp->level_size[k] = h.cnt[0][k] * h.cnt[1][k] * h.cnt[2][k] * h.cnt[3][k];
        if (k >= 1) {
            dp->level_off[k] = acc;
            acc += (dp->level_size[k] + 31) & ~int64_t(31);
        }
    }
    dp->coarse_arena = acc;
    DevPlan &ref = *dp;
    plans[key] = std::move(dp);
    plan_lru.push_back(key);
    while (plan_lru.size() > 8) {   // bounded table cache
        auto victim = plan_lru.front();
        plan_lru.erase(plan_lru.begin());
        auto v = plans.find(victim);
        if (v != plans.end()) {
            cudaFree(v->second->dbuf);
            plans.erase(v);
        }
    }
    return ref;
}

extern "C" {

const char *hpdr_last_error(int64_t *bit_offset) {
    if (bit_offset) *bit_offset = tl_bit;
    return tl_msg.c_str();
}

uint64_t hpdr_launch_count(int reset) {
    uint64_t v = reset ? g_launches.exchange(0) : g_launches.load();
    return v;
}

void hpdr_prof_enable(int on) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_on = on != 0;
    g_prof_serial = on == 2;
    g_prof.clear();
    g_prof_used = 0;
}

// Per-kernel aggregate since the last enable/read as JSON:
// {"kernel": [launches, total_ms, total_algorithmic_bytes, max_ms], ...}
int hpdr_prof_read(char *buf, uint64_t cap) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    std::map<std::string, std::vector<double>> agg;
    for (auto &r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) { cudaGetLastError(); ms = 0.f; }
        auto &v = agg[r.name];
        if (v.empty()) v.assign(4, 0.0);
        v[0] += 1;
        v[1] += ms;
        v[2] += r.bytes;
        v[3] = std::max(v[3], (double)ms);
    }
    std::string s = "{";
    for (auto &kv : agg) {
        char tmp[256];
        snprintf(tmp, sizeof(tmp), "%s\"%s\": [%.0f, %.6f, %.0f, %.6f]", s.size() > 1 ? ", " : "", kv.first.c_str(),
                 kv.second[0], kv.second[1], kv.second[2], kv.second[3]);
        s += tmp;
    }
    s += "}";
    g_prof.clear();
    g_prof_used = 0;
    if (s.size() + 1 > cap) return HPDR_ERR_BUFFER;
    memcpy(buf, s.c_str(), s.size() + 1);
    return HPDR_OK;
}

void *hpdr_ctx_stream(const hpdr_ctx *c) { return c ? (void *)c->stream : nullptr; }

int hpdr_ctx_create(int device, hpdr_ctx **out) {
    try {
        int n = 0;
        CUDA_CHECK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw Error{HPDR_ERR_CUDA, "no such CUDA device", -1};
        CUDA_CHECK(cudaSetDevice(device));
        hpdr_ctx *c = new hpdr_ctx();
        c->device = device;
        // the level chain (critical path) outranks side work (aux) when both have blocks waiting
        int lo_pri = 0, hi_pri = 0;
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        CUDA_CHECK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_pri));
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
        // aux: the finest quantization of a relative-mode compress (off the level chain), low;
        // aux_hi: the finest correction of a decompress, the longest chain before the output, high
        // (1024^3: the first output slab 0.5 ms earlier than at low priority)
        CUDA_CHECK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, lo_pri));
        CUDA_CHECK(cudaStreamCreateWithPriority(&c->aux_hi, cudaStreamNonBlocking, hi_pri));
        for (auto &x : c->side) CUDA_CHECK(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, hi_pri));
        *out = c;
        return HPDR_OK;
    } catch (const Error &e) {
        set_error(e.code, e.msg, e.bit_offset);
        return e.code;
    }
}

void hpdr_ctx_trim(hpdr_ctx *c) {
    if (!c) return;
    for (hpdr_ctx *q : c->queues) hpdr_ctx_trim(q);
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto &kv : c->dev) if (kv.second.ptr) cudaFree(kv.second.ptr);
    for (auto &kv : c->pinned) if (kv.second.ptr) cudaFreeHost(kv.second.ptr);
    c->dev.clear();
    c->pinned.clear();
}

void hpdr_ctx_destroy(hpdr_ctx *c) {
    if (!c) return;
    for (hpdr_ctx *q : c->queues) hpdr_ctx_destroy(q);
    c->queues.clear();
    hpdr_ctx_trim(c);
    for (auto &kv : c->plans) cudaFree(kv.second->dbuf);
    for (auto &v : c->events)
        for (cudaEvent_t e : v) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->h2d);
    cudaStreamDestroy(c->d2h);
    cudaStreamDestroy(c->aux);
    cudaStreamDestroy(c->aux_hi);
    for (auto x : c->side) cudaStreamDestroy(x);
    delete c;
}

uint64_t hpdr_ctx_alloc_events(const hpdr_ctx *c) {
    if (!c) return 0;
    uint64_t n = c->alloc_events;
    for (const hpdr_ctx *q : c->queues) n += q->alloc_events;
    return n;
}
int hpdr_ctx_device(const hpdr_ctx *c) { return c ? c->device : -1; }

void hpdr_ctx_set_range_hook(hpdr_ctx *c, hpdr_range_hook hook, void *user) {
    if (!c) return;
    c->range_hook = hook;
    c->range_user = user;
}

void hpdr_host_copy(void *dst, const void *src, uint64_t n) { hpdr::parallel_memcpy(dst, src, n); }

// First-touch a fresh pageable buffer on background threads (huge pages where the kernel allows),
// so that a later staged copy into it runs at warm-memory speed.  The touch writes zeros: nothing
// else may write the buffer before hpdr_host_prefault_wait returns.
struct hpdr_prefault {
    std::vector<std::thread> th;
};

void *hpdr_host_prefault_begin(void *p, uint64_t n) {
    if (!p || !n) return nullptr;
    const uintptr_t a = ((uintptr_t)p + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
    const uintptr_t e = ((uintptr_t)p + n) & ~uintptr_t((2u << 20) - 1);
    if (e > a) madvise((void *)a, e - a, MADV_HUGEPAGE);
    auto *h = new hpdr_prefault;
    const int T = std::max(1, std::min(4, hpdr::host_threads() / 4));   // light: the input DMA shares host memory
    const size_t per = ((n + T - 1) / T + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
    for (int t = 0; t < T; t++) {
        const size_t lo = (size_t)t * per;
        if (lo >= n) break;
        const size_t hi = std::min<size_t>(n, lo + per);
        h->th.emplace_back([p, lo, hi] {
            char *c = (char *)p;
            for (size_t o = lo; o < hi; o += 4096) c[o] = 0;
        });
    }
    return h;
}

void hpdr_host_prefault_wait(void *handle) {
    auto *h = (hpdr_prefault *)handle;
    if (!h) return;
    for (auto &t : h->th) t.join();
    delete h;
}

void *hpdr_host_alloc(uint64_t bytes) {
    void *p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        set_error(HPDR_ERR_ALLOCATION, "cudaHostAlloc failed");
        return nullptr;
    }
    return p;
}

void hpdr_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

int hpdr_host_register(void *p, uint64_t bytes) {
    if (!p || !bytes) return HPDR_OK;
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    if (e == cudaSuccess || e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        return HPDR_OK;
    }
    cudaGetLastError();
    set_error(HPDR_ERR_ALLOCATION, std::string("cudaHostRegister failed: ") + cudaGetErrorString(e));
    return HPDR_ERR_ALLOCATION;
}

void hpdr_host_unregister(void *p) {
    if (p && cudaHostUnregister(p) != cudaSuccess) cudaGetLastError();
}

}  // extern "C"
