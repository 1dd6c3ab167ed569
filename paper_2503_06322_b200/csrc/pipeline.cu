// pipeline.cu -- the overlapped host<->device reduction pipeline of the paper (HDEM, Fig. 7,
// PAPER.md:413-533), rebuilt on CUDA streams.
//
// The field is split into dim-0 chunks, chunk k going to queue k mod Q (Fig. 7's queues; Q = 3 by
// default, HPDR_PIPE_QUEUES).  A queue is a full device context (its own compute / H2D / D2H
// streams, buffers and operator tables) driven by its own host thread, so up to Q chunks are
// reduced concurrently: the per-chunk kernels that are latency-bound on a thin slab (axis
// marches, Thomas lines, Huffman units) overlap each other, and the copy engines stream chunk
// k+1 in and chunk k-1 out meanwhile.  Per queue, in order:
//   H2D(k) -> reduce(k) into a reference-identical MGARD blob (global value range,
//   SPEC.md:425) -> D2H(k) into the HPDR container
// with the reuse edges of Fig. 7 as stream order / events on the queue (H2D(k+Q) after
// reduce(k); reduce(k+Q) after D2H(k)).  The only cross-queue dependency is the container
// offset: D2H(k) starts once the sizes of chunks < k are known (right after their reduction,
// not their copies).  Decompression mirrors it (blob in, field slab out at a fixed offset).
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>

#include "stages.cuh"
#include "transform.cuh"

namespace hpdr {

void compress_core(hpdr_ctx *ctx, const void *in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                   uint32_t dict_size, int has_range, double range_min, double range_max, bool allow_stream,
                   void *fetch_out = nullptr, uint64_t fetch_cap = 0, const OutAlloc *alloc = nullptr);
void decompress_core(hpdr_ctx *ctx, const void *blob_in, uint64_t len, const uint8_t *dev_blob, void *out,
                     uint64_t out_bytes, bool sync);
void compress_from_coef(hpdr_ctx *ctx, const double *coef, int dtype, int rank, const uint64_t *dims, double eb_rel,
                        uint32_t dict_size, double u_min, double u_max);
void decompose_chunk(hpdr_ctx *ctx, const void *d_in, int dtype, int rank, const uint64_t *dims, double *coef,
                     unsigned long long *mm);
void fetch_pending_on(hpdr_ctx *ctx, const hpdr_ctx::Pending &P, void *out, uint64_t cap, cudaStream_t s, bool sync);
int zfp_container_decompress(hpdr_ctx *ctx, const uint8_t *c, uint64_t len, void *out, uint64_t out_bytes,
                             double *trace);   // zfp.cu: pipeline id 1

namespace {

struct CrcTable {
    uint32_t t[256];
    CrcTable() {
        for (uint32_t i = 0; i < 256; i++) {
            uint32_t c = i;
            for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[i] = c;
        }
    }
};

uint32_t crc32(const uint8_t *p, size_t n) {   // zlib polynomial, as container.py's zlib.crc32
    static const CrcTable table;                // thread-safe one-time initialisation
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; i++) c = table.t[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

template <class T>
void put(std::vector<uint8_t> &v, T x) {
    size_t o = v.size();
    v.resize(o + sizeof(T));
    memcpy(v.data() + o, &x, sizeof(T));
}

struct Chunk {
    uint64_t raw_off, raw_size, pay_off, pay_size;
};

std::vector<uint8_t> container_header(int dtype, int rank, const uint64_t *dims, double eb_rel, uint32_t dict,
                                      double vmin, double vmax, const std::vector<Chunk> &chunks) {
    std::vector<uint8_t> h = {'H', 'P', 'D', 'R'};
    put<uint16_t>(h, 1);
    put<uint8_t>(h, 2);   // MGARD
    put<uint8_t>(h, (uint8_t)dtype);
    put<uint8_t>(h, (uint8_t)rank);
    for (int d = 0; d < rank; d++) put<uint64_t>(h, dims[d]);
    put<double>(h, eb_rel);
    put<uint32_t>(h, dict);
    put<double>(h, vmin);
    put<double>(h, vmax);
    put<uint32_t>(h, (uint32_t)chunks.size());
    for (const Chunk &c : chunks) {
        put<uint64_t>(h, c.raw_off);
        put<uint64_t>(h, c.raw_size);
        put<uint64_t>(h, c.pay_off);
        put<uint64_t>(h, c.pay_size);
    }
    put<uint32_t>(h, crc32(h.data(), h.size()));
    return h;
}

// numpy min/max semantics (NaN propagates) over a host array, on all host cores.
void host_minmax(const void *in, int dtype, uint64_t n, double *vmin, double *vmax) {
    const unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<double> mn(T, INFINITY), mx(T, -INFINITY);
    std::vector<int> nan(T, 0);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; t++)
        th.emplace_back([&, t] {
            const uint64_t a = n * t / T, b = n * (t + 1) / T;
            double lo = INFINITY, hi = -INFINITY;
            int bad = 0;
            for (uint64_t i = a; i < b; i++) {
                const double v = dtype == 0 ? (double)((const float *)in)[i] : ((const double *)in)[i];
                if (v != v) bad = 1;
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
            mn[t] = lo;
            mx[t] = hi;
            nan[t] = bad;
        });
    for (auto &x : th) x.join();
    double lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    for (unsigned t = 0; t < T; t++) {
        lo = std::min(lo, mn[t]);
        hi = std::max(hi, mx[t]);
        bad |= nan[t] != 0;
    }
    *vmin = bad ? __builtin_nan("") : lo;
    *vmax = bad ? __builtin_nan("") : hi;
}

struct Timer {   // per-task CUDA-event timestamps for the pipeline trace
    std::vector<cudaEvent_t> ev;
    cudaEvent_t t0 = nullptr;
    bool on;
    explicit Timer(bool on_, size_t n) : on(on_) {
        if (!on) return;
        CUDA_CHECK(cudaEventCreate(&t0));
        ev.resize(n);
        for (auto &e : ev) CUDA_CHECK(cudaEventCreate(&e));
    }
    ~Timer() {
        if (t0) cudaEventDestroy(t0);
        for (auto e : ev) cudaEventDestroy(e);
    }
    void mark(size_t i, cudaStream_t s) {
        if (on) CUDA_CHECK(cudaEventRecord(ev[i], s));
    }
    void dump(double *out) {
        if (!on) return;
        for (size_t i = 0; i < ev.size(); i++) {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, t0, ev[i]));
            out[i] = ms;
        }
    }
};

}  // namespace
}  // namespace hpdr

using namespace hpdr;

namespace {

int pipe_queues(uint64_t K) {
    static const int q_env = [] {
        const char *e = getenv("HPDR_PIPE_QUEUES");
        return e ? std::max(1, atoi(e)) : 3;
    }();
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)q_env, K));
}

// Runs fn(q) for q = 0..Q-1 on Q host threads; the first error (in chunk order of detection) is rethrown.
struct QueueRun {
    std::mutex mu;
    std::condition_variable cv;
    bool failed = false;
    Error err{HPDR_OK, "", -1};
    void fail(const Error &e) {
        std::lock_guard<std::mutex> g(mu);
        if (!failed) {
            failed = true;
            err = e;
        }
        cv.notify_all();
    }
    template <class F>
    void run(int Q, F &&fn) {
        std::vector<std::thread> th;
        for (int q = 0; q < Q; q++)
            th.emplace_back([&, q] {
                try {
                    fn(q);
                } catch (const Error &e) {
                    fail(e);
                } catch (const std::exception &e) {
                    fail(Error{HPDR_ERR_CUDA, e.what(), -1});
                }
            });
        for (auto &t : th) t.join();
        if (failed) throw err;
    }
};

}  // namespace

extern "C" {

int hpdr_pipeline_compress(hpdr_ctx *ctx, const void *host_in, int dtype, int rank, const uint64_t *dims, double eb_rel,
                           uint32_t dict_size, int has_range, double range_min, double range_max,
                           uint64_t chunk_planes, const uint64_t *chunk_list, uint64_t n_list, void *out,
                           uint64_t out_cap, uint64_t *out_len, double *trace) {
    try {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        if (dtype != 0 && dtype != 1) throw Error{HPDR_ERR_VALIDATION, "lossy compression needs F32/F64", -1};
        if (rank < 1 || rank > 4) throw Error{HPDR_ERR_VALIDATION, "rank must be 1..4", -1};
        const size_t isz = dtype == 0 ? 4 : 8;
        uint64_t plane = 1;
        for (int d = 1; d < rank; d++) plane *= dims[d];
        const uint64_t n0 = dims[0], N = n0 * plane;
        // chunk sequence: explicit plane counts (e.g. from the adaptive Algorithm-4 schedule) or fixed
        std::vector<uint64_t> sizes;
        if (chunk_list && n_list) {
            uint64_t tot = 0;
            for (uint64_t i = 0; i < n_list; i++) {
                if (!chunk_list[i]) throw Error{HPDR_ERR_VALIDATION, "empty chunk in the chunk list", -1};
                sizes.push_back(chunk_list[i]);
                tot += chunk_list[i];
            }
            if (tot != n0) throw Error{HPDR_ERR_VALIDATION, "chunk list does not tile dim 0", -1};
        } else {
            if (!chunk_planes) chunk_planes = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(1, plane * isz));
            chunk_planes = std::min(chunk_planes, n0);
            for (uint64_t a = 0; a < n0; a += chunk_planes) sizes.push_back(std::min(chunk_planes, n0 - a));
        }
        const uint64_t K = sizes.size();
        const bool in_pageable = classify(host_in) == MemKind::Host;   // staged through pinned rings
        double vmin = range_min, vmax = range_max;
        // Relative mode needs the global range before any chunk is quantized.  The
        // decomposition does not depend on it, so by default the chunks are streamed in and
        // decomposed first (phase A, per-chunk min/max on the device), and quantized, coded and
        // streamed out once the range is known (phase B).  HPDR_PIPE_HOST_RANGE=1: a host pre-pass.
        static const bool host_range = getenv("HPDR_PIPE_HOST_RANGE") != nullptr;
        const bool two_phase = !has_range && !host_range;
        if (!has_range && host_range) host_minmax(host_in, dtype, N, &vmin, &vmax);
        std::vector<Chunk> chunks(K);
        uint64_t maxp = 1;
        for (uint64_t k = 0, a = 0; k < K; a += sizes[k], k++) {
            chunks[k] = Chunk{a * plane, sizes[k] * plane, 0, 0};
            maxp = std::max(maxp, sizes[k]);
        }
        const size_t hdr_len = container_header(dtype, rank, dims, eb_rel, dict_size, vmin, vmax, chunks).size();
        if (out_cap < hdr_len) throw Error{HPDR_ERR_BUFFER, "output buffer too small for the container header", -1};
        const size_t cbytes = maxp * plane * isz;
        const int Q = pipe_queues(K);
        std::vector<hpdr_ctx *> qc(Q);
        for (int q = 0; q < Q; q++) qc[q] = ctx->queue(q);
        // relative mode: phase B (quantize + code + copy out, once the range is known) runs on QB
        // contexts of its own (streams, buffers), so chunk k's phase B is not queued behind the
        // phase-A decompositions of later chunks.  QB = Q threads by default (measured: 3 / 6 / 9 phase-B
        // threads -> 13.3 / 13.6 / 14.3 ms at 513^3); HPDR_PIPE_QUEUES_B (>= Q) overrides.
        static const int qb_env = [] {
            const char *e = getenv("HPDR_PIPE_QUEUES_B");
            return e ? std::max(1, atoi(e)) : 0;
        }();
        const int QB = two_phase ? (int)std::min<uint64_t>(K, (uint64_t)(qb_env ? std::max(qb_env, Q) : Q)) : Q;
        std::vector<hpdr_ctx *> qb(QB);
        for (int q = 0; q < QB; q++) qb[q] = two_phase ? ctx->queue(Q + q) : qc[q];
        for (hpdr_ctx *x : qc) x->graphs_ok = false;   // several host threads on one device
        for (hpdr_ctx *x : qb) x->graphs_ok = false;
        struct GraphsBack {
            hpdr_ctx *c;
            ~GraphsBack() { c->graphs_ok = true; }
        } graphs_back{ctx};
        Timer tm(trace != nullptr, 6 * K);
        // every queue starts after the caller's prior work on the main context
        CUDA_CHECK(cudaEventRecord(ctx->event(0), ctx->stream));
        if (tm.on) CUDA_CHECK(cudaEventRecord(tm.t0, ctx->stream));
        // container offsets: pos[k] is known once the sizes of chunks < k are
        std::vector<uint64_t> pos(K + 1, 0), psize(K, 0);
        std::vector<char> have(K, 0);
        uint64_t next_pos = 0;   // first chunk whose offset is not yet known
        pos[0] = hdr_len;
        double *coef_all = nullptr;
        // Relative mode, per queue thread: phase A streams its chunks in, folds their min/max on the
        // copy stream (so the range is known as soon as the data is, not after the decompositions)
        // and decomposes them on the compute stream; once every queue has reported its min/max the
        // thread runs phase B (quantize + code + copy out) for its chunks, overlapping the other
        // queues' phase-A tails.
        std::mutex rmu;
        std::condition_variable rcv;
        int reported = 0;
        unsigned long long gkey[3] = {~0ULL, 0ULL, 0ULL};
        if (two_phase) coef_all = (double *)ctx->dbuf("pipe_coef", N * 8);
        auto phase_a = [&](int q, QueueRun &RR) {
            hpdr_ctx *c = qc[q];
            if (c != ctx) CUDA_CHECK(cudaStreamWaitEvent(c->stream, ctx->event(0), 0));
            CUDA_CHECK(cudaStreamWaitEvent(c->h2d, ctx->event(0), 0));
            char *din = (char *)c->dbuf("pipe_in", cbytes);
            unsigned long long *mm = (unsigned long long *)c->dbuf("pipe_mm", 32);
            unsigned long long *hmm = (unsigned long long *)c->hbuf("pipe_mm_h", 32);
            hmm[0] = ~0ULL;
            hmm[1] = 0ULL;
            hmm[2] = 0ULL;
            CUDA_CHECK(cudaMemcpyAsync(mm, hmm, 24, cudaMemcpyHostToDevice, c->h2d));
            cudaEvent_t ev_in = c->event(300), ev_red = c->event(301);
            bool first = true;
            for (uint64_t k = q; k < K; k += Q) {
                if (RR.failed) return false;
                if (!first) CUDA_CHECK(cudaStreamWaitEvent(c->h2d, ev_red, 0));   // input buffer reuse edge
                tm.mark(6 * k, c->h2d);
                if (in_pageable)
                    stage_h2d(c, din, (const char *)host_in + chunks[k].raw_off * isz, chunks[k].raw_size * isz, c->h2d);
                else
                    CUDA_CHECK(cudaMemcpyAsync(din, (const char *)host_in + chunks[k].raw_off * isz,
                                               chunks[k].raw_size * isz, cudaMemcpyDefault, c->h2d));
                tm.mark(6 * k + 1, c->h2d);
                minmax_accumulate(din, dtype, (int64_t)chunks[k].raw_size, mm, c->h2d);
                CUDA_CHECK(cudaEventRecord(ev_in, c->h2d));
                CUDA_CHECK(cudaStreamWaitEvent(c->stream, ev_in, 0));
                tm.mark(6 * k + 2, c->stream);
                uint64_t sd[4] = {chunks[k].raw_size / plane, 0, 0, 0};
                for (int d = 1; d < rank; d++) sd[d] = dims[d];
                decompose_chunk(c, din, dtype, rank, sd, coef_all + chunks[k].raw_off, nullptr);
                CUDA_CHECK(cudaEventRecord(ev_red, c->stream));
                CUDA_CHECK(cudaEventRecord(c->event(EvPipeCoef, k), c->stream));   // chunk k's coefficients
                first = false;
            }
            CUDA_CHECK(cudaMemcpyAsync(hmm, mm, 24, cudaMemcpyDeviceToHost, c->h2d));
            CUDA_CHECK(cudaStreamSynchronize(c->h2d));   // copies + min/max only, not the decompositions
            std::unique_lock<std::mutex> lk(rmu);
            gkey[0] = std::min(gkey[0], hmm[0]);
            gkey[1] = std::max(gkey[1], hmm[1]);
            gkey[2] |= hmm[2];
            if (++reported == Q) {
                minmax_from_keys(gkey, &vmin, &vmax);
                rcv.notify_all();
            } else {
                rcv.wait(lk, [&] { return reported >= Q || RR.failed; });
            }
            return !RR.failed;
        };
        const int QA = Q;   // phase-A threads (relative mode); every thread runs phase B
        QueueRun R;
        R.run(std::max(QA, QB), [&](int q) {
            if (q >= QB) {   // phase A only (cannot happen: QB >= QA)
                if (two_phase) phase_a(q, R);
                return;
            }
            const int Q = QB;
            hpdr_ctx *c = q < QA ? qc[q] : nullptr;
            CUDA_CHECK(cudaSetDevice(ctx->device));
            if (two_phase) {
                try {
                    if (q < QA) {
                        if (!phase_a(q, R)) return;
                    } else {   // phase-B-only thread: wait for the range
                        std::unique_lock<std::mutex> lk(rmu);
                        rcv.wait(lk, [&] { return reported >= QA || R.failed; });
                        if (R.failed) return;
                    }
                } catch (...) {
                    {
                        std::lock_guard<std::mutex> g(rmu);
                        reported = std::max(reported, QA);   // release the others; R.fail() marks the run failed
                    }
                    rcv.notify_all();
                    throw;
                }
                c = qb[q];
            }
            if (c != ctx) {
                CUDA_CHECK(cudaStreamWaitEvent(c->stream, ctx->event(0), 0));
            }
            CUDA_CHECK(cudaStreamWaitEvent(c->h2d, ctx->event(0), 0));
            CUDA_CHECK(cudaStreamWaitEvent(c->d2h, ctx->event(0), 0));
            char *din = two_phase ? nullptr : (char *)c->dbuf("pipe_in", cbytes);
            // event ids 300-303 are reserved for the runner; the output buffer sets alternate
            cudaEvent_t ev_in = c->event(300), ev_red = c->event(301), ev_outs[2] = {c->event(302), c->event(303)};
            bool first = true;
            uint64_t t = 0;
            for (uint64_t k = q; k < K; k += Q, t++) {
                if (R.failed) return;
                cudaEvent_t ev_out = ev_outs[t & 1];
                c->out_slot = (int)(t & 1);
                if (!two_phase) {
                    if (!first) CUDA_CHECK(cudaStreamWaitEvent(c->h2d, ev_red, 0));   // input buffer reuse edge
                    tm.mark(6 * k, c->h2d);
                    if (in_pageable)
                        stage_h2d(c, din, (const char *)host_in + chunks[k].raw_off * isz, chunks[k].raw_size * isz,
                                  c->h2d);
                    else
                        CUDA_CHECK(cudaMemcpyAsync(din, (const char *)host_in + chunks[k].raw_off * isz,
                                                   chunks[k].raw_size * isz, cudaMemcpyDefault, c->h2d));
                    tm.mark(6 * k + 1, c->h2d);
                    CUDA_CHECK(cudaEventRecord(ev_in, c->h2d));
                    CUDA_CHECK(cudaStreamWaitEvent(c->stream, ev_in, 0));
                }
                if (t >= 2) CUDA_CHECK(cudaStreamWaitEvent(c->stream, ev_out, 0));   // output set reuse edge (k - 2Q)
                if (two_phase)   // chunk k decomposed by phase-A queue k mod QA
                    CUDA_CHECK(cudaStreamWaitEvent(c->stream, qc[k % QA]->event(EvPipeCoef, k), 0));
                if (!two_phase) tm.mark(6 * k + 2, c->stream);
                uint64_t sd[4] = {chunks[k].raw_size / plane, 0, 0, 0};
                for (int d = 1; d < rank; d++) sd[d] = dims[d];
                if (two_phase)
                    compress_from_coef(c, coef_all + chunks[k].raw_off, dtype, rank, sd, eb_rel, dict_size, vmin, vmax);
                else
                    compress_core(c, din, dtype, rank, sd, eb_rel, dict_size, 1, vmin, vmax, false);
                const hpdr_ctx::Pending P = c->pending;
                tm.mark(6 * k + 3, c->stream);
                CUDA_CHECK(cudaEventRecord(ev_red, c->stream));
                uint64_t at;
                {
                    std::unique_lock<std::mutex> lk(R.mu);
                    psize[k] = P.total_len;
                    have[k] = 1;
                    while (next_pos < K && have[next_pos]) {
                        pos[next_pos + 1] = pos[next_pos] + psize[next_pos];
                        next_pos++;
                    }
                    R.cv.notify_all();
                    R.cv.wait(lk, [&] { return next_pos >= k || R.failed; });
                    if (R.failed) return;
                    at = pos[k];
                }
                if (at + P.total_len > out_cap) throw Error{HPDR_ERR_BUFFER, "output buffer too small for the container", -1};
                chunks[k].pay_off = at - hdr_len;
                chunks[k].pay_size = P.total_len;
                CUDA_CHECK(cudaStreamWaitEvent(c->d2h, ev_red, 0));
                tm.mark(6 * k + 4, c->d2h);
                fetch_pending_on(c, P, (char *)out + at, out_cap - at, c->d2h, false);
                tm.mark(6 * k + 5, c->d2h);
                CUDA_CHECK(cudaEventRecord(ev_out, c->d2h));
                first = false;
            }
            CUDA_CHECK(cudaStreamSynchronize(c->d2h));
            c->out_slot = 0;
        });
        const std::vector<uint8_t> hdr = container_header(dtype, rank, dims, eb_rel, dict_size, vmin, vmax, chunks);
        if (classify(out) == MemKind::Device) {
            CUDA_CHECK(cudaMemcpyAsync(out, hdr.data(), hdr.size(), cudaMemcpyHostToDevice, ctx->stream));
            CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } else {
            memcpy(out, hdr.data(), hdr.size());
        }
        *out_len = pos[K];
        tm.dump(trace);
        return HPDR_OK;
    } catch (const Error &e) {
        cudaDeviceSynchronize();
        set_error(e.code, e.msg, e.bit_offset);
        return e.code;
    }
}

int hpdr_pipeline_decompress(hpdr_ctx *ctx, const void *container, uint64_t len, void *out, uint64_t out_bytes,
                             double *trace) {
    try {
        CUDA_CHECK(cudaSetDevice(ctx->device));
        const uint8_t *c = (const uint8_t *)container;
        auto need = [&](uint64_t p, uint64_t n) {
            if (p > len || n > len - p) throw Error{HPDR_ERR_FORMAT, "container truncated", -1};
        };
        need(0, 9);
        if (memcmp(c, "HPDR", 4) != 0) throw Error{HPDR_ERR_FORMAT, "bad magic", -1};
        uint16_t ver;
        memcpy(&ver, c + 4, 2);
        if (ver != 1) throw Error{HPDR_ERR_FORMAT, "unsupported container version", -1};
        if (c[6] == 1) return zfp_container_decompress(ctx, c, len, out, out_bytes, trace);
        if (c[6] != 2) throw Error{HPDR_ERR_FORMAT, "unknown pipeline id", -1};
        const int dtype = c[7], rank = c[8];
        uint64_t pos = 9;
        need(pos, 8ull * rank + 28 + 4);
        std::vector<uint64_t> dims(rank);
        memcpy(dims.data(), c + pos, 8ull * rank);
        pos += 8ull * rank + 28;
        uint32_t K;
        memcpy(&K, c + pos, 4);
        pos += 4;
        need(pos, 32ull * K + 4);
        std::vector<Chunk> chunks(K);
        memcpy(chunks.data(), c + pos, 32ull * K);
        pos += 32ull * K;
        uint32_t crc;
        memcpy(&crc, c + pos, 4);
        if (crc32(c, pos) != crc) throw Error{HPDR_ERR_FORMAT, "header checksum mismatch", -1};
        pos += 4;
        const uint64_t base = pos;
        static const int isz_tab[7] = {4, 8, 4, 8, 4, 8, 1};
        if (dtype > 6) throw Error{HPDR_ERR_FORMAT, "unknown dtype", -1};
        const size_t isz = isz_tab[dtype];
        uint64_t N = 1;
        for (uint64_t d : dims) N *= d;
        if (out_bytes < N * isz) throw Error{HPDR_ERR_BUFFER, "output buffer too small", -1};
        uint64_t maxpay = 1, maxraw = 1;
        for (const Chunk &ch : chunks) {
            need(base + ch.pay_off, ch.pay_size);
            if (ch.raw_off + ch.raw_size > N) throw Error{HPDR_ERR_FORMAT, "chunk outside the field", -1};
            maxpay = std::max(maxpay, ch.pay_size);
            maxraw = std::max(maxraw, ch.raw_size);
        }
        const MemKind omk = classify(out);
        const bool host_out = omk != MemKind::Device, out_pageable = omk == MemKind::Host;
        const bool blob_pageable = classify(container) == MemKind::Host;
        const int Q = pipe_queues(K);
        std::vector<hpdr_ctx *> qc(Q);
        for (int q = 0; q < Q; q++) qc[q] = ctx->queue(q);
        for (hpdr_ctx *x : qc) x->graphs_ok = false;   // several host threads on one device
        struct GraphsBack {
            hpdr_ctx *c;
            ~GraphsBack() { c->graphs_ok = true; }
        } graphs_back{ctx};
        Timer tm(trace != nullptr, 6 * (size_t)K);
        CUDA_CHECK(cudaEventRecord(ctx->event(0), ctx->stream));
        if (tm.on) CUDA_CHECK(cudaEventRecord(tm.t0, ctx->stream));
        QueueRun R;
        R.run(Q, [&](int q) {
            hpdr_ctx *x = qc[q];
            CUDA_CHECK(cudaSetDevice(x->device));
            if (x != ctx) CUDA_CHECK(cudaStreamWaitEvent(x->stream, ctx->event(0), 0));
            CUDA_CHECK(cudaStreamWaitEvent(x->h2d, ctx->event(0), 0));
            CUDA_CHECK(cudaStreamWaitEvent(x->d2h, ctx->event(0), 0));
            // two blob buffers: chunk k+Q's H2D overlaps chunk k's recomposition (the blob is read by
            // its decode and outlier scatter only)
            uint8_t *dblobs[2] = {(uint8_t *)x->dbuf("pipe_blob", maxpay), (uint8_t *)x->dbuf("pipe_blob#1", maxpay)};
            cudaEvent_t ev_reds[2] = {x->event(304), x->event(305)};
            char *douts[2] = {host_out ? (char *)x->dbuf("pipe_out0", maxraw * isz) : nullptr,
                              host_out ? (char *)x->dbuf("pipe_out1", maxraw * isz) : nullptr};
            cudaEvent_t ev_in = x->event(300), ev_red = x->event(301), ev_outs[2] = {x->event(302), x->event(303)};
            uint64_t t = 0;
            for (uint64_t k = q; k < K; k += Q, t++) {
                if (R.failed) return;
                char *dout = douts[t & 1];
                cudaEvent_t ev_out = ev_outs[t & 1];
                uint8_t *dblob = dblobs[t & 1];
                if (t >= 2) CUDA_CHECK(cudaStreamWaitEvent(x->h2d, ev_reds[t & 1], 0));   // blob buffer reuse edge
                tm.mark(6 * k, x->h2d);
                if (blob_pageable)
                    stage_h2d(x, dblob, c + base + chunks[k].pay_off, chunks[k].pay_size, x->h2d);
                else
                    CUDA_CHECK(cudaMemcpyAsync(dblob, c + base + chunks[k].pay_off, chunks[k].pay_size,
                                               cudaMemcpyDefault, x->h2d));
                tm.mark(6 * k + 1, x->h2d);
                CUDA_CHECK(cudaEventRecord(ev_in, x->h2d));
                CUDA_CHECK(cudaStreamWaitEvent(x->stream, ev_in, 0));
                if (t >= 2 && host_out) CUDA_CHECK(cudaStreamWaitEvent(x->stream, ev_out, 0));   // output slab reuse (k - 2Q)
                tm.mark(6 * k + 2, x->stream);
                char *dst = host_out ? dout : (char *)out + chunks[k].raw_off * isz;
                decompress_core(x, c + base + chunks[k].pay_off, chunks[k].pay_size, dblob, dst,
                                chunks[k].raw_size * isz, false);
                tm.mark(6 * k + 3, x->stream);
                CUDA_CHECK(cudaEventRecord(ev_red, x->stream));
                CUDA_CHECK(cudaEventRecord(ev_reds[t & 1], x->stream));
                CUDA_CHECK(cudaStreamWaitEvent(x->d2h, ev_red, 0));
                tm.mark(6 * k + 4, x->d2h);
                if (host_out && out_pageable)   // host-blocking; the other queues keep the GPU busy
                    stage_d2h(x, (char *)out + chunks[k].raw_off * isz, dout, chunks[k].raw_size * isz, x->d2h);
                else if (host_out)
                    CUDA_CHECK(cudaMemcpyAsync((char *)out + chunks[k].raw_off * isz, dout, chunks[k].raw_size * isz,
                                               cudaMemcpyDeviceToHost, x->d2h));
                tm.mark(6 * k + 5, x->d2h);
                CUDA_CHECK(cudaEventRecord(ev_out, x->d2h));
            }
            CUDA_CHECK(cudaStreamSynchronize(x->d2h));
            CUDA_CHECK(cudaStreamSynchronize(x->stream));
        });
        tm.dump(trace);
        return HPDR_OK;
    } catch (const Error &e) {
        cudaDeviceSynchronize();
        set_error(e.code, e.msg, e.bit_offset);
        return e.code;
    }
}

}  // extern "C"
