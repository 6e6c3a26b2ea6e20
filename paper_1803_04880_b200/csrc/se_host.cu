// se_host.cu — host-resident streaming protect / recover (NEXT row f1).
//
// The paper's end-to-end scenario moves chunks over PCIe and overlaps the
// transfer with GPU work (PCIe named as the bottleneck,
// P:1958).  Here the library does that itself: the input is cut into
// chunks of whole block-rows (aligned so each chunk's stream slices start on
// byte boundaries and its AES-CTR start is integral), and chunk k runs on
// stream k mod S as H2D copy -> fused kernel -> D2H copies, so copies of one
// chunk overlap the kernel of another.  Device staging buffers come from the
// stream-ordered pool.  Host buffers should be pinned for the copies to be
// asynchronous (pageable buffers still work, with driver staging).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "se_internal.h"

namespace se {

static uint64_t gcd64(uint64_t a, uint64_t b) {
    while (b) { const uint64_t t = a % b; a = b; b = t; }
    return a;
}

// smallest block count g: g*a_bits % 128 == 0 and g*{b,c}_bits % 8 == 0
// (and a multiple of min_blocks)
static uint64_t chunk_block_align(const se_layout& lay, uint64_t min_blocks = 1) {
    uint64_t g = 128 / gcd64(128, lay.a_bits);
    g = g / gcd64(g, min_blocks) * min_blocks;
    for (uint64_t bits : {(uint64_t)lay.b_bits, (uint64_t)lay.c_bits}) {
        if (!bits) continue;
        const uint64_t h = 8 / gcd64(8, bits);
        g = g / gcd64(g, h) * h;
    }
    return g;
}

struct Chunk {
    uint64_t byte0, byte1;   // input slice
    uint64_t blk0;           // first local block
    uint64_t nblk;
};

// SE_HOST_RAMP: chunk sizes ramping up at the start and down at the end
// (1/8, 1/4, 1/2 of the nominal size) to shorten the pipeline's fill and
// drain.  Measured slower on C2 (11.3 vs 12.5 GB/s at 4 MiB: the per-chunk
// copy and launch costs of the extra chunks outweigh it), so off.
#ifndef SE_HOST_RAMP
#define SE_HOST_RAMP 0
#endif
#ifndef SE_HOST_BALANCE
#define SE_HOST_BALANCE 1
#endif
// chunk_bytes == 0: a quarter of the input, within [4 MiB, 16 MiB] — small
// files need >= 3-4 chunks to overlap at all, large ones lose ~15 % of the
// PCIe rate to per-chunk costs below ~16 MiB (tools/e2e_probe.py: 256 MiB
// protect 28.7 GB/s at 4 MiB, 34.9 at 16 MiB, 92 % of the D2H-bound model).
static uint64_t auto_chunk(uint64_t n) {
    return std::min<uint64_t>(16ull << 20, std::max<uint64_t>(4ull << 20, n / 4));
}

static std::vector<Chunk> make_chunks(const se_geom* g, const se_layout& lay, uint64_t chunk_bytes,
                                      uint64_t min_blocks = 1) {
    const uint64_t bpr = g->width / 8, block_rows = lay.rows / 8;
    const uint64_t ga = chunk_block_align(lay, min_blocks);
    const uint64_t unit = ga / gcd64(ga, bpr);                 // block-rows per alignment unit
    const uint64_t row_bytes = 8ull * g->width;
    uint64_t rows_per = std::max<uint64_t>(1, chunk_bytes / row_bytes);
    if (SE_HOST_BALANCE && rows_per < block_rows) {
        // equal chunks near the requested size, no short remainder chunk (C2 at
        // 4 MiB: 86 + 85 + 85 block rows, not 85 + 85 + 85 + 1, whose extra
        // pipeline step cost as much as a full chunk's)
        const uint64_t k = std::max<uint64_t>(1, (block_rows + rows_per / 2) / rows_per);
        rows_per = (block_rows + k - 1) / k;
        rows_per = (rows_per + unit - 1) / unit * unit;
    }
    rows_per = std::max<uint64_t>(unit, rows_per / unit * unit);
    auto units = [&](uint64_t rows) { return std::max<uint64_t>(unit, rows / unit * unit); };
    // sizes in block rows: ramp up, full chunks, ramp down
    std::vector<uint64_t> head, tail;
    if (SE_HOST_RAMP)
        for (uint64_t d = 8; d >= 2; d /= 2) head.push_back(units(rows_per / d));
    uint64_t ramp = 0;
    for (uint64_t h : head) ramp += 2 * h;
    std::vector<uint64_t> sizes;
    if (head.empty() || block_rows < ramp + rows_per) {
        for (uint64_t br = 0; br < block_rows; br += rows_per) sizes.push_back(std::min(rows_per, block_rows - br));
    } else {
        sizes = head;
        uint64_t mid = block_rows - ramp;
        while (mid > 0) {
            const uint64_t r = std::min(rows_per, mid);
            sizes.push_back(r);
            mid -= r;
        }
        for (auto it = head.rbegin(); it != head.rend(); ++it) sizes.push_back(*it);
    }
    std::vector<Chunk> v;
    uint64_t br = 0;
    for (uint64_t r : sizes) {
        const uint64_t br1 = std::min(block_rows, br + r);
        if (br1 <= br) break;
        Chunk c;
        c.byte0 = std::min(g->n_bytes, br * row_bytes);
        c.byte1 = std::min(g->n_bytes, br1 * row_bytes);
        c.blk0 = br * bpr;
        c.nblk = (br1 - br) * bpr;
        v.push_back(c);
        br = br1;
    }
    return v;
}

// Per-device streaming context, created on first use and kept for the life of
// the process: S non-blocking streams and one staging slot per stream (device
// buffers for one chunk's input / output and its three fragment slices, grown
// on demand).  Chunk k uses slot k mod S on stream k mod S, so stream order
// alone makes slot reuse safe; steady-state calls allocate nothing.
//
// The per-chunk work is ~8 API calls (copies, keystream and fused kernels),
// which at 1-4 MiB chunks costs as much host time as the PCIe transfer it
// pipelines.  So each call's whole chunk sequence (on all streams, fork/join
// by events) is captured once into a CUDA graph, cached per (operation,
// geometry, key, IV, host pointers, chunking) and replayed by one
// cudaGraphLaunch on later calls with the same arguments (host data is read
// at replay time, so new contents in the same buffers are fine).  Any
// staging-buffer reallocation drops the cache.  SE_HOST_GRAPHS=0 in the
// environment disables it.
struct Slot {
    void* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};   // bytes, A, B, C, keystream scratch
    size_t cap[5] = {0, 0, 0, 0, 0};
};

}  // namespace se

// Asynchronous host calls (fragment_*_host_async): the per-chunk completion
// events, in chunk order with each chunk's first block, so a dependent call
// can wait chunk by chunk; recover tickets also carry the chunk reports.
struct se_host_ticket {
    int op = 0;                             // 0 protect, 1 recover
    std::vector<uint64_t> blk0, nblk;       // chunk block ranges
    std::vector<cudaEvent_t> done;          // chunk k's results are in host memory
    std::vector<cudaEvent_t> tail;          // one per stream: everything enqueued has finished
    std::vector<se_report> reps;            // recover: per-chunk reports, read at se_host_wait
    const se_report* hreps = nullptr;       // recover: the context's pinned mirror until then
    void* ctx = nullptr;                    // the HostCtx it runs in
    bool collected = false;
    int status = SE_OK;
};

namespace se {

struct GraphKey {
    int op;                   // 0 protect, 1 recover
    uint32_t n_streams;
    uint64_t chunk_bytes;
    se_geom g;
    uint8_t key[16], iv[16];
    const void* ptr[4];       // host buffers: bytes (in or out), A, B, C
};

struct GraphEntry {
    GraphKey k;
    cudaGraphExec_t exec;
};

struct HostCtx {
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;      // fork / join events for graph capture
    std::vector<GraphEntry> graphs;       // small cache, most recent last
    std::vector<Slot> slots;
    se_report* reps = nullptr;            // device: one report per chunk
    se_report* hreps = nullptr;           // pinned host mirror (async D2H, no per-chunk sync)
    se_report* hinit = nullptr;           // pinned {-1, 0} per chunk: one H2D initialises a report
    size_t reps_cap = 0;
    std::mutex mu;
    se_host_ticket* pending = nullptr;    // the asynchronous call still using this context, if any
};

// One context per (device, direction): a protect and a recover can be in
// flight at the same time (the asynchronous calls below), each with its own
// streams and staging slots.
static HostCtx& host_ctx(int dev, int op) {
    static std::mutex m;
    static std::map<std::pair<int, int>, HostCtx*> ctxs;
    std::lock_guard<std::mutex> g(m);
    HostCtx*& c = ctxs[{dev, op}];
    if (!c) c = new HostCtx();
    return *c;
}

static int ensure(HostCtx& c, uint32_t n_streams) {
    while (c.streams.size() < n_streams) {
        cudaStream_t s;
        cudaEvent_t e;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return SE_ECUDA;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SE_ECUDA;
        c.streams.push_back(s);
        c.events.push_back(e);
        c.slots.emplace_back();
    }
    return SE_OK;
}

static void drop_graphs(HostCtx& c) {
    for (auto& g : c.graphs) cudaGraphExecDestroy(g.exec);
    c.graphs.clear();
}

static bool graphs_enabled() {
    static const bool on = [] {
        const char* e = getenv("SE_HOST_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

static GraphKey make_key(int op, const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* p0,
                         const void* p1, const void* p2, const void* p3, uint64_t chunk_bytes, uint32_t n_streams) {
    GraphKey k;
    memset(&k, 0, sizeof k);
    k.op = op; k.n_streams = n_streams; k.chunk_bytes = chunk_bytes; k.g = *g;
    memcpy(k.key, key, 16); memcpy(k.iv, iv, 16);
    k.ptr[0] = p0; k.ptr[1] = p1; k.ptr[2] = p2; k.ptr[3] = p3;
    return k;
}

static cudaGraphExec_t find_graph(HostCtx& c, const GraphKey& k) {
    for (auto& g : c.graphs)
        if (memcmp(&g.k, &k, sizeof k) == 0) return g.exec;
    return nullptr;
}

// Run issue(streams) either captured into a (cached) graph or directly.
// issue() enqueues every chunk op on c.streams[k % S] and returns a status.
static bool g_graph_broken = false;       // capture unsupported here: issue directly from then on

template <typename F>
static int run_direct(HostCtx& c, uint32_t n_streams, F& issue) {
    int status = issue();
    for (uint32_t i = 0; i < n_streams; ++i)
        if (cudaStreamSynchronize(c.streams[i]) != cudaSuccess) status = SE_ECUDA;
    return status;
}

// Run issue() — which enqueues every chunk op on c.streams[k % S] — either
// captured into a (cached) graph and replayed, or directly.
// Page-locked (or registered) host memory?  Copies from pageable memory are
// staged synchronously by the driver and cannot be captured into a graph.
static bool pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

template <typename F>
static int run_chunks(HostCtx& c, const GraphKey& key, uint32_t n_streams, F issue) {
    if (!graphs_enabled() || g_graph_broken) return run_direct(c, n_streams, issue);
    for (const void* p : key.ptr)
        if (!pinned(p)) return run_direct(c, n_streams, issue);
    cudaStream_t s0 = c.streams[0];
    cudaGraphExec_t exec = find_graph(c, key);
    if (!exec) {
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            g_graph_broken = true;
            return run_direct(c, n_streams, issue);
        }
        cudaEventRecord(c.events[0], s0);                                 // fork
        for (uint32_t i = 1; i < n_streams; ++i) cudaStreamWaitEvent(c.streams[i], c.events[0], 0);
        const int status = issue();
        for (uint32_t i = 1; i < n_streams; ++i) {                        // join
            cudaEventRecord(c.events[i], c.streams[i]);
            cudaStreamWaitEvent(s0, c.events[i], 0);
        }
        const cudaError_t ce = cudaStreamEndCapture(s0, &graph);
        if (status != SE_OK && status != SE_ECUDA) {                      // argument error: report it
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            return status;
        }
        if (ce != cudaSuccess || status != SE_OK || !graph ||
            cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            g_graph_broken = true;
            return run_direct(c, n_streams, issue);
        }
        cudaGraphDestroy(graph);
        if (c.graphs.size() >= 8) {
            cudaGraphExecDestroy(c.graphs.front().exec);
            c.graphs.erase(c.graphs.begin());
        }
        c.graphs.push_back(GraphEntry{key, exec});
    }
    if (cudaGraphLaunch(exec, s0) != cudaSuccess) return SE_ECUDA;
    return cudaStreamSynchronize(s0) == cudaSuccess ? SE_OK : SE_ECUDA;
}

static int grow(void*& p, size_t& cap, size_t need, HostCtx& c) {
    if (need <= cap) return SE_OK;
    drop_graphs(c);                       // cached graphs hold the old pointer
    if (p) cudaFree(p);                   // synchronous, only while the slot grows
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, need) != cudaSuccess) return SE_ECUDA;
    cap = need;
    return SE_OK;
}

// Mapped (zero-copy) mode: the device address of a page-locked host buffer
// (with unified addressing it is the host address itself).
static int mapped_ptr(const void* h, void** d) {
    *d = nullptr;
    if (!h) return SE_OK;
    if (cudaHostGetDevicePointer(d, const_cast<void*>(h), 0) != cudaSuccess) {
        cudaGetLastError();
        return SE_EINVAL;                    // not page-locked / not mapped
    }
    return SE_OK;
}

// Hybrid staging (BLOCK8, page-locked host buffers): inputs go H2D by copy
// engine, the fused kernel writes its outputs straight into the host buffers
// over PCIe, so a chunk is one H2D copy and two kernels and the device-to-
// host direction needs no copy-engine pass after the kernel.  Chunks are
// whole 128-block CTA groups so every slice stays 16-byte aligned.
// SE_HOST_HYBRID bit 0: protect (fragments leave as the CTAs' 128-bit slice
// stores: C2 protect_host 510 -> 475 us, 256 MiB 7.69 -> 7.46 ms); bit 1:
// recover (its 8-byte row stores over PCIe measured slower, 511 -> 541 us
// and 7.44 -> 8.63 ms); bit 2: recover reads its fragment slices from the host
// buffers (zero-copy input; C2 e2e 12.9 -> 12.1 GB/s, slower).  Default 1.
static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static bool hybrid_enabled(int op) {
    static const int mask = [] {
        const char* e = getenv("SE_HOST_HYBRID");
        return e ? atoi(e) : 1;
    }();
    return (mask >> op) & 1;
}

// Finish the asynchronous call still using ctx (if any): wait for all its
// work, keep its chunk reports in the ticket, release the context.
static void settle(HostCtx& c) {
    se_host_ticket* t = c.pending;
    if (!t) return;
    for (cudaEvent_t e : t->tail)
        if (cudaEventSynchronize(e) != cudaSuccess) t->status = SE_ECUDA;
    if (t->op == 1 && t->hreps && !t->collected) {
        t->reps.assign(t->hreps, t->hreps + t->done.size());
        t->collected = true;
    }
    c.pending = nullptr;
}

// Record chunk k's completion on its stream (asynchronous calls).
static int ticket_chunk(se_host_ticket* t, size_t k, cudaStream_t s) {
    if (!t) return SE_OK;
    return cudaEventRecord(t->done[k], s) == cudaSuccess ? SE_OK : SE_ECUDA;
}

// Make stream s wait for every chunk of `after` overlapping blocks [b0, b1).
static int ticket_wait(const se_host_ticket* after, uint64_t b0, uint64_t b1, cudaStream_t s) {
    if (!after) return SE_OK;
    for (size_t j = 0; j < after->done.size(); ++j)
        if (after->blk0[j] < b1 && b0 < after->blk0[j] + after->nblk[j] &&
            cudaStreamWaitEvent(s, after->done[j], 0) != cudaSuccess)
            return SE_ECUDA;
    return SE_OK;
}

static int ticket_open(se_host_ticket* t, int op, HostCtx& c, const std::vector<Chunk>& chunks) {
    if (!t) return SE_OK;
    t->op = op;
    t->ctx = &c;
    for (const Chunk& ch : chunks) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SE_ECUDA;
        t->done.push_back(e);
        t->blk0.push_back(ch.blk0);
        t->nblk.push_back(ch.nblk);
    }
    return SE_OK;
}

// Close an asynchronous call: one tail event per stream it used.
static int ticket_close(se_host_ticket* t, HostCtx& c, uint32_t n_streams) {
    for (uint32_t i = 0; i < n_streams; ++i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SE_ECUDA;
        t->tail.push_back(e);
        if (cudaEventRecord(e, c.streams[i]) != cudaSuccess) return SE_ECUDA;
    }
    c.pending = t;
    return SE_OK;
}

static void ticket_free(se_host_ticket* t) {
    if (!t) return;
    for (cudaEvent_t e : t->done) cudaEventDestroy(e);
    for (cudaEvent_t e : t->tail) cudaEventDestroy(e);
    delete t;
}

}  // namespace se

using namespace se;

extern "C" {

}  // extern "C"

// fragment_protect_host / fragment_protect_host_async.  t != nullptr: the
// asynchronous form (no final synchronisation; chunk events in t).
static int protect_host_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_in,
                             void* h_a, void* h_b, void* h_c, uint64_t chunk_bytes, uint32_t n_streams,
                             se_host_ticket* t) {
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv) return SE_EINVAL;
    if (g->n_bytes == 0) return SE_OK;
    if (!h_in || !h_a || !h_c || (lay.b_bytes && !h_b)) return SE_EINVAL;
    if (g->flags & SE_FLAG_HOST_MAPPED) {      // zero-copy: one pass, the kernels move the bytes over PCIe
        if (g->mode != SE_MODE_BLOCK8) return SE_ENOTSUP;
        void *din, *da, *db, *dc;
        if (mapped_ptr(h_in, &din) || mapped_ptr(h_a, &da) || mapped_ptr(h_b, &db) || mapped_ptr(h_c, &dc))
            return SE_EINVAL;
        se_geom g2 = *g;
        g2.flags &= ~(uint32_t)SE_FLAG_HOST_MAPPED;
        int dev = 0;
        cudaGetDevice(&dev);
        HostCtx& ctx = host_ctx(dev, 0);
        std::lock_guard<std::mutex> lock(ctx.mu);
        settle(ctx);
        if (ensure(ctx, 1)) return SE_ECUDA;
        ImplOpts o;
        o.mapped = true;
        const std::vector<Chunk> one{Chunk{0, g->n_bytes, 0, lay.n_blocks}};
        if (ticket_open(t, 0, ctx, one)) return SE_ECUDA;
        int st = protect_impl(&g2, key, iv, din, da, db, dc, o, ctx.streams[0]);
        if (t) {
            if (st == SE_OK) st = ticket_chunk(t, 0, ctx.streams[0]);
            if (st == SE_OK) st = ticket_close(t, ctx, 1);
            return st;
        }
        if (cudaStreamSynchronize(ctx.streams[0]) != cudaSuccess) st = SE_ECUDA;
        return st;
    }
    if (chunk_bytes == 0) chunk_bytes = auto_chunk(g->n_bytes);
    if (n_streams == 0) n_streams = 3;
    // hybrid: fragments written by the kernels into the (mapped) host buffers
    void* dmap[3] = {nullptr, nullptr, nullptr};
    bool hybrid = hybrid_enabled(0) && g->mode == SE_MODE_BLOCK8 && pinned(h_a) && pinned(h_b) && pinned(h_c) &&
                  aligned16(h_a) && aligned16(h_c) && (!h_b || aligned16(h_b)) && pinned(h_in);
    if (hybrid && (mapped_ptr(h_a, &dmap[0]) || mapped_ptr(h_b, &dmap[1]) || mapped_ptr(h_c, &dmap[2])))
        hybrid = false;
    // FULL mode transforms the whole matrix: one chunk
    const std::vector<Chunk> chunks = g->mode == SE_MODE_FULL
        ? std::vector<Chunk>{Chunk{0, g->n_bytes, 0, lay.n_blocks}}
        : make_chunks(g, lay, chunk_bytes, hybrid ? kBlocksPerCta : 1);
    int dev = 0;
    cudaGetDevice(&dev);
    HostCtx& ctx = host_ctx(dev, 0);
    std::lock_guard<std::mutex> lock(ctx.mu);
    settle(ctx);
    if (ensure(ctx, n_streams)) return SE_ECUDA;
    if (ticket_open(t, 0, ctx, chunks)) return SE_ECUDA;
    const uint32_t bits[3] = {lay.a_bits, lay.b_bits, lay.c_bits};
    uint8_t* hout[3] = {(uint8_t*)h_a, (uint8_t*)h_b, (uint8_t*)h_c};
    std::vector<se_geom> cgs(chunks.size());
    std::vector<se_layout> cls(chunks.size());
    // pass 1: per-chunk geometry and staging capacity (may synchronise and reallocate)
    for (size_t k = 0; k < chunks.size(); ++k) {
        const Chunk& c = chunks[k];
        Slot& sl = ctx.slots[k % n_streams];
        cgs[k] = *g;
        cgs[k].n_bytes = c.byte1 - c.byte0;
        cgs[k].block_offset = g->block_offset + c.blk0;
        fragment_layout(&cgs[k], &cls[k]);
        // staged: input + three fragment slices (+ FULL mode: the coefficient workspace); hybrid: input
        const uint64_t ws = g->mode == SE_MODE_FULL ? cls[k].rows * g->width * sizeof(int16_t) : 0;
        const uint64_t sizes[5] = {cgs[k].n_bytes, hybrid ? 0 : cls[k].a_bytes, hybrid ? 0 : cls[k].b_bytes,
                                   hybrid ? 0 : cls[k].c_bytes, ws};
        for (int i = 0; i < 5; ++i) {
            if (!sizes[i] && i) continue;
            if (sizes[i] + 16 > sl.cap[i]) cudaStreamSynchronize(ctx.streams[k % n_streams]);
            if (grow(sl.buf[i], sl.cap[i], sizes[i] + 16, ctx)) return SE_ECUDA;
        }
    }
    // pass 2: H2D -> keystream + fused kernel -> D2H per chunk, chunk k on stream k mod S
    auto issue = [&]() -> int {
        if (hybrid) {
            for (size_t k = 0; k < chunks.size(); ++k) {
                const Chunk& c = chunks[k];
                cudaStream_t s = ctx.streams[k % n_streams];
                Slot& sl = ctx.slots[k % n_streams];
                if (cudaMemcpyAsync(sl.buf[0], (const uint8_t*)h_in + c.byte0, cgs[k].n_bytes,
                                    cudaMemcpyHostToDevice, s) != cudaSuccess)
                    return SE_ECUDA;
                uint8_t* d[3];
                for (int i = 0; i < 3; ++i) d[i] = dmap[i] ? (uint8_t*)dmap[i] + c.blk0 * bits[i] / 8 : nullptr;
                ImplOpts o;
                o.mapped = true;
                int st = protect_impl(&cgs[k], key, iv, sl.buf[0], d[0], cls[k].b_bytes ? d[1] : nullptr, d[2], o, s);
                if (!st) st = ticket_chunk(t, k, s);
                if (st) return st;
            }
            return SE_OK;
        }
        for (size_t k = 0; k < chunks.size(); ++k) {
            const Chunk& c = chunks[k];
            cudaStream_t s = ctx.streams[k % n_streams];
            Slot& sl = ctx.slots[k % n_streams];
            const se_layout& cl = cls[k];
            const uint64_t sizes[4] = {cgs[k].n_bytes, cl.a_bytes, cl.b_bytes, cl.c_bytes};
            if (cudaMemcpyAsync(sl.buf[0], (const uint8_t*)h_in + c.byte0, sizes[0], cudaMemcpyHostToDevice, s) !=
                cudaSuccess)
                return SE_ECUDA;
            ImplOpts o;
            o.ws = sl.buf[4];
            o.ws_bytes = sl.cap[4];
            int st = protect_impl(&cgs[k], key, iv, sl.buf[0], sl.buf[1], cl.b_bytes ? sl.buf[2] : nullptr,
                                  sl.buf[3], o, s);
            if (st) return st;
            for (int i = 0; i < 3; ++i)
                if (sizes[i + 1] && cudaMemcpyAsync(hout[i] + c.blk0 * bits[i] / 8, sl.buf[i + 1], sizes[i + 1],
                                                    cudaMemcpyDeviceToHost, s) != cudaSuccess)
                    return SE_ECUDA;
            if (ticket_chunk(t, k, s)) return SE_ECUDA;
        }
        return SE_OK;
    };
    if (t) {                                  // asynchronous: issue directly, no final synchronisation
        const int st = issue();
        return st ? st : ticket_close(t, ctx, n_streams);
    }
    const GraphKey gk = make_key(0, g, key, iv, h_in, h_a, h_b, h_c, chunk_bytes, n_streams);
    return run_chunks(ctx, gk, n_streams, issue);
}

extern "C" {

int fragment_protect_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_in,
                          void* h_a, void* h_b, void* h_c, uint64_t chunk_bytes, uint32_t n_streams) {
    SE_RANGE("fragment_protect_host");
    return protect_host_impl(g, key, iv, h_in, h_a, h_b, h_c, chunk_bytes, n_streams, nullptr);
}

int fragment_protect_host_async(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_in,
                                void* h_a, void* h_b, void* h_c, uint64_t chunk_bytes, uint32_t n_streams,
                                se_host_ticket** out) {
    SE_RANGE("fragment_protect_host_async");
    if (!out) return SE_EINVAL;
    *out = nullptr;
    se_host_ticket* t = new se_host_ticket();
    const int st = protect_host_impl(g, key, iv, h_in, h_a, h_b, h_c, chunk_bytes, n_streams, t);
    if (st != SE_OK) {
        HostCtx* c = (HostCtx*)t->ctx;
        if (c && c->pending == t) c->pending = nullptr;
        for (uint32_t i = 0; c && i < c->streams.size(); ++i) cudaStreamSynchronize(c->streams[i]);
        ticket_free(t);
        return st;
    }
    *out = t;
    return SE_OK;
}

}  // extern "C"

// fragment_recover_host / fragment_recover_host_async (t != nullptr; `after`:
// a protect ticket whose chunks must reach host memory before the chunks of
// this call that read them are copied).
static int recover_host_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_a,
                             const void* h_b, const void* h_c, void* h_out, se_report* h_report,
                             uint64_t chunk_bytes, uint32_t n_streams, const se_host_ticket* after,
                             se_host_ticket* t) {
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv) return SE_EINVAL;
    if (h_report) { h_report->first_bad_block = -1; h_report->bad_blocks = 0; }
    if (g->n_bytes == 0) return SE_OK;
    if (!h_out || !h_a || !h_c || (lay.b_bytes && !h_b)) return SE_EINVAL;
    if (g->flags & SE_FLAG_HOST_MAPPED) {      // zero-copy recovery
        if (g->mode != SE_MODE_BLOCK8) return SE_ENOTSUP;
        void *da, *db, *dc, *dout;
        if (mapped_ptr(h_a, &da) || mapped_ptr(h_b, &db) || mapped_ptr(h_c, &dc) || mapped_ptr(h_out, &dout))
            return SE_EINVAL;
        se_geom g2 = *g;
        g2.flags &= ~(uint32_t)SE_FLAG_HOST_MAPPED;
        int dev = 0;
        cudaGetDevice(&dev);
        HostCtx& ctx = host_ctx(dev, 1);
        std::lock_guard<std::mutex> lock(ctx.mu);
        settle(ctx);
        if (ensure(ctx, 1)) return SE_ECUDA;
        if (ctx.reps_cap < 1) {
            drop_graphs(ctx);
            if (cudaMalloc((void**)&ctx.reps, sizeof(se_report)) != cudaSuccess ||
                cudaMallocHost((void**)&ctx.hreps, sizeof(se_report)) != cudaSuccess ||
                cudaMallocHost((void**)&ctx.hinit, sizeof(se_report)) != cudaSuccess)
                return SE_ECUDA;
            ctx.hinit[0].first_bad_block = -1;
            ctx.hinit[0].bad_blocks = 0;
            ctx.reps_cap = 1;
        }
        cudaStream_t s0 = ctx.streams[0];
        ImplOpts o;
        o.mapped = true;
        const std::vector<Chunk> one{Chunk{0, g->n_bytes, 0, lay.n_blocks}};
        if (ticket_open(t, 1, ctx, one) || ticket_wait(after, 0, lay.n_blocks, s0)) return SE_ECUDA;
        int st = recover_impl(&g2, key, iv, da, db, dc, dout, ctx.reps, o, s0);
        if (st == SE_OK &&
            cudaMemcpyAsync(ctx.hreps, ctx.reps, sizeof(se_report), cudaMemcpyDeviceToHost, s0) != cudaSuccess)
            st = SE_ECUDA;
        if (t) {
            t->hreps = ctx.hreps;
            if (st == SE_OK) st = ticket_chunk(t, 0, s0);
            if (st == SE_OK) st = ticket_close(t, ctx, 1);
            return st;
        }
        if (cudaStreamSynchronize(s0) != cudaSuccess) st = SE_ECUDA;
        if (st == SE_OK && h_report) *h_report = ctx.hreps[0];
        return st;
    }
    if (chunk_bytes == 0) chunk_bytes = auto_chunk(g->n_bytes);
    if (n_streams == 0) n_streams = 3;
    // hybrid: the recovered bytes written by the kernels into the (mapped) host buffer
    void* dout = nullptr;
    bool hybrid = hybrid_enabled(1) && g->mode == SE_MODE_BLOCK8 && pinned(h_out) && aligned16(h_out) &&
                  pinned(h_a) && pinned(h_b) && pinned(h_c);
    if (hybrid && mapped_ptr(h_out, &dout)) hybrid = false;
    // zero-copy input: the fused kernels read the fragment slices from the (mapped) host buffers
    void* din[3] = {nullptr, nullptr, nullptr};
    bool zin = hybrid_enabled(2) && g->mode == SE_MODE_BLOCK8 && pinned(h_a) && pinned(h_b) && pinned(h_c) &&
               aligned16(h_a) && aligned16(h_c) && (!h_b || aligned16(h_b));
    if (zin && (mapped_ptr(h_a, &din[0]) || mapped_ptr(h_b, &din[1]) || mapped_ptr(h_c, &din[2]))) zin = false;
    const std::vector<Chunk> chunks = g->mode == SE_MODE_FULL
        ? std::vector<Chunk>{Chunk{0, g->n_bytes, 0, lay.n_blocks}}
        : make_chunks(g, lay, chunk_bytes, (hybrid || zin) ? kBlocksPerCta : 1);
    int dev = 0;
    cudaGetDevice(&dev);
    HostCtx& ctx = host_ctx(dev, 1);
    std::lock_guard<std::mutex> lock(ctx.mu);
    settle(ctx);
    if (ensure(ctx, n_streams)) return SE_ECUDA;
    if (chunks.size() > ctx.reps_cap) {
        for (auto s : ctx.streams) cudaStreamSynchronize(s);
        drop_graphs(ctx);
        if (ctx.reps) cudaFree(ctx.reps);
        if (ctx.hreps) cudaFreeHost(ctx.hreps);
        if (ctx.hinit) cudaFreeHost(ctx.hinit);
        ctx.reps = ctx.hreps = ctx.hinit = nullptr;
        ctx.reps_cap = 0;
        if (cudaMalloc((void**)&ctx.reps, sizeof(se_report) * chunks.size()) != cudaSuccess) return SE_ECUDA;
        if (cudaMallocHost((void**)&ctx.hreps, sizeof(se_report) * chunks.size()) != cudaSuccess) return SE_ECUDA;
        if (cudaMallocHost((void**)&ctx.hinit, sizeof(se_report) * chunks.size()) != cudaSuccess) return SE_ECUDA;
        for (size_t k = 0; k < chunks.size(); ++k) { ctx.hinit[k].first_bad_block = -1; ctx.hinit[k].bad_blocks = 0; }
        ctx.reps_cap = chunks.size();
    }
    const uint32_t bits[3] = {lay.a_bits, lay.b_bits, lay.c_bits};
    const uint8_t* hin[3] = {(const uint8_t*)h_a, (const uint8_t*)h_b, (const uint8_t*)h_c};
    std::vector<se_geom> cgs(chunks.size());
    std::vector<se_layout> cls(chunks.size());
    for (size_t k = 0; k < chunks.size(); ++k) {
        const Chunk& c = chunks[k];
        Slot& sl = ctx.slots[k % n_streams];
        cgs[k] = *g;
        cgs[k].n_bytes = c.byte1 - c.byte0;
        cgs[k].block_offset = g->block_offset + c.blk0;
        fragment_layout(&cgs[k], &cls[k]);
        const uint64_t ws = g->mode == SE_MODE_FULL ? cls[k].rows * g->width * sizeof(int16_t) : 0;
        const uint64_t sizes[5] = {cgs[k].n_bytes, cls[k].a_bytes, cls[k].b_bytes, cls[k].c_bytes, ws};
        for (int i = 0; i < 5; ++i) {
            if (i == 4 && !sizes[i]) continue;
            if (sizes[i] + 16 > sl.cap[i]) cudaStreamSynchronize(ctx.streams[k % n_streams]);
            if (grow(sl.buf[i], sl.cap[i], sizes[i] + 16, ctx)) return SE_ECUDA;
        }
    }
    se_report* reps = ctx.hreps;          // pinned: the per-chunk copies stay asynchronous
    if (ticket_open(t, 1, ctx, chunks)) return SE_ECUDA;
    if (t) t->hreps = ctx.hreps;
    auto issue = [&]() -> int {
        for (size_t k = 0; k < chunks.size(); ++k) {
            const Chunk& c = chunks[k];
            cudaStream_t s = ctx.streams[k % n_streams];
            Slot& sl = ctx.slots[k % n_streams];
            const se_layout& cl = cls[k];
            if (ticket_wait(after, c.blk0, c.blk0 + c.nblk, s)) return SE_ECUDA;
            const uint64_t sizes[4] = {cgs[k].n_bytes, cl.a_bytes, cl.b_bytes, cl.c_bytes};
            const void* src[3] = {sl.buf[1], sl.buf[2], sl.buf[3]};
            for (int i = 0; i < 3; ++i) {
                if (zin) {
                    src[i] = din[i] ? (const uint8_t*)din[i] + c.blk0 * bits[i] / 8 : nullptr;
                } else if (sizes[i + 1] && cudaMemcpyAsync(sl.buf[i + 1], hin[i] + c.blk0 * bits[i] / 8,
                                                           sizes[i + 1], cudaMemcpyHostToDevice, s) != cudaSuccess) {
                    return SE_ECUDA;
                }
            }
            // the chunk's report is initialised by recover_impl (two memsets)
            uint8_t* dst = hybrid ? (uint8_t*)dout + c.byte0 : (uint8_t*)sl.buf[0];
            ImplOpts o;
            o.mapped = hybrid || zin;          // host-mapped buffers: the per-CTA kernels' plain accesses
            o.ws = sl.buf[4];
            o.ws_bytes = sl.cap[4];
            int st = recover_impl(&cgs[k], key, iv, src[0], cl.b_bytes ? src[1] : nullptr, src[2],
                                  dst, ctx.reps + k, o, s);
            if (st) return st;
            if ((!hybrid && cudaMemcpyAsync((uint8_t*)h_out + c.byte0, sl.buf[0], sizes[0], cudaMemcpyDeviceToHost,
                                            s) != cudaSuccess) ||
                cudaMemcpyAsync(&reps[k], ctx.reps + k, sizeof(se_report), cudaMemcpyDeviceToHost, s) != cudaSuccess)
                return SE_ECUDA;
            if (ticket_chunk(t, k, s)) return SE_ECUDA;
        }
        return SE_OK;
    };
    if (t) {                                  // asynchronous: issue directly, no final synchronisation
        const int st = issue();
        return st ? st : ticket_close(t, ctx, n_streams);
    }
    const GraphKey gk = make_key(1, g, key, iv, h_out, h_a, h_b, h_c, chunk_bytes, n_streams);
    int status = run_chunks(ctx, gk, n_streams, issue);
    if (status == SE_OK && h_report) {
        for (size_t k = 0; k < chunks.size(); ++k) {
            if (reps[k].bad_blocks) {
                const int64_t fb = (int64_t)chunks[k].blk0 + reps[k].first_bad_block;
                if (h_report->first_bad_block < 0 || fb < h_report->first_bad_block) h_report->first_bad_block = fb;
                h_report->bad_blocks += reps[k].bad_blocks;
            }
        }
    }
    return status;
}

extern "C" {

int fragment_recover_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_a,
                          const void* h_b, const void* h_c, void* h_out, se_report* h_report, uint64_t chunk_bytes,
                          uint32_t n_streams) {
    SE_RANGE("fragment_recover_host");
    return recover_host_impl(g, key, iv, h_a, h_b, h_c, h_out, h_report, chunk_bytes, n_streams, nullptr, nullptr);
}

int fragment_recover_host_async(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_a,
                                const void* h_b, const void* h_c, void* h_out, uint64_t chunk_bytes,
                                uint32_t n_streams, const se_host_ticket* after, se_host_ticket** out) {
    SE_RANGE("fragment_recover_host_async");
    if (!out) return SE_EINVAL;
    *out = nullptr;
    if (after && after->op != 0) return SE_EINVAL;
    se_host_ticket* t = new se_host_ticket();
    const int st = recover_host_impl(g, key, iv, h_a, h_b, h_c, h_out, nullptr, chunk_bytes, n_streams, after, t);
    if (st != SE_OK) {
        HostCtx* c = (HostCtx*)t->ctx;
        if (c && c->pending == t) c->pending = nullptr;
        for (uint32_t i = 0; c && i < c->streams.size(); ++i) cudaStreamSynchronize(c->streams[i]);
        ticket_free(t);
        return st;
    }
    *out = t;
    return SE_OK;
}

int se_host_wait(se_host_ticket* t, se_report* h_report) {
    SE_RANGE("se_host_wait");
    if (!t) return SE_EINVAL;
    HostCtx* c = (HostCtx*)t->ctx;
    int st;
    {
        std::lock_guard<std::mutex> lock(c->mu);
        if (c->pending == t) settle(*c);
        for (cudaEvent_t e : t->tail)           // settled earlier by a later call: already complete
            if (cudaEventSynchronize(e) != cudaSuccess) t->status = SE_ECUDA;
        st = t->status;
    }
    if (h_report) {
        h_report->first_bad_block = -1;
        h_report->bad_blocks = 0;
        if (t->op == 1 && st == SE_OK) {
            for (size_t k = 0; k < t->reps.size(); ++k) {
                if (t->reps[k].bad_blocks) {
                    const int64_t fb = (int64_t)t->blk0[k] + t->reps[k].first_bad_block;
                    if (h_report->first_bad_block < 0 || fb < h_report->first_bad_block) h_report->first_bad_block = fb;
                    h_report->bad_blocks += t->reps[k].bad_blocks;
                }
            }
        }
    }
    ticket_free(t);
    return st;
}

}  // extern "C"
