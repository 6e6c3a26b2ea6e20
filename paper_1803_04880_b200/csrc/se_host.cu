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
static uint64_t chunk_block_align(const se_layout& lay) {
    uint64_t g = 128 / gcd64(128, lay.a_bits);
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

static std::vector<Chunk> make_chunks(const se_geom* g, const se_layout& lay, uint64_t chunk_bytes) {
    const uint64_t bpr = g->width / 8, block_rows = lay.rows / 8;
    const uint64_t ga = chunk_block_align(lay);
    const uint64_t unit = ga / gcd64(ga, bpr);                 // block-rows per alignment unit
    const uint64_t row_bytes = 8ull * g->width;
    uint64_t rows_per = std::max<uint64_t>(1, chunk_bytes / row_bytes);
    rows_per = std::max<uint64_t>(unit, rows_per / unit * unit);
    std::vector<Chunk> v;
    for (uint64_t br = 0; br < block_rows; br += rows_per) {
        const uint64_t br1 = std::min(block_rows, br + rows_per);
        Chunk c;
        c.byte0 = std::min(g->n_bytes, br * row_bytes);
        c.byte1 = std::min(g->n_bytes, br1 * row_bytes);
        c.blk0 = br * bpr;
        c.nblk = (br1 - br) * bpr;
        v.push_back(c);
    }
    return v;
}

// Per-device streaming context, created on first use and kept for the life of
// the process: S non-blocking streams and one staging slot per stream (device
// buffers for one chunk's input / output and its three fragment slices, grown
// on demand).  Chunk k uses slot k mod S on stream k mod S, so stream order
// alone makes slot reuse safe; steady-state calls allocate nothing.
struct Slot {
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};   // bytes, A, B, C
    size_t cap[4] = {0, 0, 0, 0};
};

struct HostCtx {
    std::vector<cudaStream_t> streams;
    std::vector<Slot> slots;
    se_report* reps = nullptr;
    size_t reps_cap = 0;
    std::mutex mu;
};

static HostCtx& host_ctx(int dev) {
    static std::mutex m;
    static std::map<int, HostCtx*> ctxs;
    std::lock_guard<std::mutex> g(m);
    HostCtx*& c = ctxs[dev];
    if (!c) c = new HostCtx();
    return *c;
}

static int ensure(HostCtx& c, uint32_t n_streams) {
    while (c.streams.size() < n_streams) {
        cudaStream_t s;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return SE_ECUDA;
        c.streams.push_back(s);
        c.slots.emplace_back();
    }
    return SE_OK;
}

static int grow(void*& p, size_t& cap, size_t need) {
    if (need <= cap) return SE_OK;
    if (p) cudaFree(p);                   // synchronous, only while the slot grows
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, need) != cudaSuccess) return SE_ECUDA;
    cap = need;
    return SE_OK;
}

}  // namespace se

using namespace se;

extern "C" {

int fragment_protect_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_in,
                          void* h_a, void* h_b, void* h_c, uint64_t chunk_bytes, uint32_t n_streams) {
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv) return SE_EINVAL;
    if (g->n_bytes == 0) return SE_OK;
    if (!h_in || !h_a || !h_c || (lay.b_bytes && !h_b)) return SE_EINVAL;
    if (chunk_bytes == 0) chunk_bytes = 32ull << 20;
    if (n_streams == 0) n_streams = 3;
    // FULL mode transforms the whole matrix: one chunk
    const std::vector<Chunk> chunks = g->mode == SE_MODE_FULL
        ? std::vector<Chunk>{Chunk{0, g->n_bytes, 0, lay.n_blocks}} : make_chunks(g, lay, chunk_bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    HostCtx& ctx = host_ctx(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (ensure(ctx, n_streams)) return SE_ECUDA;
    const uint32_t bits[3] = {lay.a_bits, lay.b_bits, lay.c_bits};
    uint8_t* hout[3] = {(uint8_t*)h_a, (uint8_t*)h_b, (uint8_t*)h_c};
    int status = SE_OK;
    for (size_t k = 0; k < chunks.size() && status == SE_OK; ++k) {
        const Chunk& c = chunks[k];
        cudaStream_t s = ctx.streams[k % n_streams];
        Slot& sl = ctx.slots[k % n_streams];
        se_geom cg = *g;
        cg.n_bytes = c.byte1 - c.byte0;
        cg.block_offset = g->block_offset + c.blk0;
        se_layout cl;
        fragment_layout(&cg, &cl);
        const uint64_t sizes[4] = {cg.n_bytes, cl.a_bytes, cl.b_bytes, cl.c_bytes};
        for (int i = 0; i < 4 && status == SE_OK; ++i) {
            if (sizes[i] > sl.cap[i]) cudaStreamSynchronize(s);          // slot busy until its stream drains
            status = grow(sl.buf[i], sl.cap[i], sizes[i] + 16);
        }
        if (status == SE_OK &&
            cudaMemcpyAsync(sl.buf[0], (const uint8_t*)h_in + c.byte0, cg.n_bytes, cudaMemcpyHostToDevice, s) !=
                cudaSuccess)
            status = SE_ECUDA;
        if (status == SE_OK)
            status = fragment_protect(&cg, key, iv, sl.buf[0], sl.buf[1], cl.b_bytes ? sl.buf[2] : nullptr,
                                      sl.buf[3], s);
        for (int i = 0; i < 3 && status == SE_OK; ++i)
            if (sizes[i + 1] && cudaMemcpyAsync(hout[i] + c.blk0 * bits[i] / 8, sl.buf[i + 1], sizes[i + 1],
                                                cudaMemcpyDeviceToHost, s) != cudaSuccess)
                status = SE_ECUDA;
    }
    for (uint32_t i = 0; i < n_streams; ++i)
        if (cudaStreamSynchronize(ctx.streams[i]) != cudaSuccess) status = SE_ECUDA;
    return status;
}

int fragment_recover_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* h_a,
                          const void* h_b, const void* h_c, void* h_out, se_report* h_report, uint64_t chunk_bytes,
                          uint32_t n_streams) {
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv) return SE_EINVAL;
    if (h_report) { h_report->first_bad_block = -1; h_report->bad_blocks = 0; }
    if (g->n_bytes == 0) return SE_OK;
    if (!h_out || !h_a || !h_c || (lay.b_bytes && !h_b)) return SE_EINVAL;
    if (chunk_bytes == 0) chunk_bytes = 32ull << 20;
    if (n_streams == 0) n_streams = 3;
    const std::vector<Chunk> chunks = g->mode == SE_MODE_FULL
        ? std::vector<Chunk>{Chunk{0, g->n_bytes, 0, lay.n_blocks}} : make_chunks(g, lay, chunk_bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    HostCtx& ctx = host_ctx(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (ensure(ctx, n_streams)) return SE_ECUDA;
    if (chunks.size() > ctx.reps_cap) {
        for (auto s : ctx.streams) cudaStreamSynchronize(s);
        if (ctx.reps) cudaFree(ctx.reps);
        ctx.reps = nullptr;
        ctx.reps_cap = 0;
        if (cudaMalloc((void**)&ctx.reps, sizeof(se_report) * chunks.size()) != cudaSuccess) return SE_ECUDA;
        ctx.reps_cap = chunks.size();
    }
    const uint32_t bits[3] = {lay.a_bits, lay.b_bits, lay.c_bits};
    const uint8_t* hin[3] = {(const uint8_t*)h_a, (const uint8_t*)h_b, (const uint8_t*)h_c};
    std::vector<se_report> reps(chunks.size());
    int status = SE_OK;
    for (size_t k = 0; k < chunks.size() && status == SE_OK; ++k) {
        const Chunk& c = chunks[k];
        cudaStream_t s = ctx.streams[k % n_streams];
        Slot& sl = ctx.slots[k % n_streams];
        se_geom cg = *g;
        cg.n_bytes = c.byte1 - c.byte0;
        cg.block_offset = g->block_offset + c.blk0;
        se_layout cl;
        fragment_layout(&cg, &cl);
        const uint64_t sizes[4] = {cg.n_bytes, cl.a_bytes, cl.b_bytes, cl.c_bytes};
        for (int i = 0; i < 4 && status == SE_OK; ++i) {
            if (sizes[i] > sl.cap[i]) cudaStreamSynchronize(s);
            status = grow(sl.buf[i], sl.cap[i], sizes[i] + 16);
        }
        for (int i = 0; i < 3 && status == SE_OK; ++i)
            if (sizes[i + 1] && cudaMemcpyAsync(sl.buf[i + 1], hin[i] + c.blk0 * bits[i] / 8, sizes[i + 1],
                                                cudaMemcpyHostToDevice, s) != cudaSuccess)
                status = SE_ECUDA;
        if (status == SE_OK)
            status = fragment_recover(&cg, key, iv, sl.buf[1], cl.b_bytes ? sl.buf[2] : nullptr, sl.buf[3],
                                      sl.buf[0], ctx.reps + k, s);
        if (status == SE_OK &&
            cudaMemcpyAsync((uint8_t*)h_out + c.byte0, sl.buf[0], cg.n_bytes, cudaMemcpyDeviceToHost, s) !=
                cudaSuccess)
            status = SE_ECUDA;
        if (status == SE_OK &&
            cudaMemcpyAsync(&reps[k], ctx.reps + k, sizeof(se_report), cudaMemcpyDeviceToHost, s) != cudaSuccess)
            status = SE_ECUDA;
    }
    for (uint32_t i = 0; i < n_streams; ++i)
        if (cudaStreamSynchronize(ctx.streams[i]) != cudaSuccess) status = SE_ECUDA;
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

}  // extern "C"
