// k_tile.cu — persistent, warp-specialised BLOCK8 protect / recover of one
// file (rows a1-a10 of SURVEY.md §8.1), sm_100a.
//
// One CTA per SM, looping over tiles of TILE consecutive 8x8 blocks (512 at
// L = 2, 3; 256 at L = 1), one block per consumer thread.  Roles:
//   * consumer warps (TILE/32): each thread lifts its block in registers
//     (Eq. 5.1-5.2), packs the A/B/C records, masks B and
//     C with SHA-256 / SHA-512, and writes its records into the
//     tile's stream slices in shared memory;
//   * AES warps (5): AES-128-CTR keystream of each tile's A slice (P:2117,
//     reading C12/C13) into a ring in shared memory, computed from the kernel
//     parameters alone, ahead of the consumers (a 160-block tile slice at
//     L = 2 is exactly one AES block per AES lane);
//   * one elected consumer thread moves the data: TMA bulk copies
//     (cp.async.bulk) bring tile k+2's input into a two-stage ring while tile
//     k is computed, and bulk stores write the finished stream slices (or, in
//     recovery, the tile's bytes) from shared memory.
// The private fragment is encrypted on its way into shared memory and never
// reaches HBM in plaintext; no keystream kernel, no device scratch.
//
// Programmatic dependent launch: the AES warps and the table setup run
// before griddepcontrol.wait; consumers wait before any global access.
//
// Tiles whose bytes do not all lie inside the file (the ragged end), or files
// whose width is not a multiple of 16 bytes (no 16-byte aligned rows for the
// bulk copies), take the per-thread load / store path of fused_cta.cuh inside
// the same loop.
#include <cuda_runtime.h>

#include <algorithm>

#include "fused_cta.cuh"

// SE_TILE_LUT_BY_AES 1: only the AES warps fill the lane table, the consumers
// start their bulk copies at once.  Measured slower (tools/gpu_r2_call58.sh:
// C4 PUBLIC_PLAIN 852 -> 832 GB/s, C2 / C3 lower too), so 0.
// AES warps of the PUBLIC_PLAIN tile kernels.  Measured (tools/gpu_r2_call61.sh):
// 4 -> 859 GB/s C4 round trip, 3 / 2 -> 737 / 736 (the keystream falls
// behind: 120 AES blocks per tile need one pass of 128 lanes); the mbarrier
// suspend hint (1000 / 4000 / 20000 ns) makes no difference.
#ifndef SE_TILE_NAW_PLAIN
#define SE_TILE_NAW_PLAIN 4
#endif
#ifndef SE_TILE_LUT_BY_AES
#define SE_TILE_LUT_BY_AES 0
#endif
#ifndef SE_TILE_ORV_IMAD
#define SE_TILE_ORV_IMAD 1      // measured: C4 PUBLIC_PLAIN recover 0.654 -> 0.638 ms (tools/gpu_r2_call38.sh)
#endif

namespace se {

// TILE: masked kernels (ALU-bound on SHA-2) 512 blocks = 16 consumer warps;
// PUBLIC_PLAIN kernels (issue-bound) 384 blocks = 12 consumer warps, so the
// tile's 120 AES blocks (L = 2) are one pass of the 4 AES warps and keep
// ahead of the consumers (at 512, the 160-block second pass on one warp fell
// behind: consumers spun ~100 mbarrier polls per tile waiting for keystream).
template <int L, bool MASK>
struct TileCfg {
    using R = Rec<L>;
    static constexpr int TILE = (L == 1) ? 256 : MASK ? 512 : 384;
    static constexpr int NCW = TILE / 32;
    // AES warps.  masked: 20 warps = 5 per SM sub-partition: 96 registers per
    // thread.  PUBLIC_PLAIN: SE_TILE_NAW_PLAIN.
    static constexpr int NAW = MASK ? 4 : SE_TILE_NAW_PLAIN;
    static constexpr int NC = 32 * NCW;
    static constexpr int NT = 32 * (NCW + NAW);
    static constexpr int A_BYTES = TILE * R::ABITS / 8;
    static constexpr int B_BYTES = TILE * R::BBITS / 8;
    static constexpr int C_BYTES = TILE * R::CBITS / 8;
    static constexpr int REC_BYTES = A_BYTES + B_BYTES + C_BYTES;
    static constexpr int IN_BYTES = TILE * 64;
    static constexpr int NS = 2;      // input stages
    static constexpr int KS = 4;      // keystream slots
    static constexpr int AES_BLOCKS = A_BYTES / 16;
    static_assert(A_BYTES % 16 == 0 && B_BYTES % 16 == 0 && C_BYTES % 16 == 0, "16-byte slices");
    __host__ __device__ static constexpr int al(int x) { return (x + 127) / 128 * 128; }
    // shared memory carve (bytes): lut | in[NS] | stage[2] | ks[KS] | barriers
    template <bool REC>
    struct Smem {
        static constexpr int IN = REC ? REC_BYTES : IN_BYTES;
        static constexpr int OUT = REC ? IN_BYTES : REC_BYTES;
        static constexpr int LUT_OFF = 0;
        static constexpr int IN_OFF = kAesLutBytes;
        static constexpr int OUT_OFF = IN_OFF + NS * al(IN);
        static constexpr int KS_OFF = OUT_OFF + 2 * al(OUT);
        static constexpr int BAR_OFF = KS_OFF + KS * al(A_BYTES);
        static constexpr int BYTES = BAR_OFF + 8 * (NS + 2 * KS) + 16;
    };
};

// ---------------------------------------------------------------- PTX helpers

#ifndef SE_MBAR_SUSPEND_NS
#define SE_MBAR_SUSPEND_NS 4000
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps (up to the hint)
// until the phase completes instead of re-polling, which cost ~30 issue slots
// per block in the PUBLIC_PLAIN kernels
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p;}"
                     : "=r"(done) : "r"(bar), "r"(parity), "n"(SE_MBAR_SUSPEND_NS) : "memory");
    } while (!done);
}
// global -> shared bulk copy, completion counted on `bar` (bytes and addresses 16-aligned)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void named_bar() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- tile geometry

// Tile t's bytes in shared memory: row i of tile-local block u at
// base(u) + i * stride.  "contiguous": W/8 divides TILE, so the tile is whole
// block rows, one contiguous range of the file, copied as is (stride W);
// else "runs": row i of the tile at i * 8*TILE, block u at 8u (stride 8*TILE),
// one bulk copy per (block-row run, pixel row).
struct TileMap {
    bool contig;
    // contiguous: u = brl * bpr + bc -> 8W*brl + 8bc = 8u + 7W*brl, brl = u / bpr
    // by multiply-shift (p.bpr_magic = ceil(2^20 / bpr), exact for u < 2^10)
    __device__ __forceinline__ uint32_t base(const FusedParams& p, uint64_t, uint32_t u, int) const {
        if (contig) return 8u * u + 7u * p.width * ((u * p.bpr_magic) >> 20);
        return 8u * u;
    }
    __device__ __forceinline__ uint32_t stride(const FusedParams& p, int tile) const {
        return contig ? p.width : 8u * tile;
    }
};

// Issue (protect: load; recover: store) the bulk copies of tile t's bytes
// between the file at `g` and shared memory at `s`.
template <int TILE, bool LOAD>
__device__ __forceinline__ void tile_bytes_copy(const FusedParams& p, const TileMap& m, uint64_t t, uint32_t s,
                                                uint8_t* g, uint32_t bar) {
    const uint64_t b0 = t * TILE;
    if (m.contig) {
        const uint64_t off = (b0 / p.bpr) * 8ull * p.width;
        if (LOAD) bulk_g2s(s, g + off, TILE * 64, bar);
        else bulk_s2g(g + off, s, TILE * 64);
        return;
    }
    uint64_t b = b0;
    const uint64_t end = b0 + TILE;
    while (b < end) {
        const uint64_t br = b / p.bpr, bc = b - br * p.bpr;
        const uint64_t len = min(end - b, (uint64_t)p.bpr - bc);
#pragma unroll 1
        for (int i = 0; i < 8; ++i) {
            uint8_t* gp = g + (8 * br + i) * (uint64_t)p.width + 8 * bc;
            const uint32_t sp = s + i * (8u * TILE) + 8u * (uint32_t)(b - b0);
            if (LOAD) bulk_g2s(sp, gp, (uint32_t)len * 8, bar);
            else bulk_s2g(gp, sp, (uint32_t)len * 8);
        }
        b += len;
    }
}

// ---------------------------------------------------------------- AES producer warps

template <int L, bool MASK>
__device__ __forceinline__ void aes_producer(const FusedParams& p, const uint32_t* lut, uint8_t* ks_base,
                                             uint32_t ks_full, uint32_t ks_empty) {
    using T = TileCfg<L, MASK>;
    const AesLane al = aes_lane(lut);
    const int at = threadIdx.x - T::NC;                  // 0 .. 32*NAW-1
    uint32_t k = 0;
    for (uint64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++k) {
        const uint32_t slot = k % T::KS;
        mbar_wait(ks_empty + 8 * slot, ((k / T::KS) & 1) ^ 1);
        uint32_t* ks = reinterpret_cast<uint32_t*>(ks_base + slot * T::al(T::A_BYTES));
        const uint64_t a0 = t * T::A_BYTES;                 // tile's byte offset in the A stream
        const uint32_t nblk = (uint32_t)min((uint64_t)T::AES_BLOCKS, (p.a_bytes - a0 + 15) / 16);
        for (uint32_t j = at; j < nblk; j += 32 * T::NAW) {
            uint32_t x[4];
            ctr_add(p.ctr, a0 / 16 + j, x);
            aes128_block(al, p.rk, x);
            *reinterpret_cast<uint4*>(ks + 4 * j) = make_uint4(bswap32(x[0]), bswap32(x[1]), bswap32(x[2]),
                                                               bswap32(x[3]));
        }
        mbar_arrive(ks_full + 8 * slot);
    }
}

// ---------------------------------------------------------------- the kernel

template <int L, bool MASK, bool RECOVER>
__global__ void __launch_bounds__(TileCfg<L, MASK>::NT, 1) k_tile(const __grid_constant__ FusedParams p) {
    using T = TileCfg<L, MASK>;
    using R = Rec<L>;
    using S = typename T::template Smem<RECOVER>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* lut = reinterpret_cast<uint32_t*>(smem + S::LUT_OFF);
    const uint32_t bar0 = smem_u32(smem + S::BAR_OFF);
    const uint32_t full = bar0, ks_full = bar0 + 8 * T::NS, ks_empty = ks_full + 8 * T::KS;
    __shared__ unsigned long long s_first;
    __shared__ unsigned int s_bad;

    if (threadIdx.x == 0) {
        for (int s = 0; s < T::NS; ++s) mbar_init(full + 8 * s, 1);
        for (int s = 0; s < T::KS; ++s) {
            mbar_init(ks_full + 8 * s, 32 * T::NAW);
            mbar_init(ks_empty + 8 * s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_first = ~0ull;
        s_bad = 0;
    }
#if SE_TILE_LUT_BY_AES
    // the AES warps fill their table alone (bar 2 among them) while the
    // consumers go straight to their first bulk copies
    __syncthreads();                                      // barrier init visible
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x >= T::NC) {                           // AES warps
        aes_load_lut(lut, threadIdx.x - T::NC, 32 * T::NAW);   // constant tables only
        asm volatile("bar.sync 2, %0;" ::"n"(32 * T::NAW) : "memory");
        aes_producer<L, MASK>(p, lut, smem + S::KS_OFF, ks_full, ks_empty);
        return;
    }
#else
    aes_load_lut(lut, threadIdx.x, T::NT);               // constant tables only: before the grid dependency
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x >= T::NC) {                           // AES warps
        aes_producer<L, MASK>(p, lut, smem + S::KS_OFF, ks_full, ks_empty);
        return;
    }
#endif

    // ---- consumers
    asm volatile("griddepcontrol.wait;" ::: "memory");   // inputs written / buffers read by earlier work
    const int ct = threadIdx.x;
    const TileMap map{(uint32_t)T::TILE % p.bpr == 0};
    const uint32_t in_s = smem_u32(smem + S::IN_OFF);
    constexpr uint32_t IN_STRIDE = T::al(S::IN);
    auto is_fast = [&](uint64_t t) { return t < p.fast_tiles; };
    auto issue_in = [&](uint64_t t, uint32_t slot) {
        const uint32_t dst = in_s + slot * IN_STRIDE, bar = full + 8 * slot;
        if constexpr (RECOVER) {
            mbar_expect_tx(bar, T::REC_BYTES);
            bulk_g2s(dst, p.a + t * T::A_BYTES, T::A_BYTES, bar);
            if (T::B_BYTES) bulk_g2s(dst + T::A_BYTES, p.b + t * T::B_BYTES, T::B_BYTES, bar);
            bulk_g2s(dst + T::A_BYTES + T::B_BYTES, p.c + t * T::C_BYTES, T::C_BYTES, bar);
        } else {
            mbar_expect_tx(bar, T::IN_BYTES);
            tile_bytes_copy<T::TILE, true>(p, map, t, dst, const_cast<uint8_t*>(p.in), bar);
        }
    };
    if (ct == 0) {
        uint64_t t = blockIdx.x;
        for (int s = 0; s < T::NS && t < p.n_tiles; ++s, t += gridDim.x)
            if (is_fast(t)) issue_in(t, s);
    }
    uint32_t phase = 0;                                   // bit s: parity of input slot s's next completion
    uint32_t k = 0;
    for (uint64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++k) {
        const uint32_t slot = k % T::NS, ob = k & 1, kslot = k % T::KS;
        const bool fast = is_fast(t);
        uint8_t* in = smem + S::IN_OFF + slot * IN_STRIDE;
        uint8_t* out = smem + S::OUT_OFF + ob * T::al(S::OUT);
        const uint32_t* ks = reinterpret_cast<const uint32_t*>(smem + S::KS_OFF + kslot * T::al(T::A_BYTES));
        const uint64_t blk = t * T::TILE + ct;
        const bool valid = blk < p.n_blocks;
        const uint64_t gb = p.block_offset + blk;
        if (fast) {
            mbar_wait(full + 8 * slot, (phase >> slot) & 1);
            phase ^= 1u << slot;
        }
        if constexpr (!RECOVER) {
            // ---------------- protect: rows a1-a9
            uint32_t A[R::AW], B[R::BW], C[R::CW];
#pragma unroll
            for (int q = 0; q < R::AW; ++q) A[q] = 0;
#pragma unroll
            for (int q = 0; q < R::BW; ++q) B[q] = 0;
#pragma unroll
            for (int q = 0; q < R::CW; ++q) C[q] = 0;
            if (valid) {
                int v[8][8];
                if (fast) {
                    const uint32_t base = map.base(p, t, ct, T::TILE), st = map.stride(p, T::TILE);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint2 q = *reinterpret_cast<const uint2*>(in + base + i * st);
                        if (MASK) {
                            unpack4(q.x, v[i][0], v[i][1], v[i][2], v[i][3]);
                            unpack4(q.y, v[i][4], v[i][5], v[i][6], v[i][7]);
                        } else {                  // one PRMT per byte (the shift-and-mask form takes two)
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                v[i][j] = (int)__byte_perm(q.x, 0, 0x4440 | j);
                                v[i][4 + j] = (int)__byte_perm(q.y, 0, 0x4440 | j);
                            }
                        }
                    }
                } else {
                    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
                    load_block(p.in, p.n_bytes, p.width, br, bc, v);
                }
                if (MASK) dwt8_fwd<L>(v, p.one);                                  // rows a2-a4 (adds on the FMA pipe)
                else dwt8_fwd_lean<L>(v, p.one);                                  // rows a2-a4 (fewest instructions)
                for_each_field<L, 0>([&](int s, int pos, int i, int j, int w) {     // row a5
                    // C9 (+ C8 on LL); the mixed-pipe forward lifting leaves +1 on every band but LL
                    const int off = (s == 0) ? (1 << (w - 1)) - 128 : (1 << (w - 1)) - (MASK ? 0 : (SE_LEAN_MIX & 1));
                    if (MASK) {
                        if (s == 0) put_field(A, pos, v[i][j], off, w, p.one);
                        else if (s == 1) put_field(B, pos, v[i][j], off, w, p.one);
                        else put_field(C, pos, v[i][j], off, w, p.one);
                    } else {
                        if (s == 0) put_field_lean(A, pos, v[i][j], off, w, p.one);
                        else if (s == 1) put_field_lean(B, pos, v[i][j], off, w, p.one);
                        else put_field_lean(C, pos, v[i][j], off, w, p.one);
                    }
                });
                if (MASK) {
                    if (R::BBITS) {
                        mask_b<L, 0>(p, gb, A, B);                                // row a7
                        mask_c<R::BW, R::BBYTES>(p, gb, B, C);                    // row a8
                    } else {
                        mask_c<R::AW, R::ABYTES>(p, gb, A, C);                    // C21 (L = 1)
                    }
                }
            }
            // row a9 (+ a6): records into the tile's stream slices, A' = A ^ keystream
            uint32_t* sw = reinterpret_cast<uint32_t*>(out);
            mbar_wait(ks_full + 8 * kslot, (k / T::KS) & 1);
            put_stream<R::ABITS, R::AW>(sw, ks, A, ct);
            if (R::BBITS) put_stream<R::BBITS, R::BW>(sw + T::A_BYTES / 4, nullptr, B, ct);
            put_stream<R::CBITS, R::CW>(sw + (T::A_BYTES + T::B_BYTES) / 4, nullptr, C, ct);
        } else {
            // ---------------- recover: row a10
            if (!fast) {
                // ragged end: copy the tile's (partial) slices, zero filled
                const uint64_t a0 = t * T::A_BYTES, b0 = t * T::B_BYTES, c0 = t * T::C_BYTES;
                uint32_t* s32 = reinterpret_cast<uint32_t*>(in);
                copy_g2s<T::NC>(s32, p.a + a0, min((uint64_t)T::A_BYTES, p.a_bytes - a0), T::A_BYTES, ct);
                if (T::B_BYTES)
                    copy_g2s<T::NC>(s32 + T::A_BYTES / 4, p.b + b0, min((uint64_t)T::B_BYTES, p.b_bytes - b0),
                                    T::B_BYTES, ct);
                copy_g2s<T::NC>(s32 + (T::A_BYTES + T::B_BYTES) / 4, p.c + c0,
                                min((uint64_t)T::C_BYTES, p.c_bytes - c0), T::C_BYTES, ct);
                named_bar<T::NC>();
            }
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(in);
            uint32_t A[R::AW], B[R::BW], C[R::CW];
            bool bad = false;
            if (valid) {
                if (R::BBITS) get_stream<R::BBITS, R::BW>(sw + T::A_BYTES / 4, nullptr, (uint32_t)ct, B);
                else B[0] = 0;
                get_stream<R::CBITS, R::CW>(sw + (T::A_BYTES + T::B_BYTES) / 4, nullptr, (uint32_t)ct, C);
                if (MASK && R::BBITS) mask_c<R::BW, R::BBYTES>(p, gb, B, C);      // C from B' (C19)
            }
            mbar_wait(ks_full + 8 * kslot, (k / T::KS) & 1);
            if (valid) {
                get_stream<R::ABITS, R::AW>(sw, ks, (uint32_t)ct, A);              // A = A' ^ keystream
                if (MASK) {
                    if (R::BBITS) mask_b<L, 0>(p, gb, A, B);                      // B from A
                    else mask_c<R::AW, R::ABYTES>(p, gb, A, C);                   // C21 (L = 1)
                }
                int v[8][8];
                if (MASK) {
                    for_each_field<L, 0>([&](int s, int pos, int i, int j, int w) {
                        const int off = (s == 0) ? (1 << (w - 1)) - 128 : (1 << (w - 1));
                        if (s == 0) v[i][j] = get_field(A, pos, off, w, p.one);
                        else if (s == 1) v[i][j] = get_field(B, pos, off, w, p.one);
                        else v[i][j] = get_field(C, pos, off, w, p.one);
                    });
                    dwt8_inv<L>(v, p.one);
                } else {
                    for_each_field<L, 0>([&](int s, int pos, int, int, int) {
                        if (s == 0) flip_top(A, pos);
                        else if (s == 1) flip_top(B, pos);
                        else flip_top(C, pos);
                    });
                    for_each_field<L, 0>([&](int s, int pos, int i, int j, int w) {
                        if (s == 0) v[i][j] = get_field_lean(A, pos, w, p.one) + 128;   // LL: uncentered (C8)
                        else if (s == 1) v[i][j] = get_field_lean(B, pos, w, p.one);
                        else v[i][j] = get_field_lean(C, pos, w, p.one);
                    });
                    dwt8_inv_lean<L>(v, p.one);
                }
                // a reconstructed sample outside [0, 255]?
#if SE_TILE_ORV_IMAD
                bad = out_of_range_pairs(v, p.one);
#else
                int orv = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) orv |= v[i][j];
                bad = (orv & ~0xff) != 0;
#endif
                if (fast) {
                    const uint32_t base = map.base(p, t, ct, T::TILE), st = map.stride(p, T::TILE);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        uint2 q;
                        q.x = __byte_perm(__byte_perm(v[i][0], v[i][1], 0x0040), __byte_perm(v[i][2], v[i][3], 0x0040), 0x5410);
                        q.y = __byte_perm(__byte_perm(v[i][4], v[i][5], 0x0040), __byte_perm(v[i][6], v[i][7], 0x0040), 0x5410);
                        *reinterpret_cast<uint2*>(out + base + i * st) = q;
                    }
                } else {
                    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
                    store_block(p.out, p.n_bytes, p.width, br, bc, v);
                }
            }
            if (p.report != nullptr) {
                const uint32_t m = __ballot_sync(0xffffffffu, bad);
                if (m) {
                    if ((ct & 31) == __ffs(m) - 1) {
                        atomicMin(&s_first, (unsigned long long)blk);
                        atomicAdd(&s_bad, (unsigned)__popc(m));
                    }
                }
            }
        }
        fence_async_smem();                                  // generic smem writes -> bulk stores
        if (ct == 0) bulk_wait_read0();                      // tile k-1's stores have read stage[ob ^ 1]
        named_bar<T::NC>();                                  // stage[ob] complete; in[slot] and ks[kslot] consumed
        if (ct == 0) {
            mbar_arrive(ks_empty + 8 * kslot);
            if (fast) {
                if constexpr (RECOVER) {
                    tile_bytes_copy<T::TILE, false>(p, map, t, smem_u32(out), p.out, 0);
                } else {
                    const uint32_t so = smem_u32(out);
                    bulk_s2g(p.a + t * T::A_BYTES, so, T::A_BYTES);
                    if (T::B_BYTES) bulk_s2g(p.b + t * T::B_BYTES, so + T::A_BYTES, T::B_BYTES);
                    bulk_s2g(p.c + t * T::C_BYTES, so + T::A_BYTES + T::B_BYTES, T::C_BYTES);
                }
                bulk_commit();
            }
            const uint64_t tn = t + (uint64_t)T::NS * gridDim.x;
            if (tn < p.n_tiles && is_fast(tn)) issue_in(tn, slot);
        }
        if constexpr (!RECOVER) {
            if (!fast) {                                     // ragged end: partial slices by all consumers
                const uint32_t* so = reinterpret_cast<const uint32_t*>(out);
                const uint64_t a0 = t * T::A_BYTES, b0 = t * T::B_BYTES, c0 = t * T::C_BYTES;
                copy_s2g<T::NC>(p.a + a0, so, min((uint64_t)T::A_BYTES, p.a_bytes - a0), ct);
                if (T::B_BYTES) copy_s2g<T::NC>(p.b + b0, so + T::A_BYTES / 4, min((uint64_t)T::B_BYTES, p.b_bytes - b0), ct);
                copy_s2g<T::NC>(p.c + c0, so + (T::A_BYTES + T::B_BYTES) / 4, min((uint64_t)T::C_BYTES, p.c_bytes - c0), ct);
            }
        }
    }
    if constexpr (RECOVER) {
        if (p.report != nullptr) {
            named_bar<T::NC>();                              // every consumer's report update is in s_bad / s_first
            if (ct == 0 && s_bad) {
                atomicMin(reinterpret_cast<unsigned long long*>(&p.report->first_bad_block), s_first);
                atomicAdd(reinterpret_cast<unsigned long long*>(&p.report->bad_blocks), (unsigned long long)s_bad);
            }
        }
    }
    if (ct == 0) bulk_wait0();                               // all bulk stores complete before exit
}

// ---------------------------------------------------------------- launcher

static int sm_count() {
    static int count[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && count[dev] == 0) cudaDeviceGetAttribute(&count[dev], cudaDevAttrMultiProcessorCount, dev);
    return dev < 64 ? count[dev] : 148;
}

template <int L, bool MASK, bool RECOVER>
static void tile_l(FusedParams p, cudaStream_t s) {
    using T = TileCfg<L, MASK>;
    using S = typename T::template Smem<RECOVER>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !attr_set[dev]) {
        cudaFuncSetAttribute(k_tile<L, MASK, RECOVER>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES);
        if (dev < 64) attr_set[dev] = true;
    }
    p.n_tiles = (p.n_blocks + T::TILE - 1) / T::TILE;
    // fast tiles: whole tiles whose bytes all lie inside the file, on 16-byte aligned rows
    uint64_t fast = 0;
    if (p.width % 16 == 0) {
        fast = p.n_blocks / T::TILE;
        while (fast > 0) {
            const uint64_t last = fast * T::TILE - 1, br = last / p.bpr, bc = last % p.bpr;
            if ((8 * br + 7) * (uint64_t)p.width + 8 * bc + 7 < p.n_bytes) break;
            --fast;
        }
    }
    p.fast_tiles = fast;
    p.bpr_magic = (uint32_t)(((1u << 20) + p.bpr - 1) / p.bpr);
    const unsigned grid = (unsigned)std::min<uint64_t>(p.n_tiles, (uint64_t)sm_count());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(T::NT);
    cfg.dynamicSmemBytes = S::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_tile<L, MASK, RECOVER>, p);
}

int launch_tile_block8(const FusedParams& p, uint32_t levels, bool mask, bool recover, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (p.n_blocks == 0) return 0;
#define SE_TILE_CASE(LL)                                                           \
    if (levels == LL) {                                                            \
        if (recover) mask ? tile_l<LL, true, true>(p, s) : tile_l<LL, false, true>(p, s);   \
        else mask ? tile_l<LL, true, false>(p, s) : tile_l<LL, false, false>(p, s);         \
    }
    SE_TILE_CASE(1)
    SE_TILE_CASE(2)
    SE_TILE_CASE(3)
#undef SE_TILE_CASE
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
