// k_block8.cu — fused BLOCK8 protect / recover kernels and the transform-only
// kernels (rows a1-a10 of SURVEY.md §8.1), sm_100a.
//
// Mapping: one thread owns one 8x8 block end to end; one CTA owns 128
// consecutive blocks (row-major block order).  Per CTA the fragment streams
// are contiguous and 16-byte aligned (A' 16*a_bits B, B' 16*b_bits B, C'
// 7680 B), so each CTA assembles its records in shared memory and writes
// them with 128-bit coalesced stores; the A stream of the CTA is exactly
// a_bits AES blocks, so the AES-CTR keystream for it is computed by the CTA
// itself, fused with the LL-band extraction: the private fragment never
// leaves the SM in plaintext and is never re-read from HBM.
//
// Loads: each thread issues 8 x 64-bit loads (one per block row); a warp's
// 32 consecutive blocks cover 256 contiguous bytes per row instruction.
#include <cuda_runtime.h>

#include "se_device.cuh"

#ifndef SE_MIN_CTAS
#define SE_MIN_CTAS 4      // resident 128-thread CTAs per SM the register budget must allow
#endif

namespace se {

// ---------------------------------------------------------------- helpers

// Load the 8x8 block (br, bc) as raw byte values; zero fill past n (C18).
// Centering (C8) is applied to LL_L only, after the transform (see lift_fwd).
__device__ __forceinline__ void load_block(const uint8_t* __restrict__ in, uint64_t n, uint32_t W,
                                           uint64_t br, uint64_t bc, int (&v)[8][8]) {
    const uint64_t row0 = 8 * br * (uint64_t)W + 8 * bc;
    if (row0 + 7ull * W + 8 <= n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint2 q = __ldg(reinterpret_cast<const uint2*>(in + row0 + (uint64_t)i * W));
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[i][j] = (int)((q.x >> (8 * j)) & 0xffu);
                v[i][4 + j] = (int)((q.y >> (8 * j)) & 0xffu);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t idx = row0 + (uint64_t)i * W + j;
                v[i][j] = idx < n ? (int)in[idx] : 0;
            }
    }
}

// Store a block of byte-valued samples, clipped to n.
__device__ __forceinline__ void store_block(uint8_t* __restrict__ out, uint64_t n, uint32_t W,
                                            uint64_t br, uint64_t bc, const int (&x)[8][8]) {
    const uint64_t row0 = 8 * br * (uint64_t)W + 8 * bc;
    if (row0 + 7ull * W + 8 <= n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint2 q;
            q.x = __byte_perm(__byte_perm(x[i][0], x[i][1], 0x0040), __byte_perm(x[i][2], x[i][3], 0x0040), 0x5410);
            q.y = __byte_perm(__byte_perm(x[i][4], x[i][5], 0x0040), __byte_perm(x[i][6], x[i][7], 0x0040), 0x5410);
            *reinterpret_cast<uint2*>(out + row0 + (uint64_t)i * W) = q;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t idx = row0 + (uint64_t)i * W + j;
                if (idx < n) out[idx] = (uint8_t)x[i][j];
            }
    }
}

// OR a BITS-bit record (logical big-endian words) into a shared byte stream
// (stored in memory byte order) at bit offset `off`.
template <int NW, int BITS>
__device__ __forceinline__ void smem_put_record(uint32_t* s, uint32_t off, const uint32_t (&r)[NW]) {
    if (BITS % 32 == 0) {
        const uint32_t w0 = off >> 5;
#pragma unroll
        for (int k = 0; k < NW; ++k) s[w0 + k] = bswap32(r[k]);
    } else {
        const uint32_t w0 = off >> 5, sh = off & 31;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const uint32_t hi = r[k] >> sh;
            const uint32_t lo = sh ? (r[k] << (32 - sh)) : 0u;
            if (hi) atomicOr(&s[w0 + k], bswap32(hi));
            if (lo) atomicOr(&s[w0 + k + 1], bswap32(lo));
        }
    }
}

// Read a BITS-bit record at bit offset `off` from a shared byte stream of
// `nwords` words; bits past the record are cleared.
template <int NW, int BITS>
__device__ __forceinline__ void smem_get_record(const uint32_t* s, uint32_t nwords, uint32_t off,
                                                uint32_t (&r)[NW]) {
    const uint32_t w0 = off >> 5, sh = off & 31;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint32_t a = bswap32(s[w0 + k]);
        const uint32_t b = (w0 + k + 1 < nwords) ? bswap32(s[w0 + k + 1]) : 0u;
        r[k] = sh ? __funnelshift_l(b, a, sh) : a;
    }
    r[NW - 1] &= head_mask(BITS % 32);
}

__device__ __forceinline__ void copy_g2s(uint32_t* s, const uint8_t* __restrict__ g, uint64_t len,
                                         uint32_t cap_bytes, int tid) {
    // zero-filled copy of `len` bytes (<= cap) from 16-byte aligned global memory
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += kBlocksPerCta)
        reinterpret_cast<uint4*>(s)[i] = __ldg(reinterpret_cast<const uint4*>(g) + i);
    uint8_t* sb = reinterpret_cast<uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < cap_bytes; i += kBlocksPerCta) sb[i] = (i < len) ? g[i] : 0;
}

__device__ __forceinline__ void copy_s2g(uint8_t* __restrict__ g, const uint32_t* s, uint64_t len, int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += kBlocksPerCta)
        reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(s)[i];
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < len; i += kBlocksPerCta) g[i] = sb[i];
}

// The AES-CTR keystream of the CTA's A bytes, in memory byte order.
template <int ABITS>
__device__ __forceinline__ void ctr_keystream_cta(const FusedParams& p, const AesSmem& aes, uint32_t* ks,
                                                  uint64_t cta, int tid) {
    for (int t = tid; t < ABITS; t += kBlocksPerCta) {
        uint32_t x[4];
        ctr_add(p.ctr, cta * (uint64_t)ABITS + (uint64_t)t, x);
        aes128_block(aes, p.rk, x);
        reinterpret_cast<uint4*>(ks)[t] = make_uint4(bswap32(x[0]), bswap32(x[1]), bswap32(x[2]), bswap32(x[3]));
    }
}

__device__ __forceinline__ void copy_s2g_xor(uint8_t* __restrict__ g, const uint32_t* s, const uint32_t* ks,
                                             uint64_t len, int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += kBlocksPerCta) {
        const uint4 a = reinterpret_cast<const uint4*>(s)[i], k = reinterpret_cast<const uint4*>(ks)[i];
        reinterpret_cast<uint4*>(g)[i] = make_uint4(a.x ^ k.x, a.y ^ k.y, a.z ^ k.z, a.w ^ k.w);
    }
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    const uint8_t* kb = reinterpret_cast<const uint8_t*>(ks);
    for (uint32_t i = nv * 16 + tid; i < len; i += kBlocksPerCta) g[i] = sb[i] ^ kb[i];
}

// XOR the AES-CTR keystream over the CTA's A bytes held in shared memory.
template <int ABITS>
__device__ __forceinline__ void ctr_xor_cta(const FusedParams& p, const AesSmem& aes, uint32_t* sa,
                                            uint64_t cta, int tid) {
    // CTA A offset = cta * 128 * ABITS bits = cta * ABITS AES blocks
    for (int t = tid; t < ABITS; t += kBlocksPerCta) {
        uint32_t x[4];
        ctr_add(p.ctr, cta * (uint64_t)ABITS + (uint64_t)t, x);
        aes128_block(aes, p.rk, x);
#pragma unroll
        for (int k = 0; k < 4; ++k) sa[4 * t + k] ^= bswap32(x[k]);
    }
}

// SHA-256 mask of B from the plain A record (framing C15: K||IV||be64(b)||A).
template <int L>
__device__ __forceinline__ void mask_b(const FusedParams& p, uint64_t gb, const uint32_t (&A)[Rec<L>::AW],
                                       uint32_t (&B)[Rec<L>::BW]) {
    using R = Rec<L>;
    uint32_t W[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) W[k] = p.kiv[k];
    W[8] = (uint32_t)(gb >> 32);
    W[9] = (uint32_t)gb;
#pragma unroll
    for (int k = 10; k < 16; ++k) W[k] = 0;
#pragma unroll
    for (int k = 0; k < R::AW; ++k) W[10 + k] = A[k];
    constexpr int len = 40 + R::ABYTES;                       // message bytes
    W[len / 4] |= 0x80u << (8 * (3 - len % 4));                // FIPS 180-4 §5.1.1
    W[15] = (uint32_t)(len * 8);
    const uint32_t st[8] = {p.mid256[0], p.mid256[1], p.mid256[2], p.mid256[3],
                            p.mid256[4], p.mid256[5], p.mid256[6], p.mid256[7]};
    const uint32_t h0[8] = {p.h256[0], p.h256[1], p.h256[2], p.h256[3],
                            p.h256[4], p.h256[5], p.h256[6], p.h256[7]};
    uint32_t H[8];
    sha256_from_round8(st, h0, W, H, p.one);
#pragma unroll
    for (int k = 0; k < R::BW; ++k) {
        const uint32_t m = (k == R::BW - 1) ? (H[k] & head_mask(R::BBITS % 32)) : H[k];
        B[k] ^= m;                                             // first |B| bits (C17)
    }
}

// SHA-512 mask of C from the record `src` (B' for L >= 2, plain A for L = 1).
template <int NW, int SBYTES>
__device__ __forceinline__ void mask_c(const FusedParams& p, uint64_t gb, const uint32_t (&src)[NW],
                                       uint32_t (&C)[15]) {
    W64 W[16];
    W[0] = W64{p.kiv[1], p.kiv[0]};
    W[1] = W64{p.kiv[3], p.kiv[2]};
    W[2] = W64{p.kiv[5], p.kiv[4]};
    W[3] = W64{p.kiv[7], p.kiv[6]};
    W[4] = W64{(uint32_t)gb, (uint32_t)(gb >> 32)};
#pragma unroll
    for (int k = 5; k < 16; ++k) W[k] = W64{0u, 0u};
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        if (k & 1) W[5 + k / 2].lo = src[k];
        else W[5 + k / 2].hi = src[k];
    }
    constexpr int len = 40 + SBYTES;
    constexpr int pw = len / 8, pb = 7 - len % 8;                // pad byte position
    if constexpr (pb >= 4) W[pw].hi |= 0x80u << (8 * (pb - 4));
    else W[pw].lo |= 0x80u << (8 * pb);
    W[15].lo = (uint32_t)(len * 8);
    const uint64_t st[8] = {p.mid512[0], p.mid512[1], p.mid512[2], p.mid512[3],
                            p.mid512[4], p.mid512[5], p.mid512[6], p.mid512[7]};
    const uint64_t h0[8] = {p.h512[0], p.h512[1], p.h512[2], p.h512[3],
                            p.h512[4], p.h512[5], p.h512[6], p.h512[7]};
    uint64_t H[8];
    sha512_from_round4(st, h0, W, H, p.one);
#pragma unroll
    for (int k = 0; k < 15; ++k) C[k] ^= (k & 1) ? (uint32_t)H[k / 2] : (uint32_t)(H[k / 2] >> 32);
}

// ---------------------------------------------------------------- protect

// One CTA of protect: 128 consecutive blocks starting at local block cta*128
// of the file described by p (kernel parameters, or a batch job in smem).
template <int L, bool MASK>
__device__ __forceinline__ void protect_cta(const FusedParams& p, const uint64_t cta) {
    using R = Rec<L>;
    constexpr int SA_W = 4 * R::ABITS;             // 16*ABITS bytes per CTA
    constexpr int SB_W = R::BBITS ? 4 * R::BBITS : 4;
    constexpr int SC_W = 4 * R::CBITS;
    __shared__ AesSmem aes;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ __align__(16) uint32_t sks[SA_W];     // AES-CTR keystream for the CTA's A bytes
    __shared__ __align__(16) uint32_t sb[SB_W];
    __shared__ __align__(16) uint32_t sc[SC_W];

    const int tid = threadIdx.x;
    const uint64_t blk = cta * kBlocksPerCta + tid;
    for (int i = tid; i < SA_W; i += kBlocksPerCta) sa[i] = 0;
    for (int i = tid; i < SB_W; i += kBlocksPerCta) sb[i] = 0;
    aes_load_tables(aes, tid, kBlocksPerCta);
    __syncthreads();
    // row a6, keystream half: the CTA's a_bits counter blocks, computed first so
    // the few warps doing AES overlap with the others' lifting and hashing.
    ctr_keystream_cta<R::ABITS>(p, aes, sks, cta, tid);

    if (blk < p.n_blocks) {
        const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
        int v[8][8];
        load_block(p.in, p.n_bytes, p.width, br, bc, v);
        dwt8_fwd<L>(v, p.one);                                              // rows a2-a4
        uint32_t A[R::AW], B[R::BW], C[R::CW];
#pragma unroll
        for (int k = 0; k < R::AW; ++k) A[k] = 0;
#pragma unroll
        for (int k = 0; k < R::BW; ++k) B[k] = 0;
#pragma unroll
        for (int k = 0; k < R::CW; ++k) C[k] = 0;
        for_each_field<L>([&](int s, int pos, int i, int j, int w) {       // row a5
            // offset-binary (C9); LL_L also absorbs the -128 centering (C8)
            const int off = (s == 0) ? (1 << (w - 1)) - 128 : (1 << (w - 1));
            if (s == 0) put_field(A, pos, v[i][j], off, w, p.one);
            else if (s == 1) put_field(B, pos, v[i][j], off, w, p.one);
            else put_field(C, pos, v[i][j], off, w, p.one);
        });
        if (MASK) {
            const uint64_t gb = p.block_offset + blk;
            if (R::BBITS) {
                mask_b<L>(p, gb, A, B);                                     // row a7
                mask_c<R::BW, R::BBYTES>(p, gb, B, C);                      // row a8
            } else {
                mask_c<R::AW, R::ABYTES>(p, gb, A, C);                      // C21 (L = 1)
            }
        }
        smem_put_record<R::AW, R::ABITS>(sa, (uint32_t)tid * R::ABITS, A);
        if (R::BBITS) smem_put_record<R::BW, R::BBITS>(sb, (uint32_t)tid * R::BBITS, B);
        smem_put_record<R::CW, R::CBITS>(sc, (uint32_t)tid * R::CBITS, C);
    }
    __syncthreads();

    // row a9: 128-bit coalesced stores of the CTA's slice of each stream;
    // A' = A ^ keystream on the way out (row a6, XOR half)
    const uint64_t a0 = cta * 16ull * R::ABITS, c0 = cta * 16ull * R::CBITS;
    copy_s2g_xor(p.a + a0, sa, sks, min((uint64_t)SA_W * 4, p.a_bytes - a0), tid);
    if (R::BBITS) {
        const uint64_t b0 = cta * 16ull * R::BBITS;
        copy_s2g(p.b + b0, sb, min((uint64_t)SB_W * 4, p.b_bytes - b0), tid);
    }
    copy_s2g(p.c + c0, sc, min((uint64_t)SC_W * 4, p.c_bytes - c0), tid);
}

// ---------------------------------------------------------------- recover

template <int L, bool MASK>
__device__ __forceinline__ void recover_cta(const FusedParams& p, const uint64_t cta) {
    using R = Rec<L>;
    constexpr int SA_W = 4 * R::ABITS;
    constexpr int SB_W = R::BBITS ? 4 * R::BBITS : 4;
    constexpr int SC_W = 4 * R::CBITS;
    __shared__ AesSmem aes;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ __align__(16) uint32_t sb[SB_W];
    __shared__ __align__(16) uint32_t sc[SC_W];
    __shared__ unsigned long long s_first;
    __shared__ unsigned int s_bad;

    const int tid = threadIdx.x;
    const uint64_t blk = cta * kBlocksPerCta + tid;
    const uint64_t a0 = cta * 16ull * R::ABITS, c0 = cta * 16ull * R::CBITS;
    if (tid == 0) { s_first = ~0ull; s_bad = 0; }
    copy_g2s(sa, p.a + a0, min((uint64_t)SA_W * 4, p.a_bytes - a0), SA_W * 4, tid);
    if (R::BBITS) {
        const uint64_t b0 = cta * 16ull * R::BBITS;
        copy_g2s(sb, p.b + b0, min((uint64_t)SB_W * 4, p.b_bytes - b0), SB_W * 4, tid);
    }
    copy_g2s(sc, p.c + c0, min((uint64_t)SC_W * 4, p.c_bytes - c0), SC_W * 4, tid);
    aes_load_tables(aes, tid, kBlocksPerCta);
    __syncthreads();
    ctr_xor_cta<R::ABITS>(p, aes, sa, cta, tid);                             // A' -> A (few warps)

    // C needs only B' (C19), so its SHA-512 unmask runs while the AES warps work
    const bool valid = blk < p.n_blocks;
    const uint64_t gb = p.block_offset + blk;
    uint32_t A[R::AW], B[R::BW], C[R::CW];
    if (valid) {
        if (R::BBITS) smem_get_record<R::BW, R::BBITS>(sb, SB_W, (uint32_t)tid * R::BBITS, B);
        else B[0] = 0;
        smem_get_record<R::CW, R::CBITS>(sc, SC_W, (uint32_t)tid * R::CBITS, C);
        if (MASK && R::BBITS) mask_c<R::BW, R::BBYTES>(p, gb, B, C);          // C from B'
    }
    __syncthreads();                                                         // plain A ready

    bool bad = false;
    if (valid) {
        smem_get_record<R::AW, R::ABITS>(sa, SA_W, (uint32_t)tid * R::ABITS, A);
        if (MASK) {
            if (R::BBITS) mask_b<L>(p, gb, A, B);                            // B from A
            else mask_c<R::AW, R::ABYTES>(p, gb, A, C);                      // C21 (L = 1)
        }
        int v[8][8];
        for_each_field<L>([&](int s, int pos, int i, int j, int w) {
            const int off = (s == 0) ? (1 << (w - 1)) - 128 : (1 << (w - 1));   // see protect
            if (s == 0) v[i][j] = get_field(A, pos, off, w, p.one);
            else if (s == 1) v[i][j] = get_field(B, pos, off, w, p.one);
            else v[i][j] = get_field(C, pos, off, w, p.one);
        });
        dwt8_inv<L>(v, p.one);                                               // uncentered bytes
        int orv = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) orv |= v[i][j];
        bad = (orv & ~0xff) != 0;      // any sample outside [0, 255]
        const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
        store_block(p.out, p.n_bytes, p.width, br, bc, v);
    }
    if (p.report != nullptr) {
        if (bad) {
            atomicMin(&s_first, (unsigned long long)blk);
            atomicAdd(&s_bad, 1u);
        }
        __syncthreads();
        if (tid == 0 && s_bad) {
            atomicMin(reinterpret_cast<unsigned long long*>(&p.report->first_bad_block), s_first);
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.report->bad_blocks), (unsigned long long)s_bad);
        }
    }
}

// ---------------------------------------------------------------- kernels

template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS)
k_protect_block8(const __grid_constant__ FusedParams p) {
    protect_cta<L, MASK>(p, blockIdx.x);
}

template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS)
k_recover_block8(const __grid_constant__ FusedParams p) {
    recover_cta<L, MASK>(p, blockIdx.x);
}

// Many independent files in one launch (C5; SURVEY §8.6 "sharded by file").
// Each CTA finds its job by binary search over cta_begin, assembles that job's
// parameters in shared memory (the per-job counter base and SHA midstates were
// derived on the host by fragment_batch_plan) and runs the same CTA body.
template <int L, bool MASK, bool RECOVER>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS)
k_batch_block8(const __grid_constant__ BatchParams bp) {
    __shared__ FusedParams sp;
    __shared__ uint32_t s_job;
    using R = Rec<L>;
    const uint32_t x = blockIdx.x;
    if (threadIdx.x == 0) {
        uint32_t lo = 0, hi = bp.n_jobs - 1;          // largest j with cta_begin <= x
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) / 2;
            if (bp.jobs[mid].cta_begin <= x) lo = mid;
            else hi = mid - 1;
        }
        s_job = lo;
    }
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&bp.base);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&sp);
        for (uint32_t i = threadIdx.x; i < sizeof(FusedParams) / 4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const se_job& job = bp.jobs[s_job];
    const JobDerived& dv = *reinterpret_cast<const JobDerived*>(job.derived);
    const uint32_t t = threadIdx.x;
    if (t == 0) {
        sp.in = job.in;
        sp.out = job.out;
        sp.a = job.a; sp.b = job.b; sp.c = job.c;
        sp.report = bp.reports ? bp.reports + s_job : nullptr;
        sp.n_bytes = job.n_bytes;
        sp.width = job.width;
        sp.bpr = job.width / 8;
        const uint64_t rows = ((job.n_bytes + job.width - 1) / job.width + 7) / 8 * 8;
        sp.n_blocks = rows / 8 * sp.bpr;
        sp.block_offset = job.block_offset;
        sp.a_bytes = (sp.n_blocks * R::ABITS + 7) / 8;
        sp.b_bytes = (sp.n_blocks * R::BBITS + 7) / 8;
        sp.c_bytes = (sp.n_blocks * R::CBITS + 7) / 8;
    } else if (t >= 32 && t < 36) {
        sp.ctr[t - 32] = dv.ctr[t - 32];
    } else if (t >= 36 && t < 44) {
        sp.kiv[t - 36] = dv.kiv[t - 36];
    } else if (t >= 44 && t < 52) {
        sp.mid256[t - 44] = dv.mid256[t - 44];
    } else if (t >= 52 && t < 60) {
        sp.mid512[t - 52] = dv.mid512[t - 52];
    }
    __syncthreads();
    const uint64_t cta = x - job.cta_begin;
    if (RECOVER) recover_cta<L, MASK>(sp, cta);
    else protect_cta<L, MASK>(sp, cta);
}

__global__ void k_report_init(se_report* r, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { r[i].first_bad_block = -1; r[i].bad_blocks = 0; }
}

// ---------------------------------------------------------------- transform only

template <int L>
__global__ void __launch_bounds__(kBlocksPerCta) k_dwt_fwd_block8(const __grid_constant__ DwtParams p) {
    const uint64_t blk = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (blk >= p.n_blocks) return;
    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
    int v[8][8];
    load_block(p.in, p.n_bytes, p.width, br, bc, v);
    dwt8_fwd<L>(v, p.one);
#pragma unroll
    for (int i = 0; i < (8 >> L); ++i)
#pragma unroll
        for (int j = 0; j < (8 >> L); ++j) v[i][j] -= 128;     // centering (C8) lands on LL_L only
    int16_t* base = p.coef + 8 * br * (uint64_t)p.width + 8 * bc;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint4 q;
        q.x = (uint32_t)(v[i][0] & 0xffff) | ((uint32_t)v[i][1] << 16);
        q.y = (uint32_t)(v[i][2] & 0xffff) | ((uint32_t)v[i][3] << 16);
        q.z = (uint32_t)(v[i][4] & 0xffff) | ((uint32_t)v[i][5] << 16);
        q.w = (uint32_t)(v[i][6] & 0xffff) | ((uint32_t)v[i][7] << 16);
        *reinterpret_cast<uint4*>(base + (uint64_t)i * p.width) = q;
    }
}

template <int L>
__global__ void __launch_bounds__(kBlocksPerCta) k_dwt_inv_block8(const __grid_constant__ DwtParams p) {
    const uint64_t blk = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (blk >= p.n_blocks) return;
    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
    const int16_t* base = p.coef + 8 * br * (uint64_t)p.width + 8 * bc;
    int v[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)i * p.width));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[i][2 * k] = (int)(int16_t)(w[k] & 0xffff);
            v[i][2 * k + 1] = (int)(int16_t)(w[k] >> 16);
        }
    }
#pragma unroll
    for (int i = 0; i < (8 >> L); ++i)
#pragma unroll
        for (int j = 0; j < (8 >> L); ++j) v[i][j] += 128;
    dwt8_inv<L>(v, p.one);
    store_block(p.out, p.n_bytes, p.width, br, bc, v);
}

// ---------------------------------------------------------------- launchers

static unsigned grid_for(uint64_t n_blocks) {
    return (unsigned)((n_blocks + kBlocksPerCta - 1) / kBlocksPerCta);
}

template <int L>
static void protect_l(const FusedParams& p, bool mask, cudaStream_t s) {
    if (mask) k_protect_block8<L, true><<<grid_for(p.n_blocks), kBlocksPerCta, 0, s>>>(p);
    else k_protect_block8<L, false><<<grid_for(p.n_blocks), kBlocksPerCta, 0, s>>>(p);
}
template <int L>
static void recover_l(const FusedParams& p, bool mask, cudaStream_t s) {
    if (mask) k_recover_block8<L, true><<<grid_for(p.n_blocks), kBlocksPerCta, 0, s>>>(p);
    else k_recover_block8<L, false><<<grid_for(p.n_blocks), kBlocksPerCta, 0, s>>>(p);
}

int launch_protect_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) protect_l<1>(p, mask, s);
    else if (levels == 2) protect_l<2>(p, mask, s);
    else protect_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

int launch_recover_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) recover_l<1>(p, mask, s);
    else if (levels == 2) recover_l<2>(p, mask, s);
    else recover_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

template <int L, bool RECOVER>
static void batch_l(const BatchParams& bp, uint64_t ctas, bool mask, cudaStream_t s) {
    if (mask) k_batch_block8<L, true, RECOVER><<<(unsigned)ctas, kBlocksPerCta, 0, s>>>(bp);
    else k_batch_block8<L, false, RECOVER><<<(unsigned)ctas, kBlocksPerCta, 0, s>>>(bp);
}

int launch_batch_block8(const BatchParams& bp, uint64_t total_ctas, uint32_t levels, bool mask, bool recover,
                        void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (recover && bp.reports) {
        k_report_init<<<(bp.n_jobs + 255) / 256, 256, 0, s>>>(bp.reports, bp.n_jobs);
        note_launch();
    }
    if (total_ctas == 0) return (int)cudaGetLastError();
    if (recover) {
        if (levels == 1) batch_l<1, true>(bp, total_ctas, mask, s);
        else if (levels == 2) batch_l<2, true>(bp, total_ctas, mask, s);
        else batch_l<3, true>(bp, total_ctas, mask, s);
    } else {
        if (levels == 1) batch_l<1, false>(bp, total_ctas, mask, s);
        else if (levels == 2) batch_l<2, false>(bp, total_ctas, mask, s);
        else batch_l<3, false>(bp, total_ctas, mask, s);
    }
    note_launch();
    return (int)cudaGetLastError();
}

int launch_dwt_fwd_block8(const DwtParams& p, uint32_t levels, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = grid_for(p.n_blocks);
    if (levels == 1) k_dwt_fwd_block8<1><<<g, kBlocksPerCta, 0, s>>>(p);
    else if (levels == 2) k_dwt_fwd_block8<2><<<g, kBlocksPerCta, 0, s>>>(p);
    else k_dwt_fwd_block8<3><<<g, kBlocksPerCta, 0, s>>>(p);
    note_launch();
    return (int)cudaGetLastError();
}

int launch_dwt_inv_block8(const DwtParams& p, uint32_t levels, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = grid_for(p.n_blocks);
    if (levels == 1) k_dwt_inv_block8<1><<<g, kBlocksPerCta, 0, s>>>(p);
    else if (levels == 2) k_dwt_inv_block8<2><<<g, kBlocksPerCta, 0, s>>>(p);
    else k_dwt_inv_block8<3><<<g, kBlocksPerCta, 0, s>>>(p);
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
