// fused_cta.cuh — the CTA bodies of the fused protect / recover kernels
// (rows a1-a10), shared by the single-file, batch (k_block8.cu) and
// FULL-mode (k_full.cu) kernels.  One thread owns one 8x8 block (or, in FULL
// mode, one 8x8 input footprint); one CTA owns 128 consecutive blocks.
#pragma once
#include <cuda_runtime.h>

#include "se_device.cuh"

// Masked per-CTA kernels: mixed-pipe lifting (bit 0 forward, bit 1 inverse,
// se_device.cuh lift_*_mix) and the paired range check (bit 2).  Measured
// (C4, tools/gpu_r2_call40.sh): forward protect 4.684 -> 4.665 ms, inverse
// recover 4.668 -> 4.653 ms, paired check recover 4.668 -> 4.714 ms then;
// re-measured on the final build (three passes): paired check recover 4.643
// -> 4.595 ms: 7.
#ifndef SE_MASK_MIX
#define SE_MASK_MIX 7
#endif
#include "sha2_spec.cuh"

namespace se {

// ---------------------------------------------------------------- helpers

// Load the 8x8 block (br, bc) as raw byte values; zero fill past n (C18).
// Centering (C8) is applied to LL_L only, after the transform (see lift_fwd).
// The 4 bytes of w as ints.  SE_UNPACK 0: shifts and masks (ALU pipe);
// 1: byte conversions with selectors (I2F.U8 + F2I, conversion pipe) to free
// ALU slots in the SHA-bound masked kernels - measured slower in round 1
// (C2 masked protect 182.7 vs 185.7 GB/s); 2: one PRMT per byte - round 2,
// C4 masked protect 4.702 -> 4.681 ms (C2 within noise), so 2.
#ifndef SE_UNPACK
#define SE_UNPACK 2
#endif
__device__ __forceinline__ void unpack4(uint32_t w, int& b0, int& b1, int& b2, int& b3) {
#if SE_UNPACK == 2
    // one PRMT per byte (the shift-and-mask form takes two for the middle bytes)
    b0 = (int)__byte_perm(w, 0, 0x4440);
    b1 = (int)__byte_perm(w, 0, 0x4441);
    b2 = (int)__byte_perm(w, 0, 0x4442);
    b3 = (int)__byte_perm(w, 0, 0x4443);
#elif SE_UNPACK == 1
    int* out[4] = {&b0, &b1, &b2, &b3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float f;
        asm("cvt.rn.f32.u8 %0, %1;" : "=f"(f) : "h"((unsigned short)(unsigned char)(w >> (8 * j))));
        *out[j] = __float2int_rz(f);
    }
#else
    b0 = (int)(w & 0xffu);
    b1 = (int)((w >> 8) & 0xffu);
    b2 = (int)((w >> 16) & 0xffu);
    b3 = (int)(w >> 24);
#endif
}

__device__ __forceinline__ void load_block(const uint8_t* __restrict__ in, uint64_t n, uint32_t W,
                                           uint64_t br, uint64_t bc, int (&v)[8][8]) {
    const uint64_t row0 = 8 * br * (uint64_t)W + 8 * bc;
    if (row0 + 7ull * W + 8 <= n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint2 q = __ldg(reinterpret_cast<const uint2*>(in + row0 + (uint64_t)i * W));
            unpack4(q.x, v[i][0], v[i][1], v[i][2], v[i][3]);
            unpack4(q.y, v[i][4], v[i][5], v[i][6], v[i][7]);
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

template <int NT = kBlocksPerCta>
__device__ __forceinline__ void copy_g2s(uint32_t* s, const uint8_t* __restrict__ g, uint64_t len,
                                         uint32_t cap_bytes, int tid) {
    // zero-filled copy of `len` bytes (<= cap) from 16-byte aligned global memory
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += NT)
        reinterpret_cast<uint4*>(s)[i] = __ldg(reinterpret_cast<const uint4*>(g) + i);
    uint8_t* sb = reinterpret_cast<uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < cap_bytes; i += NT) sb[i] = (i < len) ? g[i] : 0;
}

template <int NT = kBlocksPerCta>
__device__ __forceinline__ void copy_s2g(uint8_t* __restrict__ g, const uint32_t* s, uint64_t len, int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += NT)
        reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(s)[i];
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < len; i += NT) g[i] = sb[i];
}

// A' = A ^ KS where the keystream already sits at the destination in global
// memory (written there by k_cipher_ctr); each CTA reads and rewrites only its
// own slice.
template <int NT = kBlocksPerCta>
__device__ __forceinline__ void copy_s2g_xor_global(uint8_t* __restrict__ g, const uint32_t* s, uint64_t len,
                                                    int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += NT) {
        const uint4 a = reinterpret_cast<const uint4*>(s)[i], k = reinterpret_cast<const uint4*>(g)[i];
        reinterpret_cast<uint4*>(g)[i] = make_uint4(a.x ^ k.x, a.y ^ k.y, a.z ^ k.z, a.w ^ k.w);
    }
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < len; i += NT) g[i] = sb[i] ^ g[i];
}

// A' = A ^ KS with the keystream in separate (device) memory: A' is written
// once, e.g. straight into mapped host memory.
template <int NT = kBlocksPerCta>
__device__ __forceinline__ void copy_s2g_xor(uint8_t* __restrict__ g, const uint32_t* s,
                                             const uint8_t* __restrict__ ks, uint64_t len, int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += NT) {
        const uint4 a = reinterpret_cast<const uint4*>(s)[i], k = reinterpret_cast<const uint4*>(ks)[i];
        reinterpret_cast<uint4*>(g)[i] = make_uint4(a.x ^ k.x, a.y ^ k.y, a.z ^ k.z, a.w ^ k.w);
    }
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < len; i += NT) g[i] = sb[i] ^ ks[i];
}

// A = A' ^ KS in shared memory, keystream read from global memory.
template <int NT = kBlocksPerCta>
__device__ __forceinline__ void xor_g2s(uint32_t* s, const uint8_t* __restrict__ ks, uint64_t len, int tid) {
    const uint32_t nv = (uint32_t)(len / 16);
    for (uint32_t i = tid; i < nv; i += NT) {
        const uint4 k = reinterpret_cast<const uint4*>(ks)[i];
        uint4& a = reinterpret_cast<uint4*>(s)[i];
        a.x ^= k.x; a.y ^= k.y; a.z ^= k.z; a.w ^= k.w;
    }
    uint8_t* sb = reinterpret_cast<uint8_t*>(s);
    for (uint32_t i = nv * 16 + tid; i < len; i += NT) sb[i] ^= ks[i];
}

// SHA-256 mask of B from the plain A record (framing C15: K||IV||be64(b)||A).
// SE_SHA256_BODY_P: the SHA-256 loop body of the single-file protect kernels
// (16: measured on C4, two passes, protect 4.610 -> 4.595 ms; in the batch
// kernels the 16-round body was slower, C5 108.3 -> 107.2 GB/s).
#ifndef SE_SHA256_BODY_P
#define SE_SHA256_BODY_P 16
#endif
// SE_SPEC_REC256 1: the single-file recover kernels specialise the SHA-256
// schedule too (measured on C4, two passes: recover 4.585 -> 4.567 ms, while
// protect is faster with the generic 16-round body: 4.612 vs 4.595 ms).
#ifndef SE_SPEC_REC256
#define SE_SPEC_REC256 1
#endif
#ifndef SE_SPEC
#define SE_SPEC 2      // bit 0: SHA-256 (B mask), bit 1: SHA-512 (C mask) schedules specialised
                       // (2: the SHA-256 one costs more in instruction fetch than it saves)
#endif
// SPEC: the message schedule specialised with the launch's host-computed
// constants (p.s256 / p.s512, sha2_spec.cuh); batches (per-file IV) use the
// generic schedule.
template <int L, int MODE, bool SPEC = true, bool SPEC256 = (SE_SPEC & 1) != 0, int BODY = SE_SHA_BODY>
__device__ __forceinline__ void mask_b(const FusedParams& p, uint64_t gb, const uint32_t (&A)[Rec<L, MODE>::AW],
                                       uint32_t (&B)[Rec<L, MODE>::BW]) {
    using R = Rec<L, MODE>;
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
    if constexpr (SPEC && SPEC256) sha256_from_round8_spec<msg_var256(R::ABYTES)>(st, h0, W, p.s256, H, p.one);
    else sha256_from_round8<BODY>(st, h0, W, H, p.one);
#pragma unroll
    for (int k = 0; k < R::BW; ++k) {
        const uint32_t m = (k == R::BW - 1) ? (H[k] & head_mask(R::BBITS % 32)) : H[k];
        B[k] ^= m;                                             // first |B| bits (C17)
    }
}

// SHA-512 mask of C from the record `src` (B' for L >= 2, plain A for L = 1).
template <int NW, int SBYTES, bool SPEC = true>
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
    if constexpr (SPEC && (SE_SPEC & 2)) sha512_from_round4_spec<msg_var512(SBYTES)>(st, h0, W, p.s512, H, p.one);
    else sha512_from_round4(st, h0, W, H, p.one);
#pragma unroll
    for (int k = 0; k < 15; ++k) C[k] ^= (k & 1) ? (uint32_t)H[k / 2] : (uint32_t)(H[k / 2] >> 32);
}

// ---------------------------------------------------------------- stream slices in shared memory

// Write this thread's NB-bit record (logical MSB-first words) into the warp's
// part of a dense stream slice (memory byte order) at `words`; each warp's 32
// records fill exactly NB whole words.  Record-centric for NB >= 32: a lane
// writes the words that start inside its record, taking the bits past its
// record end from the next lane's first word (one shuffle).  ks (nullable):
// keystream words XORed in (A').
template <int NB, int NW>
__device__ __forceinline__ void put_stream(uint32_t* words, const uint32_t* ks, const uint32_t (&rec)[NW], int ct) {
    const int lane = ct & 31, warp = ct >> 5;
    const uint32_t wbase = (uint32_t)warp * NB;
    if constexpr (NB % 32 == 0) {
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const uint32_t w = wbase + lane * NW + k;
            uint32_t v = bswap32(rec[k]);
            if (ks) v ^= ks[w];
            words[w] = v;
        }
    } else if constexpr (NB >= 32) {
        constexpr int r = NB % 32;
        const uint32_t nx = __shfl_down_sync(0xffffffffu, rec[0], 1);
        uint32_t Z[NW + 1];
#pragma unroll
        for (int k = 0; k < NW - 1; ++k) Z[k] = rec[k];
        Z[NW - 1] = rec[NW - 1] | (nx >> r);
        Z[NW] = nx << (32 - r);
        const uint32_t s0 = (uint32_t)lane * NB;
        const uint32_t w0 = (s0 + 31) >> 5, o = (w0 << 5) - s0;          // first word starting in the record
        const uint32_t w1 = (s0 + NB + 31) >> 5;                          // one past the last
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            if (w0 + k < w1) {
                const uint32_t w = wbase + w0 + k;
                uint32_t v = bswap32(__funnelshift_l(Z[k + 1], Z[k], o));
                if (ks) v ^= ks[w];
                words[w] = v;
            }
        }
    } else {
        // NB < 32 (A at L = 3): word-centric, lane w < NB assembles word w
        // from the <= ceil(32/NB) + 1 records it overlaps
        uint32_t acc = 0;
        const int w = lane;
        const int r0 = (32 * w) / NB;
#pragma unroll
        for (int j = 0; j <= 32 / NB + 1; ++j) {
            const int rr = r0 + j;
            const uint32_t val = __shfl_sync(0xffffffffu, rec[0], rr & 31);
            const int pos = NB * rr - 32 * w;                 // record start relative to the word's MSB
            if (rr < 32 && pos < 32 && pos > -NB) acc |= pos >= 0 ? (val >> pos) : (val << -pos);
        }
        if (w < NB) {
            const uint32_t ww = wbase + w;
            uint32_t v = bswap32(acc);
            if (ks) v ^= ks[ww];
            words[ww] = v;
        }
    }
}

// Read record `u` (NB bits, tile-local) of a dense stream slice in shared
// memory (memory byte order) as logical MSB-first words; ks (nullable) is
// XORed in first.
template <int NB, int NW>
__device__ __forceinline__ void get_stream(const uint32_t* words, const uint32_t* ks, uint32_t u, uint32_t (&rec)[NW]) {
    const uint32_t s0 = u * NB, w = s0 >> 5, sh = s0 & 31;
    uint32_t S[NW + 1];
#pragma unroll
    for (int k = 0; k <= NW; ++k) {
        if (k == NW && (NB % 32) == 0) { S[k] = 0; continue; }
        uint32_t m = words[w + k];
        if (ks) m ^= ks[w + k];
        S[k] = bswap32(m);
    }
#pragma unroll
    for (int k = 0; k < NW; ++k) rec[k] = (NB % 32 == 0) ? S[k] : __funnelshift_l(S[k + 1], S[k], sh);
    rec[NW - 1] &= head_mask(NB % 32);
}

// ---------------------------------------------------------------- FULL-mode footprints (row a11)

// The coefficients of input footprint (br, bc) inside the R x W Mallat layout,
// presented in the 8x8 dyadic block layout the record code uses: dyadic
// (i, j) at level l (band side s = 8 >> l) maps to band (i >= s, j >= s) at
// band-local (i mod s, j mod s), i.e. Mallat row (i >= s ? R>>l : 0) +
// (8br >> l) + i mod s, column likewise.  Each band row of the footprint is
// s contiguous int16, moved as one 2s-byte access.
template <int L, bool STORE>
__device__ __forceinline__ void footprint_full(const FusedParams& p, uint64_t br, uint64_t bc, int (&v)[8][8]) {
    const uint64_t W = p.width, R = p.rows;
#pragma unroll
    for (int l = 1; l <= L; ++l) {
        const int s = 8 >> l;
#pragma unroll
        for (int band = (l == L ? 0 : 1); band < 4; ++band) {
            const bool hr = band >= 2, hc = band & 1;         // 0 LL, 1 HL, 2 LH, 3 HH
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const uint64_t row = (hr ? (R >> l) : 0) + ((8 * br) >> l) + i;
                const uint64_t col = (hc ? (W >> l) : 0) + ((8 * bc) >> l);
                int16_t* g = p.ws + row * W + col;
                const int di = (hr ? s : 0) + i, dj = hc ? s : 0;
                if (s == 4) {
                    if (STORE) {
                        uint2 q;
                        q.x = (uint32_t)(v[di][dj] & 0xffff) | ((uint32_t)v[di][dj + 1] << 16);
                        q.y = (uint32_t)(v[di][dj + 2] & 0xffff) | ((uint32_t)v[di][dj + 3] << 16);
                        *reinterpret_cast<uint2*>(g) = q;
                    } else {
                        const uint2 q = *reinterpret_cast<const uint2*>(g);
                        v[di][dj] = (int)(int16_t)(q.x & 0xffff);
                        v[di][dj + 1] = (int)(int16_t)(q.x >> 16);
                        v[di][dj + 2] = (int)(int16_t)(q.y & 0xffff);
                        v[di][dj + 3] = (int)(int16_t)(q.y >> 16);
                    }
                } else if (s == 2) {
                    if (STORE) {
                        *reinterpret_cast<uint32_t*>(g) =
                            (uint32_t)(v[di][dj] & 0xffff) | ((uint32_t)v[di][dj + 1] << 16);
                    } else {
                        const uint32_t q = *reinterpret_cast<const uint32_t*>(g);
                        v[di][dj] = (int)(int16_t)(q & 0xffff);
                        v[di][dj + 1] = (int)(int16_t)(q >> 16);
                    }
                } else {
                    if (STORE) *g = (int16_t)v[di][dj];
                    else v[di][dj] = *g;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- protect

// One CTA of protect: 128 consecutive blocks starting at local block cta*128
// of the file described by p (kernel parameters, or a batch job in smem).
// MODE 0 (BLOCK8): load + per-block lifting.  MODE 1 (FULL): gather the
// footprint from the whole-matrix coefficients in p.ws (k_full.cu).
//
// Row a6: the AES-CTR keystream of the whole A stream was written into p.a by
// k_cipher_ctr (k_batch_keystream for batches), launched just before this
// kernel with programmatic stream serialization; the CTA waits for it
// (griddepcontrol.wait) only at the copy-out, so the keystream kernel overlaps
// the lifting and hashing and the fused kernel carries no AES tables.
// BPC = blocks (threads) per CTA: 128 everywhere but the single-file BLOCK8
// kernels at L = 1, 2, where 32 or 64 give finer work units (k_block8.cu).
template <int L, bool MASK, int MODE = 0, int BPC = kBlocksPerCta, bool SPEC = true, int B256 = SE_SHA_BODY>
__device__ __forceinline__ void protect_cta(const FusedParams& p, const uint64_t cta) {
    using R = Rec<L, MODE>;
    static_assert((BPC * R::ABITS) % 128 == 0 && (BPC * R::BBITS) % 128 == 0 && (BPC * R::CBITS) % 128 == 0,
                  "CTA stream slices must be whole 16-byte units (and A whole AES blocks)");
    constexpr int SA_W = BPC * R::ABITS / 32;      // BPC*ABITS/8 bytes per CTA
    constexpr int SB_W = R::BBITS ? BPC * R::BBITS / 32 : 4;
    constexpr int SC_W = BPC * R::CBITS / 32;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ __align__(16) uint32_t sb[SB_W];
    __shared__ __align__(16) uint32_t sc[SC_W];

    const int tid = threadIdx.x;
    const uint64_t blk = cta * BPC + tid;
    __shared__ AesSmem aes;
    if (!p.ks_in_a) aes_load_tables(aes, tid, BPC);       // constant tables: before the grid dependency
    for (int i = tid; i < SA_W; i += BPC) sa[i] = 0;
    for (int i = tid; i < SB_W; i += BPC) sb[i] = 0;
    // programmatic dependent launch: inputs (and FULL-mode coefficients) are
    // written by earlier work on the stream.  With p.ks_in_a the kernel right
    // before is the keystream kernel (a normal launch, so all earlier work is
    // complete): only its keystream, needed at the copy-out, is waited for.
    if (!p.ks_in_a) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();

    if (blk < p.n_blocks) {
        const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
        int v[8][8];
        if constexpr (MODE == 0) {
            load_block(p.in, p.n_bytes, p.width, br, bc, v);
#if SE_MASK_MIX & 1
            dwt8_fwd_mix<L>(v, p.one);                                      // rows a2-a4 (+1 on all but LL)
#else
            dwt8_fwd<L>(v, p.one);                                          // rows a2-a4
#endif
        } else {
            footprint_full<L, false>(p, br, bc, v);                         // row a11
        }
        uint32_t A[R::AW], B[R::BW], C[R::CW];
#pragma unroll
        for (int k = 0; k < R::AW; ++k) A[k] = 0;
#pragma unroll
        for (int k = 0; k < R::BW; ++k) B[k] = 0;
#pragma unroll
        for (int k = 0; k < R::CW; ++k) C[k] = 0;
        for_each_field<L, MODE>([&](int s, int pos, int i, int j, int w) {  // row a5
            // offset-binary (C9); in BLOCK8 LL_L also absorbs the -128 centering (C8)
            const int off = (s == 0 && MODE == 0) ? (1 << (w - 1)) - 128
                                                  : (1 << (w - 1)) - (MODE == 0 ? (SE_MASK_MIX & 1) : 0);
            if (s == 0) put_field(A, pos, v[i][j], off, w, p.one);
            else if (s == 1) put_field(B, pos, v[i][j], off, w, p.one);
            else put_field(C, pos, v[i][j], off, w, p.one);
        });
        if (MASK) {
            const uint64_t gb = p.block_offset + blk;
            if (R::BBITS) {
                mask_b<L, MODE, SPEC, (SE_SPEC & 1) != 0, B256>(p, gb, A, B);   // row a7
                mask_c<R::BW, R::BBYTES, SPEC>(p, gb, B, C);                // row a8
            } else {
                mask_c<R::AW, R::ABYTES, SPEC>(p, gb, A, C);                // C21 (L = 1)
            }
        }
        smem_put_record<R::AW, R::ABITS>(sa, (uint32_t)tid * R::ABITS, A);
        if (R::BBITS) smem_put_record<R::BW, R::BBITS>(sb, (uint32_t)tid * R::BBITS, B);
        smem_put_record<R::CW, R::CBITS>(sc, (uint32_t)tid * R::CBITS, C);
    }
    __syncthreads();

    // row a9: 128-bit coalesced stores of the CTA's slice of each stream;
    // A' = A ^ keystream on the way out (row a6, XOR half)
    const uint64_t a0 = cta * (BPC / 8ull) * R::ABITS, c0 = cta * (BPC / 8ull) * R::CBITS;
    if (p.ks_in_a) {
        // row a6: A' = A ^ the keystream k_cipher_ctr wrote into A' just before
        asm volatile("griddepcontrol.wait;" ::: "memory");
        copy_s2g_xor_global<BPC>(p.a + a0, sa, min((uint64_t)SA_W * 4, p.a_bytes - a0), tid);
    } else {
        // row a6: encrypt the CTA's A slice (whole AES counter blocks) on the way out
        const uint64_t alen = min((uint64_t)SA_W * 4, p.a_bytes - a0);
        const uint32_t nblk = (uint32_t)((alen + 15) / 16);
        for (uint32_t j = tid; j < nblk; j += BPC) {
            uint32_t x[4];
            ctr_add(p.ctr, a0 / 16 + j, x);
            aes128_block(aes, p.rk, x);
#pragma unroll
            for (int k = 0; k < 4; ++k) sa[4 * j + k] ^= bswap32(x[k]);
        }
        __syncthreads();
        copy_s2g<BPC>(p.a + a0, sa, alen, tid);
    }
    if (R::BBITS) {
        const uint64_t b0 = cta * (BPC / 8ull) * R::BBITS;
        copy_s2g<BPC>(p.b + b0, sb, min((uint64_t)SB_W * 4, p.b_bytes - b0), tid);
    }
    copy_s2g<BPC>(p.c + c0, sc, min((uint64_t)SC_W * 4, p.c_bytes - c0), tid);
}

// ---------------------------------------------------------------- recover

// MODE 0: unmask, unpack, inverse lifting, store bytes, report.  MODE 1:
// unmask, unpack and scatter the footprint's coefficients into p.ws; the
// whole-matrix inverse (and the report) follow in k_full.cu.
// The keystream of the whole A stream sits in p.ks (k_cipher_ctr, launched
// before with programmatic stream serialization); it is waited for and
// applied after the SHA-512 unmask of C, which does not need A.
#ifndef SE_REC_STAGE
#define SE_REC_STAGE 0
#endif
// S256: the single-file recovery kernels (whose FusedParams carry the
// launch's SHA-256 schedule constants p.s256) also specialise the B-mask
// schedule (SE_SPEC_REC256; batches have no per-file s256).
template <int L, bool MASK, int MODE = 0, int BPC = kBlocksPerCta, bool SPEC = true, bool S256 = false>
__device__ __forceinline__ void recover_cta(const FusedParams& p, const uint64_t cta) {
    using R = Rec<L, MODE>;
    static_assert((BPC * R::ABITS) % 128 == 0 && (BPC * R::BBITS) % 128 == 0 && (BPC * R::CBITS) % 128 == 0,
                  "CTA stream slices must be whole 16-byte units (and A whole AES blocks)");
    constexpr int SA_W = BPC * R::ABITS / 32;
    constexpr int SB_W = R::BBITS ? BPC * R::BBITS / 32 : 4;
    constexpr int SC_W = BPC * R::CBITS / 32;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ __align__(16) uint32_t sb[SB_W];
    __shared__ __align__(16) uint32_t sc[SC_W];
    __shared__ unsigned long long s_first;
    __shared__ unsigned int s_bad;

    const int tid = threadIdx.x;
    const uint64_t blk = cta * BPC + tid;
    const uint64_t a0 = cta * (BPC / 8ull) * R::ABITS, c0 = cta * (BPC / 8ull) * R::CBITS;
    const uint64_t alen = min((uint64_t)SA_W * 4, p.a_bytes - a0);
    __shared__ AesSmem aes;
    if (!p.ks_in_out) aes_load_tables(aes, tid, BPC);     // constant tables: before the grid dependency
    if (tid == 0) { s_first = ~0ull; s_bad = 0; }
    // fragments / report written by earlier work.  With p.ks_in_out the kernel
    // right before is the keystream kernel (a normal launch: everything earlier
    // is complete), so only its keystream is waited for, just before use.
    if (!p.ks_in_out) asm volatile("griddepcontrol.wait;" ::: "memory");
    copy_g2s<BPC>(sa, p.a + a0, alen, SA_W * 4, tid);
    if (R::BBITS) {
        const uint64_t b0 = cta * (BPC / 8ull) * R::BBITS;
        copy_g2s<BPC>(sb, p.b + b0, min((uint64_t)SB_W * 4, p.b_bytes - b0), SB_W * 4, tid);
    }
    copy_g2s<BPC>(sc, p.c + c0, min((uint64_t)SC_W * 4, p.c_bytes - c0), SC_W * 4, tid);
    __syncthreads();

    // C needs only B' (C19): its SHA-512 unmask runs before the keystream is needed
    const bool valid = blk < p.n_blocks;
    const uint64_t gb = p.block_offset + blk;
    uint32_t A[R::AW], B[R::BW], C[R::CW];
    if (valid) {
        if (R::BBITS) smem_get_record<R::BW, R::BBITS>(sb, SB_W, (uint32_t)tid * R::BBITS, B);
        else B[0] = 0;
        smem_get_record<R::CW, R::CBITS>(sc, SC_W, (uint32_t)tid * R::CBITS, C);
        if (MASK && R::BBITS) mask_c<R::BW, R::BBYTES, SPEC>(p, gb, B, C);    // C from B'
    }
    if (p.ks_in_out == 1) {
        // row a6: the keystream kernel wrote this CTA's A-slice keystream into the
        // first row run of the CTA's own output region (which only this CTA
        // writes, after this read): A' -> A in shared memory
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint64_t b0 = cta * BPC, br0 = b0 / p.bpr, bc0 = b0 - br0 * p.bpr;
        xor_g2s<BPC>(sa, p.out + 8 * br0 * (uint64_t)p.width + 8 * bc0, alen, tid);
    } else if (p.ks_in_out == 2) {
        // FULL mode: the keystream of the whole A stream sits at the start of the
        // output, which only the inverse transform after this kernel writes
        asm volatile("griddepcontrol.wait;" ::: "memory");
        xor_g2s<BPC>(sa, p.out + a0, alen, tid);
    } else {
        // row a6: decrypt the CTA's A slice (whole AES counter blocks) in shared memory
        const uint32_t nblk = (uint32_t)((alen + 15) / 16);
        for (uint32_t j = tid; j < nblk; j += BPC) {
            uint32_t x[4];
            ctr_add(p.ctr, a0 / 16 + j, x);
            aes128_block(aes, p.rk, x);
#pragma unroll
            for (int k = 0; k < 4; ++k) sa[4 * j + k] ^= bswap32(x[k]);
        }
    }
    __syncthreads();                                                         // plain A ready

    // SE_REC_STAGE: the CTA's bytes (8 rows x 8*BPC) go through shared memory
    // and leave as 16-byte stores, one contiguous run per row, when the CTA's
    // blocks lie in one block row, wholly inside n, on 16-byte aligned rows.
    // Measured slower (C2 masked recover 183.5 vs 188.3 GB/s, plain 496 vs
    // 530; host-mapped output still slower than staged copies), so off.
#if SE_REC_STAGE
    __shared__ __align__(16) uint32_t so[MODE == 0 ? 16 * BPC : 4];
    const uint64_t sblk0 = cta * BPC, sbr0 = sblk0 / p.bpr, sbc0 = sblk0 - sbr0 * p.bpr;
    const bool staged = MODE == 0 && sbc0 + BPC <= p.bpr && (p.width % 16) == 0 && (sbc0 % 2) == 0 &&
                        8 * sbr0 * (uint64_t)p.width + 8 * sbc0 + 7ull * p.width + 8 * BPC <= p.n_bytes;
#endif
    bool bad = false;
    if (valid) {
        smem_get_record<R::AW, R::ABITS>(sa, SA_W, (uint32_t)tid * R::ABITS, A);
        if (MASK) {
            if (R::BBITS) mask_b<L, MODE, SPEC, S256 || (SE_SPEC & 1) != 0>(p, gb, A, B);   // B from A
            else mask_c<R::AW, R::ABYTES, SPEC>(p, gb, A, C);                // C21 (L = 1)
        }
        int v[8][8];
        for_each_field<L, MODE>([&](int s, int pos, int i, int j, int w) {
            const int off = (s == 0 && MODE == 0) ? (1 << (w - 1)) - 128 : (1 << (w - 1));   // see protect
            if (s == 0) v[i][j] = get_field(A, pos, off, w, p.one);
            else if (s == 1) v[i][j] = get_field(B, pos, off, w, p.one);
            else v[i][j] = get_field(C, pos, off, w, p.one);
        });
        const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
        if constexpr (MODE == 0) {
#if SE_MASK_MIX & 2
            dwt8_inv_mix<L>(v, p.one);                                       // uncentered bytes
#else
            dwt8_inv<L>(v, p.one);                                           // uncentered bytes
#endif
#if SE_MASK_MIX & 4
            bad = out_of_range_pairs(v, p.one);   // any sample outside [0, 255]
#else
            int orv = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) orv |= v[i][j];
            bad = (orv & ~0xff) != 0;      // any sample outside [0, 255]
#endif
#if SE_REC_STAGE
            if (staged) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint2 q;
                    q.x = __byte_perm(__byte_perm(v[i][0], v[i][1], 0x0040), __byte_perm(v[i][2], v[i][3], 0x0040), 0x5410);
                    q.y = __byte_perm(__byte_perm(v[i][4], v[i][5], 0x0040), __byte_perm(v[i][6], v[i][7], 0x0040), 0x5410);
                    *reinterpret_cast<uint2*>(so + (i * 8 * BPC + 8 * tid) / 4) = q;
                }
            } else
#endif
            store_block(p.out, p.n_bytes, p.width, br, bc, v);
        } else {
            footprint_full<L, true>(p, br, bc, v);
        }
    }
#if SE_REC_STAGE
    if (staged) {
        __syncthreads();
        for (int idx = tid; idx < 4 * BPC; idx += BPC) {
            const int row = idx / (BPC / 2), c16 = idx % (BPC / 2);
            uint8_t* dst = p.out + (8 * sbr0 + row) * (uint64_t)p.width + 8 * sbc0 + 16 * c16;
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(so + (row * 8 * BPC + 16 * c16) / 4);
        }
    }
#endif
    if (MODE == 0 && p.report != nullptr) {
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

}  // namespace se
