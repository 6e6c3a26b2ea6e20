// k_dct.cu — the Chapter 4 DCT 8x8 selective encryption of bitmaps (row f3;
// PAPER.md P:1403-1489, include/se_dct.h).
//
// One thread owns one 8x8 block position (all colour layers), one CTA 128
// consecutive positions.  Per block and layer, in fp32:
//   * the 6 selected coefficients of Eq. 4.1 by a separable pass
//     that forms only what they need: per row the sums s = f(y) + f(7-y) and
//     differences d = f(y) - f(7-y) give the row frequencies 0, 1, 2; the
//     column pass combines those into [1,0], [2,0], [0,1], [1,1], [0,2].  The
//     DC is the exact pixel sum / 8 (Eq. 4.4), so its rounding is exact;
//   * Fragment 1: rint, 11-bit sign-magnitude store, 66-bit record
//     packed into shared memory, written out XORed with the AES-CTR keystream
//     that k_cipher_ctr put into the stream before (programmatic launch);
//   * Fragment 2 = iDCT of the block with DC := 1024 and the 5 AC := 0
//     (P:1487).  By linearity that is x - (iDCT of the 6 selected real
//     coefficients), i.e. the pixel minus a rank-6 separable correction —
//     formed directly, without the 58 other coefficients the paper's
//     pad-and-invert computes and immediately inverts (f3);
//   * level 2: XOR with SHA-512 of the record.
// Recovery: the same 6 coefficients of Fragment 2, and the image = P +
// (iDCT of stored - computed) + the DC terms, rounded to bytes.  Rounding to
// bytes: clamp to [0, 255] then add 1.5 * 2^23 (round-half-even into the low
// mantissa byte), packed with PRMT.
#include <cuda_runtime.h>

#include "fused_cta.cuh"
#include "sha2_device.cuh"
#include "sha2_spec.cuh"
#include "tables.h"

namespace se {
namespace {

constexpr float kA0 = (float)SE_DCT_A0;   // alpha(0) = sqrt(1/8), Eq. 4.3

// D[u][x] = alpha(u) cos(pi (2x+1) u / 16) for u = 1, 2 and x = 0..7
// (D[1][7-x] = -D[1][x], D[2][7-x] = D[2][x]); x is a compile-time constant
// at every use, so these fold to immediates.
__device__ __forceinline__ constexpr float d1(int x) {
    constexpr float h1 = (float)SE_DCT_H1, h3 = (float)SE_DCT_H3, h5 = (float)SE_DCT_H5, h7 = (float)SE_DCT_H7;
    return x == 0 ? h1 : x == 1 ? h3 : x == 2 ? h5 : x == 3 ? h7 : x == 4 ? -h7 : x == 5 ? -h5 : x == 6 ? -h3 : -h1;
}
__device__ __forceinline__ constexpr float d2(int x) {
    constexpr float h2 = (float)SE_DCT_H2, h6 = (float)SE_DCT_H6;
    return (x == 0 || x == 7) ? h2 : (x == 1 || x == 6) ? h6 : (x == 2 || x == 5) ? -h6 : -h2;
}

// byte `k` of word w, minus 128, as an exact float: PRMT the byte under the
// exponent of 2^23, subtract 2^23 + 128 (ALU + FMA pipe) ...
__device__ __forceinline__ float px(uint32_t w, int k) {
    return __int_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | k)) - 8388736.0f;
}
// ... or I2F.U8 with a byte selector (conversion pipe, no ALU instruction):
// faster in the DCT 8x8 transform (fwd 32.9 -> 31.0 us at 4800^2), slower in
// the SE kernels (level 2: 119.3 -> 118.2 GB/s), so used there only.
__device__ __forceinline__ float px_cvt(uint32_t w, int k) {
    float f;
    asm("cvt.rn.f32.u8 %0, %1;" : "=f"(f) : "h"((unsigned short)(unsigned char)(w >> (8 * k))));
    return f - 128.0f;
}

// rint(clamp(v, 0, 255)) in the low byte of the result (D3: round half to
// even).  SE_DCT_F2I=1: one saturating conversion (cvt.rni.sat.u8.f32; the
// clamp and the rounding commute for these bounds) instead of two FMNMX on the
// ALU pipe - the level-2 kernels are ALU-bound by SHA-512.
#ifndef SE_DCT_F2I
#define SE_DCT_F2I 1
#endif
__device__ __forceinline__ uint32_t rnd_u8(float v) {
#if SE_DCT_F2I
    uint32_t r;
    asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(v));
    return r;
#else
    return __float_as_uint(fminf(fmaxf(v, 0.0f), 255.0f) + 12582912.0f);
#endif
}

// bytes a, b, c, d (each < 256) -> one word, a lowest.  SE_DCT_I2IP=1: two
// saturating pack conversions (I2IP) instead of three PRMT - measured mixed
// (level 1 +1 %, level 2 protect -1 %, 4800x4800), so 0.
#ifndef SE_DCT_I2IP
#define SE_DCT_I2IP 0
#endif
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
#if SE_DCT_I2IP
    uint32_t lo, r;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(d), "r"(c), "r"(0u));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(a), "r"(lo));
    return r;
#else
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
#endif
}

// 11-bit store (D5): rint, |q| <= 1023, sign bit then magnitude
__device__ __forceinline__ uint32_t store11(float c) {
    int q = __float_as_int(c + 12582912.0f) - 0x4B400000;
    q = max(-1023, min(1023, q));
    return q < 0 ? (0x400u | (uint32_t)(-q)) : (uint32_t)q;
}
__device__ __forceinline__ float load11(uint32_t f) {
    const float m = (float)(f & 1023u);
    return (f & 0x400u) ? -m : m;
}

// the 6 selected coefficients of one centered block (t = pixel sum: DC = t/8)
struct Sel6 { float t, c01, c10, c20, c11, c02; };


// Row-streaming: each row's 8 bytes become floats, then their row
// frequencies 0, 1, 2; the 64 floats are never live together.
__device__ __forceinline__ Sel6 select6(const uint32_t (&pw)[16]) {
    float T0[8], T1[8], T2[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        float f[8], s[4], d[4];
#pragma unroll
        for (int y = 0; y < 8; ++y) f[y] = px(pw[2 * x + (y >> 2)], y & 3);
#pragma unroll
        for (int k = 0; k < 4; ++k) { s[k] = f[k] + f[7 - k]; d[k] = f[k] - f[7 - k]; }
        T0[x] = (s[0] + s[3]) + (s[1] + s[2]);
        T1[x] = fmaf(d1(3), d[3], fmaf(d1(2), d[2], fmaf(d1(1), d[1], d1(0) * d[0])));
        T2[x] = fmaf(d2(1), s[1] - s[2], d2(0) * (s[0] - s[3]));
    }
    Sel6 r;
    float u[4], e[4], g[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        u[k] = T0[k] + T0[7 - k];
        e[k] = T0[k] - T0[7 - k];
        g[k] = T1[k] - T1[7 - k];
    }
    r.t = (u[0] + u[3]) + (u[1] + u[2]);                                        // exact
    r.c10 = kA0 * fmaf(d1(3), e[3], fmaf(d1(2), e[2], fmaf(d1(1), e[1], d1(0) * e[0])));
    r.c20 = kA0 * fmaf(d2(1), u[1] - u[2], d2(0) * (u[0] - u[3]));
    r.c01 = kA0 * (((T1[0] + T1[1]) + (T1[2] + T1[3])) + ((T1[4] + T1[5]) + (T1[6] + T1[7])));
    r.c11 = fmaf(d1(3), g[3], fmaf(d1(2), g[2], fmaf(d1(1), g[1], d1(0) * g[0])));
    r.c02 = kA0 * (((T2[0] + T2[1]) + (T2[2] + T2[3])) + ((T2[4] + T2[5]) + (T2[6] + T2[7])));
    return r;
}

// bytes of f + bias + sum_k w_k D[u_k][x] D[v_k][y] over the 5 selected AC,
// rounded to [0, 255], where f = the centered pixels held in pw (row x in
// words 2x, 2x+1); the result replaces pw row by row.  The pixels are
// converted again here (PRMT + FADD) rather than kept live as 64 floats.
__device__ __forceinline__ void rebuild(uint32_t (&pw)[16], float bias, float w10, float w20, float w01,
                                        float w11, float w02) {
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("" : "+r"(pw[k]));    // no reuse of select6's floats
    const float hA = kA0 * w02 * d2(0), hB = kA0 * w02 * d2(1);    // v = 2 terms, h(y) = hA, hB, -hB, -hA
    const float a01 = kA0 * w01;
    const float a10 = kA0 * w10, a20 = kA0 * w20;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        float f[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) f[y] = px(pw[2 * x + (y >> 2)], y & 3);
        const float R = fmaf(a20, d2(x), fmaf(a10, d1(x), bias));       // v = 0 terms + bias
        const float g1 = fmaf(w11, d1(x), a01);                          // v = 1 coefficient of row x
        uint32_t b[8];
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const float h = y == 0 ? hA : y == 1 ? hB : y == 2 ? -hB : -hA;
            const float base = R + h;
            b[y] = rnd_u8(f[y] + fmaf(g1, d1(y), base));
            b[7 - y] = rnd_u8(f[7 - y] + fmaf(-g1, d1(y), base));
        }
        pw[2 * x] = pack4(b[0], b[1], b[2], b[3]);
        pw[2 * x + 1] = pack4(b[4], b[5], b[6], b[7]);
    }
}

// raw bytes of the 8 rows of block position (br, bc), all C channels
template <int C>
__device__ __forceinline__ void load_rows(const uint8_t* __restrict__ img, uint32_t W, uint64_t br, uint64_t bc,
                                          uint32_t (&w)[8][2 * C]) {
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        const uint8_t* row = img + ((8 * br + x) * (uint64_t)W + 8 * bc) * C;
        if constexpr (C == 4) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(row) + k);
                w[x][4 * k] = q.x; w[x][4 * k + 1] = q.y; w[x][4 * k + 2] = q.z; w[x][4 * k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const uint2 q = __ldg(reinterpret_cast<const uint2*>(row) + k);
                w[x][2 * k] = q.x; w[x][2 * k + 1] = q.y;
            }
        }
    }
}

// channel CH's 64 bytes as 16 words (row x: words 2x, 2x+1)
template <int C, int CH>
__device__ __forceinline__ void gather(const uint32_t (&w)[8][2 * C], uint32_t (&pw)[16]) {
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        if constexpr (C == 1) {
            pw[2 * x] = w[x][0]; pw[2 * x + 1] = w[x][1];
        } else {
            uint32_t b[8];
#pragma unroll
            for (int y = 0; y < 8; ++y) {
                const int k = y * C + CH;
                b[y] = __byte_perm(w[x][k >> 2], 0u, 0x4440u | (k & 3));
            }
            pw[2 * x] = pack4(b[0], b[1], b[2], b[3]);
            pw[2 * x + 1] = pack4(b[4], b[5], b[6], b[7]);
        }
    }
}

template <int C, int CH>
__device__ __forceinline__ void store_rows(uint8_t* __restrict__ img, uint32_t W, uint64_t br, uint64_t bc,
                                           const uint32_t (&pw)[16]) {
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        uint8_t* row = img + ((8 * br + x) * (uint64_t)W + 8 * bc) * C;
        if constexpr (C == 1) {
            *reinterpret_cast<uint2*>(row) = make_uint2(pw[2 * x], pw[2 * x + 1]);
        } else {
#pragma unroll
            for (int y = 0; y < 8; ++y) row[y * C + CH] = (uint8_t)(pw[2 * x + (y >> 2)] >> (8 * (y & 3)));
        }
    }
}

// the 66-bit record of P:1423 / P:1483 as big-endian words (r[2]: top 2 bits)
__device__ __forceinline__ void pack_record(const uint32_t (&q)[6], uint32_t (&r)[3]) {
    r[0] = q[0] << 21 | q[1] << 10 | q[2] >> 1;
    r[1] = (q[2] & 1u) << 31 | q[3] << 20 | q[4] << 9 | q[5] >> 2;
    r[2] = (q[5] & 3u) << 30;
}
__device__ __forceinline__ void unpack_record(const uint32_t (&r)[3], uint32_t (&q)[6]) {
    q[0] = r[0] >> 21;
    q[1] = (r[0] >> 10) & 0x7ffu;
    q[2] = (r[0] & 0x3ffu) << 1 | r[1] >> 31;
    q[3] = (r[1] >> 20) & 0x7ffu;
    q[4] = (r[1] >> 9) & 0x7ffu;
    q[5] = (r[1] & 0x1ffu) << 2 | r[2] >> 30;
}

// level 2 (D9, D10): pw ^= SHA-512(message of record r)
template <bool KEYED>
__device__ __forceinline__ void mask_level2(const DctParams& p, uint64_t gr, const uint32_t (&r)[3],
                                            uint32_t (&pw)[16]) {
    W64 W[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) W[k] = W64{0u, 0u};
    const uint64_t h0[8] = {p.h512[0], p.h512[1], p.h512[2], p.h512[3],
                            p.h512[4], p.h512[5], p.h512[6], p.h512[7]};
    uint64_t H[8];
    if constexpr (KEYED) {                               // K || IV || be64(gr) || rec9, 49 bytes
#pragma unroll
        for (int k = 0; k < 4; ++k) W[k] = W64{p.kiv[2 * k + 1], p.kiv[2 * k]};
        W[4] = W64{(uint32_t)gr, (uint32_t)(gr >> 32)};
        W[5] = W64{r[1], r[0]};
        W[6] = W64{0u, r[2] | 0x00800000u};               // FIPS 180-4 §5.1.2 pad at byte 49
        W[15].lo = 49 * 8;
        const uint64_t st[8] = {p.mid512[0], p.mid512[1], p.mid512[2], p.mid512[3],
                                p.mid512[4], p.mid512[5], p.mid512[6], p.mid512[7]};
        sha512_from_round_spec<4, kDctMsgKeyed>(st, h0, W, p.s512, H, p.one);
    } else {                                             // rec9, 9 bytes
        W[0] = W64{r[1], r[0]};
        W[1] = W64{0u, r[2] | 0x00800000u};               // pad at byte 9
        W[15].lo = 9 * 8;
        sha512_from_round_spec<0, kDctMsgUnkeyed>(h0, h0, W, p.s512, H, p.one);   // zero words folded
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {                        // digest byte 8x+y on pixel (x, y)
        pw[2 * x] ^= bswap32((uint32_t)(H[x] >> 32));
        pw[2 * x + 1] ^= bswap32((uint32_t)H[x]);
    }
}

template <int C>
struct DctCta {
    static constexpr int kRecBits = 66;
    static constexpr int kSaWords = kBlocksPerCta * C * kRecBits / 32;   // 264 * C
};

template <int C, int CH, int LEVEL, bool KEYED>
__device__ __forceinline__ void protect_layer(const DctParams& p, const uint32_t (&w)[8][2 * C], uint64_t pos,
                                              uint64_t br, uint64_t bc, uint32_t* sa, int tid) {
    uint32_t pw[16];
    gather<C, CH>(w, pw);
    const Sel6 s = select6(pw);
    uint32_t q[6], r[3];
    q[0] = store11(s.t * 0.125f);                                         // Eq. 4.4, exact
    q[1] = store11(s.c01); q[2] = store11(s.c10); q[3] = store11(s.c20);
    q[4] = store11(s.c11); q[5] = store11(s.c02);
    pack_record(q, r);
    smem_put_record<3, 66>(sa, (uint32_t)(tid * C + CH) * 66u, r);
    // Fragment 2 = x - t/64 - sum of the 5 AC terms (P:1487 pad-and-invert)
    rebuild(pw, 128.0f - s.t * 0.015625f, -s.c10, -s.c20, -s.c01, -s.c11, -s.c02);
    if constexpr (LEVEL == 2) mask_level2<KEYED>(p, p.block_offset + pos * C + CH, r, pw);
    store_rows<C, CH>(p.out, p.width, br, bc, pw);
}

template <int C, int CH, int LEVEL, bool KEYED>
__device__ __forceinline__ void recover_layer(const DctParams& p, const uint32_t (&w)[8][2 * C], uint64_t pos,
                                              uint64_t br, uint64_t bc, const uint32_t* sa, int tid) {
    uint32_t r[3], q[6], pw[16];
    smem_get_record<3, 66>(sa, DctCta<C>::kSaWords, (uint32_t)(tid * C + CH) * 66u, r);
    unpack_record(r, q);
    gather<C, CH>(w, pw);
    if constexpr (LEVEL == 2) mask_level2<KEYED>(p, p.block_offset + pos * C + CH, r, pw);
    const Sel6 s = select6(pw);
    // image = P + (iDCT of stored - computed over the 6 positions), + 128
    const float bias = fmaf(load11(q[0]), 0.125f, 128.0f) - s.t * 0.015625f;
    rebuild(pw, bias, load11(q[2]) - s.c10, load11(q[3]) - s.c20, load11(q[1]) - s.c01,
            load11(q[4]) - s.c11, load11(q[5]) - s.c02);
    store_rows<C, CH>(p.out, p.width, br, bc, pw);
}

// AESF: the AES-CTR of Fragment 1 runs in this kernel (the CTA's A slice is
// 66*C whole counter blocks; 5 KB T-tables in shared memory), no keystream
// kernel.  Otherwise the keystream comes from k_cipher_ctr (programmatic
// launch) and is XORed at the copy-out.
#ifndef SE_DCT_FUSED_AES
#define SE_DCT_FUSED_AES 1
#endif

template <int C>
__device__ __forceinline__ void xor_keystream(const DctParams& p, const AesSmem& aes, uint32_t* sa, uint64_t a0,
                                              uint64_t alen, int tid) {
    const uint32_t nblk = (uint32_t)((alen + 15) / 16);
    for (uint32_t j = tid; j < nblk; j += kBlocksPerCta) {
        uint32_t x[4];
        ctr_add(p.ctr, a0 / 16 + j, x);
        aes128_block(aes, p.rk, x);
#pragma unroll
        for (int k = 0; k < 4; ++k) sa[4 * j + k] ^= bswap32(x[k]);
    }
}

template <int C, int LEVEL, bool KEYED, bool AESF>
__global__ void __launch_bounds__(kBlocksPerCta) k_dct_protect(const DctParams p) {
    constexpr int SA_W = DctCta<C>::kSaWords;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ AesSmem aes;
    const int tid = threadIdx.x;
    const uint64_t pos = (uint64_t)blockIdx.x * kBlocksPerCta + tid;
    for (int i = tid; i < SA_W; i += kBlocksPerCta) sa[i] = 0;
    if constexpr (AESF) aes_load_tables(aes, tid, kBlocksPerCta);
    __syncthreads();
    if (pos < p.n_pos) {
        const uint64_t br = pos / p.bpr, bc = pos - br * p.bpr;
        uint32_t w[8][2 * C];
        load_rows<C>(p.in, p.width, br, bc, w);
        protect_layer<C, 0, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 1) protect_layer<C, 1, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 2) protect_layer<C, 2, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 3) protect_layer<C, 3, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
    }
    __syncthreads();
    const uint64_t a0 = (uint64_t)blockIdx.x * SA_W * 4;
    const uint64_t alen = min((uint64_t)SA_W * 4, p.a_bytes - a0);
    if constexpr (AESF) {
        xor_keystream<C>(p, aes, sa, a0, alen, tid);                  // Fragment 1 encrypted
        __syncthreads();
        copy_s2g(p.a + a0, sa, alen, tid);
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");          // keystream kernel complete
        copy_s2g_xor_global(p.a + a0, sa, alen, tid);
    }
}

template <int C, int LEVEL, bool KEYED, bool AESF>
__global__ void __launch_bounds__(kBlocksPerCta) k_dct_recover(const DctParams p) {
    constexpr int SA_W = DctCta<C>::kSaWords;
    __shared__ __align__(16) uint32_t sa[SA_W];
    __shared__ AesSmem aes;
    const int tid = threadIdx.x;
    const uint64_t pos = (uint64_t)blockIdx.x * kBlocksPerCta + tid;
    const uint64_t a0 = (uint64_t)blockIdx.x * SA_W * 4;
    const uint64_t alen = min((uint64_t)SA_W * 4, p.a_bytes - a0);
    copy_g2s(sa, p.a + a0, alen, SA_W * 4, tid);
    if constexpr (AESF) aes_load_tables(aes, tid, kBlocksPerCta);
    const bool valid = pos < p.n_pos;
    const uint64_t br = valid ? pos / p.bpr : 0, bc = valid ? pos - br * p.bpr : 0;
    uint32_t w[8][2 * C];
    if (valid) load_rows<C>(p.in, p.width, br, bc, w);
    if constexpr (AESF) {
        __syncthreads();
        xor_keystream<C>(p, aes, sa, a0, alen, tid);                  // Fragment 1 decrypted
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");          // keystream kernel complete
        xor_g2s(sa, p.ks + a0, alen, tid);
    }
    __syncthreads();
    if (valid) {
        recover_layer<C, 0, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 1) recover_layer<C, 1, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 2) recover_layer<C, 2, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
        if constexpr (C > 3) recover_layer<C, 3, LEVEL, KEYED>(p, w, pos, br, bc, sa, tid);
    }
}

template <int C, int CH>
__device__ __forceinline__ void select_layer(const DctParams& p, const uint32_t (&w)[8][2 * C], uint64_t pos) {
    uint32_t pw[16];
    gather<C, CH>(w, pw);
    const Sel6 s = select6(pw);
    float* o = p.coef + (pos * C + CH) * 6;
    o[0] = s.t * 0.125f; o[1] = s.c01; o[2] = s.c10; o[3] = s.c20; o[4] = s.c11; o[5] = s.c02;
}

template <int C>
__global__ void __launch_bounds__(kBlocksPerCta) k_dct_select(const DctParams p) {
    const uint64_t pos = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (pos >= p.n_pos) return;
    const uint64_t br = pos / p.bpr, bc = pos - br * p.bpr;
    uint32_t w[8][2 * C];
    load_rows<C>(p.in, p.width, br, bc, w);
    select_layer<C, 0>(p, w, pos);
    if constexpr (C > 1) select_layer<C, 1>(p, w, pos);
    if constexpr (C > 2) select_layer<C, 2>(p, w, pos);
    if constexpr (C > 3) select_layer<C, 3>(p, w, pos);
}

// ---------------------------------------------------------------- full DCT 8x8 (Table 4.1)

// D[u][x] = alpha(u) cos(pi (2x+1) u / 16) for any u, x (Eq. 4.1, 4.3):
// reduce (2x+1)u mod 32 onto [0, 8] with the cosine's symmetries.
__device__ __forceinline__ constexpr float hcos(int k) {      // cos(k pi / 16) / 2, k = 0..8
    return k == 0 ? 0.5f : k == 1 ? (float)SE_DCT_H1 : k == 2 ? (float)SE_DCT_H2 : k == 3 ? (float)SE_DCT_H3
         : k == 4 ? (float)SE_DCT_H4 : k == 5 ? (float)SE_DCT_H5 : k == 6 ? (float)SE_DCT_H6
         : k == 7 ? (float)SE_DCT_H7 : 0.0f;
}
__device__ __forceinline__ constexpr float dm(int u, int x) {
    return u == 0 ? kA0
         : (((2 * x + 1) * u) % 32 > 16 ? 32 - ((2 * x + 1) * u) % 32 : ((2 * x + 1) * u) % 32) > 8
               ? -hcos(16 - (((2 * x + 1) * u) % 32 > 16 ? 32 - ((2 * x + 1) * u) % 32 : ((2 * x + 1) * u) % 32))
               : hcos(((2 * x + 1) * u) % 32 > 16 ? 32 - ((2 * x + 1) * u) % 32 : ((2 * x + 1) * u) % 32);
}

// 8-point orthonormal DCT-II (Eq. 4.1 in one dimension), even/odd split:
// even u use s = f(x) + f(7-x), odd u use d = f(x) - f(7-x).
__device__ __forceinline__ void dct8_1d(const float (&f)[8], float (&X)[8]) {
    float s[4], d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { s[k] = f[k] + f[7 - k]; d[k] = f[k] - f[7 - k]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const float (&v)[4] = (u & 1) ? d : s;
        X[u] = fmaf(dm(u, 3), v[3], fmaf(dm(u, 2), v[2], fmaf(dm(u, 1), v[1], dm(u, 0) * v[0])));
    }
}

// its inverse (Eq. 4.2): f(x) = e(x) + o(x), f(7-x) = e(x) - o(x)
__device__ __forceinline__ void idct8_1d(const float (&X)[8], float (&f)[8]) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const float e = fmaf(dm(6, x), X[6], fmaf(dm(4, x), X[4], fmaf(dm(2, x), X[2], dm(0, x) * X[0])));
        const float o = fmaf(dm(7, x), X[7], fmaf(dm(5, x), X[5], fmaf(dm(3, x), X[3], dm(1, x) * X[1])));
        f[x] = e + o;
        f[7 - x] = e - o;
    }
}

template <int C, int CH>
__device__ __forceinline__ void dct8_layer(const DctParams& p, const uint32_t (&w)[8][2 * C], uint64_t br,
                                           uint64_t bc) {
    uint32_t pw[16];
    gather<C, CH>(w, pw);
    float T[8][8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {                                       // rows
        float f[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) f[y] = px_cvt(pw[2 * x + (y >> 2)], y & 3);
        dct8_1d(f, T[x]);
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) {                                       // columns
        float col[8], Y[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) col[x] = T[x][v];
        dct8_1d(col, Y);
#pragma unroll
        for (int u = 0; u < 8; ++u) T[u][v] = Y[u];                     // (u, v) in place
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        float* row = p.coef + ((8 * br + u) * (uint64_t)p.width + 8 * bc) * C;
        if constexpr (C == 1) {
            reinterpret_cast<float4*>(row)[0] = make_float4(T[u][0], T[u][1], T[u][2], T[u][3]);
            reinterpret_cast<float4*>(row)[1] = make_float4(T[u][4], T[u][5], T[u][6], T[u][7]);
        } else {
#pragma unroll
            for (int v = 0; v < 8; ++v) row[v * C + CH] = T[u][v];
        }
    }
}

#ifndef SE_DCT8_MINB
#define SE_DCT8_MINB 1
#endif
template <int C>
__global__ void __launch_bounds__(kBlocksPerCta, SE_DCT8_MINB) k_dct8_fwd(const DctParams p) {
    const uint64_t pos = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (pos >= p.n_pos) return;
    const uint64_t br = pos / p.bpr, bc = pos - br * p.bpr;
    uint32_t w[8][2 * C];
    load_rows<C>(p.in, p.width, br, bc, w);
    dct8_layer<C, 0>(p, w, br, bc);
    if constexpr (C > 1) dct8_layer<C, 1>(p, w, br, bc);
    if constexpr (C > 2) dct8_layer<C, 2>(p, w, br, bc);
    if constexpr (C > 3) dct8_layer<C, 3>(p, w, br, bc);
}

template <int C, int CH>
__device__ __forceinline__ void idct8_layer(const DctParams& p, uint64_t br, uint64_t bc) {
    float T[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const float* row = p.coef + ((8 * br + u) * (uint64_t)p.width + 8 * bc) * C;
        if constexpr (C == 1) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(row)), b = __ldg(reinterpret_cast<const float4*>(row) + 1);
            T[u][0] = a.x; T[u][1] = a.y; T[u][2] = a.z; T[u][3] = a.w;
            T[u][4] = b.x; T[u][5] = b.y; T[u][6] = b.z; T[u][7] = b.w;
        } else {
#pragma unroll
            for (int v = 0; v < 8; ++v) T[u][v] = __ldg(row + v * C + CH);
        }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) {                                       // columns
        float col[8], f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) col[u] = T[u][v];
        idct8_1d(col, f);
#pragma unroll
        for (int x = 0; x < 8; ++x) T[x][v] = f[x];
    }
    uint32_t pw[16];
#pragma unroll
    for (int x = 0; x < 8; ++x) {                                       // rows, + 128, bytes
        float f[8];
        idct8_1d(T[x], f);
        uint32_t b[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) b[y] = rnd_u8(f[y] + 128.0f);
        pw[2 * x] = pack4(b[0], b[1], b[2], b[3]);
        pw[2 * x + 1] = pack4(b[4], b[5], b[6], b[7]);
    }
    store_rows<C, CH>(p.out, p.width, br, bc, pw);
}

template <int C>
__global__ void __launch_bounds__(kBlocksPerCta, SE_DCT8_MINB) k_dct8_inv(const DctParams p) {
    const uint64_t pos = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (pos >= p.n_pos) return;
    const uint64_t br = pos / p.bpr, bc = pos - br * p.bpr;
    idct8_layer<C, 0>(p, br, bc);
    if constexpr (C > 1) idct8_layer<C, 1>(p, br, bc);
    if constexpr (C > 2) idct8_layer<C, 2>(p, br, bc);
    if constexpr (C > 3) idct8_layer<C, 3>(p, br, bc);
}

template <int C, int LEVEL, bool KEYED>
void launch_c(const DctParams& p, int op, unsigned grid, cudaStream_t s) {
    if (dct_fused_aes(op, LEVEL, p.n_pos)) {
        if (op == 0) k_dct_protect<C, LEVEL, KEYED, true><<<grid, kBlocksPerCta, 0, s>>>(p);
        else k_dct_recover<C, LEVEL, KEYED, true><<<grid, kBlocksPerCta, 0, s>>>(p);
    } else {
        if (op == 0) launch_pdl(k_dct_protect<C, LEVEL, KEYED, false>, grid, kBlocksPerCta, s, p);
        else launch_pdl(k_dct_recover<C, LEVEL, KEYED, false>, grid, kBlocksPerCta, s, p);
    }
}

template <int C>
void launch_level(const DctParams& p, uint32_t level, bool keyed, int op, unsigned grid, cudaStream_t s) {
    if (op == 2) k_dct_select<C><<<grid, kBlocksPerCta, 0, s>>>(p);
    else if (op == 3) k_dct8_fwd<C><<<grid, kBlocksPerCta, 0, s>>>(p);
    else if (op == 4) k_dct8_inv<C><<<grid, kBlocksPerCta, 0, s>>>(p);
    else if (level == 1) launch_c<C, 1, false>(p, op, grid, s);
    else if (keyed) launch_c<C, 2, true>(p, op, grid, s);
    else launch_c<C, 2, false>(p, op, grid, s);
}

}  // namespace

// Measured (4800x4800): the fused AES pays off where the kernel has issue
// slots to spare (level 1, and recovery, which also skips the keystream
// scratch), not in the ALU-bound level-2 protect (100.4 vs 97.3 us).
// Level-1 protect of large images: the separate lane-table keystream kernel
// wins there (4800x4800: 28.8 -> 27.5 us) but costs a launch on small ones
// (1024x768: 10.6 -> 14.0 us), so from SE_DCT_KS_MIN_POS block positions on.
#ifndef SE_DCT_KS_MIN_POS
#define SE_DCT_KS_MIN_POS 200000
#endif
bool dct_fused_aes(int op, uint32_t level, uint64_t n_pos) {
    if (op == 1) return true;                               // recovery: always in-kernel (no scratch)
    return SE_DCT_FUSED_AES && level == 1 && n_pos < (uint64_t)SE_DCT_KS_MIN_POS;
}

int launch_dct(const DctParams& p, uint32_t channels, uint32_t level, bool keyed, int op, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned grid = (unsigned)((p.n_pos + kBlocksPerCta - 1) / kBlocksPerCta);
    if (channels == 1) launch_level<1>(p, level, keyed, op, grid, s);
    else if (channels == 3) launch_level<3>(p, level, keyed, op, grid, s);
    else launch_level<4>(p, level, keyed, op, grid, s);
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
