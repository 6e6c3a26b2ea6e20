// se_device.cuh — device building blocks of the fused sm_100a kernels.
//
// Everything here is register-resident integer code (no tensor cores: nothing
// on this path is a dense contraction):
//   * 5/3 lifting on 8 / 4 / 2 samples, Eq. 5.1-5.2, update term
//     added (reading C3), whole-sample symmetric extension (C2); floor(a/2) and
//     floor(a/4) are arithmetic shifts (exact floors on two's complement).
//   * MSB-first bit records with compile-time field positions (C9-C11).
//   * SHA-256 / SHA-512 compression on 32-bit lanes (FIPS 180-4 §6.2/§6.4),
//     resuming from a host-computed midstate: the message prefix K||IV is the
//     same for every block (framing C15), so rounds 0-7 (SHA-256) and 0-3
//     (SHA-512) are done once on the host.
//   * AES-128 T-table rounds with the tables in shared memory (FIPS-197 §5.1).
#pragma once
#include <stdint.h>

#include "se_internal.h"
#include "tables.h"

namespace se {

// ------------------------------------------------------------------ lifting
// Forward 1-D lifting of n samples in place: output [s(0..n/2) | d(0..n/2)].
template <int N>
__device__ __forceinline__ void lift_fwd(int (&x)[N]) {
    constexpr int H = N / 2;
    int s[H], d[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int right = (2 * k + 2 < N) ? x[2 * k + 2] : x[2 * k];   // x(N) = x(N-2)
        d[k] = x[2 * k + 1] - ((x[2 * k] + right) >> 1);                  // Eq. 5.1
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int dm1 = (k == 0) ? d[0] : d[k - 1];                       // d(-1) = d(0)
        s[k] = x[2 * k] + ((dm1 + d[k] + 2) >> 2);                        // Eq. 5.2 (+)
    }
#pragma unroll
    for (int k = 0; k < H; ++k) { x[k] = s[k]; x[H + k] = d[k]; }
}

// Exact inverse: undo the update, then undo the predict.
template <int N>
__device__ __forceinline__ void lift_inv(int (&y)[N]) {
    constexpr int H = N / 2;
    int x[N];
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int dm1 = (k == 0) ? y[H] : y[H + k - 1];
        x[2 * k] = y[k] - ((dm1 + y[H + k] + 2) >> 2);
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int right = (2 * k + 2 < N) ? x[2 * k + 2] : x[2 * k];
        x[2 * k + 1] = y[H + k] + ((x[2 * k] + right) >> 1);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) y[k] = x[k];
}

// One 2-D level on the top-left M x M region: rows, then columns (C5).
template <int M>
__device__ __forceinline__ void dwt2_level_fwd(int (&v)[8][8]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int t[M];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = v[i][j];
        lift_fwd<M>(t);
#pragma unroll
        for (int j = 0; j < M; ++j) v[i][j] = t[j];
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        int t[M];
#pragma unroll
        for (int i = 0; i < M; ++i) t[i] = v[i][j];
        lift_fwd<M>(t);
#pragma unroll
        for (int i = 0; i < M; ++i) v[i][j] = t[i];
    }
}

template <int M>
__device__ __forceinline__ void dwt2_level_inv(int (&v)[8][8]) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
        int t[M];
#pragma unroll
        for (int i = 0; i < M; ++i) t[i] = v[i][j];
        lift_inv<M>(t);
#pragma unroll
        for (int i = 0; i < M; ++i) v[i][j] = t[i];
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int t[M];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = v[i][j];
        lift_inv<M>(t);
#pragma unroll
        for (int j = 0; j < M; ++j) v[i][j] = t[j];
    }
}

template <int L>
__device__ __forceinline__ void dwt8_fwd(int (&v)[8][8]) {
    dwt2_level_fwd<8>(v);
    if (L >= 2) dwt2_level_fwd<4>(v);
    if (L >= 3) dwt2_level_fwd<2>(v);
}

template <int L>
__device__ __forceinline__ void dwt8_inv(int (&v)[8][8]) {
    if (L >= 3) dwt2_level_inv<2>(v);
    if (L >= 2) dwt2_level_inv<4>(v);
    dwt2_level_inv<8>(v);
}

// ------------------------------------------------------------------ records
template <int L>
struct Rec {
    static constexpr int ABITS = (L == 1) ? 160 : (L == 2) ? 40 : 10;
    static constexpr int BBITS = (L == 1) ? 0 : (L == 2) ? 124 : 155;
    static constexpr int CBITS = 480;
    static constexpr int AW = (ABITS + 31) / 32;
    static constexpr int BW = BBITS ? (BBITS + 31) / 32 : 1;
    static constexpr int CW = 15;
    static constexpr int ABYTES = (ABITS + 7) / 8;     // bytes(A_b) in the hash (C15)
    static constexpr int BBYTES = (BBITS + 7) / 8;
};

// OR a w-bit field u (already offset-binary, < 2^w) at MSB-first bit `pos`.
template <int NW>
__device__ __forceinline__ void put_field(uint32_t (&r)[NW], int pos, uint32_t u, int w) {
    const int word = pos >> 5, end = (pos & 31) + w;
    if (end <= 32) {
        r[word] |= u << (32 - end);
    } else {
        r[word] |= u >> (end - 32);
        r[word + 1] |= u << (64 - end);
    }
}

template <int NW>
__device__ __forceinline__ int get_field(const uint32_t (&r)[NW], int pos, int w) {
    const int word = pos >> 5, end = (pos & 31) + w;
    uint32_t u;
    if (end <= 32) u = r[word] >> (32 - end);
    else u = (r[word] << (end - 32)) | (r[word + 1] >> (64 - end));
    u &= (1u << w) - 1u;
    return (int)u - (1 << (w - 1));
}

// Visit every field of the three records in the canonical order (C10):
// A = LL_L; B = HL_l, LH_l, HH_l for l = L..2; C = HL1, LH1, HH1; row-major
// inside each band.  f(stream, pos, row, col, width).
template <int L, typename F>
__device__ __forceinline__ void for_each_field(F&& f) {
    constexpr int sL = 8 >> L;
    int pos = 0;
#pragma unroll
    for (int i = 0; i < sL; ++i)
#pragma unroll
        for (int j = 0; j < sL; ++j) { f(0, pos, i, j, 10); pos += 10; }
    pos = 0;
#pragma unroll
    for (int l = L; l >= 2; --l) {
        const int s = 8 >> l;
#pragma unroll
        for (int i = 0; i < s; ++i)
#pragma unroll
            for (int j = 0; j < s; ++j) { f(1, pos, i, s + j, 10); pos += 10; }   // HL
#pragma unroll
        for (int i = 0; i < s; ++i)
#pragma unroll
            for (int j = 0; j < s; ++j) { f(1, pos, s + i, j, 10); pos += 10; }   // LH
#pragma unroll
        for (int i = 0; i < s; ++i)
#pragma unroll
            for (int j = 0; j < s; ++j) { f(1, pos, s + i, s + j, 11); pos += 11; }  // HH
    }
    pos = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { f(2, pos, i, 4 + j, 10); pos += 10; }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { f(2, pos, 4 + i, j, 10); pos += 10; }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { f(2, pos, 4 + i, 4 + j, 10); pos += 10; }
}

// ------------------------------------------------------------------ SHA-2
__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    uint32_t nlo, nhi;
    if (n < 32) { nlo = __funnelshift_r(lo, hi, n); nhi = __funnelshift_r(hi, lo, n); }
    else { nlo = __funnelshift_r(hi, lo, n - 32); nhi = __funnelshift_r(lo, hi, n - 32); }
    return ((uint64_t)nhi << 32) | nlo;
}

// per-translation-unit copies (no relocatable device code needed)
static __constant__ uint32_t c_sha256_k[64] = SE_SHA256_K_INIT;
static __constant__ uint64_t c_sha512_k[80] = SE_SHA512_K_INIT;

// SHA-256 over one 64-byte block whose words W[0..7] were already consumed
// by the host midstate.  st = state after round 7; h0 = initial hash value.
// Returns the digest words in H.
__device__ __forceinline__ void sha256_from_round8(const uint32_t (&st)[8], const uint32_t (&h0)[8],
                                                   uint32_t (&W)[16], uint32_t (&H)[8]) {
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int t = 8; t < 64; ++t) {
        uint32_t w;
        if (t < 16) {
            w = W[t];
        } else {
            const uint32_t w2 = W[(t - 2) & 15], w15 = W[(t - 15) & 15];
            const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            w = s1 + W[(t - 7) & 15] + s0 + W[t & 15];
            W[t & 15] = w;
        }
        const uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = h + S1 + ch + c_sha256_k[t] + w;
        const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
    }
    H[0] = h0[0] + a; H[1] = h0[1] + b; H[2] = h0[2] + c; H[3] = h0[3] + d;
    H[4] = h0[4] + e; H[5] = h0[5] + f; H[6] = h0[6] + g; H[7] = h0[7] + h;
}

// SHA-512 resuming after round 3 (W[0..3] = K||IV consumed by the host).
__device__ __forceinline__ void sha512_from_round4(const uint64_t (&st)[8], const uint64_t (&h0)[8],
                                                   uint64_t (&W)[16], uint64_t (&H)[8]) {
    uint64_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int t = 4; t < 80; ++t) {
        uint64_t w;
        if (t < 16) {
            w = W[t];
        } else {
            const uint64_t w2 = W[(t - 2) & 15], w15 = W[(t - 15) & 15];
            const uint64_t s1 = rotr64(w2, 19) ^ rotr64(w2, 61) ^ (w2 >> 6);
            const uint64_t s0 = rotr64(w15, 1) ^ rotr64(w15, 8) ^ (w15 >> 7);
            w = s1 + W[(t - 7) & 15] + s0 + W[t & 15];
            W[t & 15] = w;
        }
        const uint64_t S1 = rotr64(e, 14) ^ rotr64(e, 18) ^ rotr64(e, 41);
        const uint64_t ch = (e & f) ^ (~e & g);
        const uint64_t t1 = h + S1 + ch + c_sha512_k[t] + w;
        const uint64_t S0 = rotr64(a, 28) ^ rotr64(a, 34) ^ rotr64(a, 39);
        const uint64_t mj = (a & b) ^ (a & c) ^ (b & c);
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
    }
    H[0] = h0[0] + a; H[1] = h0[1] + b; H[2] = h0[2] + c; H[3] = h0[3] + d;
    H[4] = h0[4] + e; H[5] = h0[5] + f; H[6] = h0[6] + g; H[7] = h0[7] + h;
}

// ------------------------------------------------------------------ AES
static __device__ const uint32_t g_aes_te0[256] = SE_AES_TE0_INIT;
static __device__ const uint8_t g_aes_sbox[256] = SE_AES_SBOX_INIT;

// Shared-memory T-tables: te[0..3][256] (Te1..3 = byte rotations of Te0) + S-box.
struct AesSmem {
    uint32_t te[4][256];
    uint32_t sb[256];
};

__device__ __forceinline__ void aes_load_tables(AesSmem& s, int tid, int nthreads) {
    for (int i = tid; i < 256; i += nthreads) {
        const uint32_t t = g_aes_te0[i];
        s.te[0][i] = t;
        s.te[1][i] = __funnelshift_r(t, t, 8);
        s.te[2][i] = __funnelshift_r(t, t, 16);
        s.te[3][i] = __funnelshift_r(t, t, 24);
        s.sb[i] = g_aes_sbox[i];
    }
}

// One AES-128 block, big-endian column words in/out; rk = 44 round-key words.
__device__ __forceinline__ void aes128_block(const AesSmem& s, const uint32_t* __restrict__ rk,
                                             uint32_t (&x)[4]) {
    uint32_t s0 = x[0] ^ rk[0], s1 = x[1] ^ rk[1], s2 = x[2] ^ rk[2], s3 = x[3] ^ rk[3];
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint32_t t0 = s.te[0][s0 >> 24] ^ s.te[1][(s1 >> 16) & 0xff] ^ s.te[2][(s2 >> 8) & 0xff] ^ s.te[3][s3 & 0xff] ^ rk[4 * r + 0];
        const uint32_t t1 = s.te[0][s1 >> 24] ^ s.te[1][(s2 >> 16) & 0xff] ^ s.te[2][(s3 >> 8) & 0xff] ^ s.te[3][s0 & 0xff] ^ rk[4 * r + 1];
        const uint32_t t2 = s.te[0][s2 >> 24] ^ s.te[1][(s3 >> 16) & 0xff] ^ s.te[2][(s0 >> 8) & 0xff] ^ s.te[3][s1 & 0xff] ^ rk[4 * r + 2];
        const uint32_t t3 = s.te[0][s3 >> 24] ^ s.te[1][(s0 >> 16) & 0xff] ^ s.te[2][(s1 >> 8) & 0xff] ^ s.te[3][s2 & 0xff] ^ rk[4 * r + 3];
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    x[0] = (s.sb[s0 >> 24] << 24) ^ (s.sb[(s1 >> 16) & 0xff] << 16) ^ (s.sb[(s2 >> 8) & 0xff] << 8) ^ s.sb[s3 & 0xff] ^ rk[40];
    x[1] = (s.sb[s1 >> 24] << 24) ^ (s.sb[(s2 >> 16) & 0xff] << 16) ^ (s.sb[(s3 >> 8) & 0xff] << 8) ^ s.sb[s0 & 0xff] ^ rk[41];
    x[2] = (s.sb[s2 >> 24] << 24) ^ (s.sb[(s3 >> 16) & 0xff] << 16) ^ (s.sb[(s0 >> 8) & 0xff] << 8) ^ s.sb[s1 & 0xff] ^ rk[42];
    x[3] = (s.sb[s3 >> 24] << 24) ^ (s.sb[(s0 >> 16) & 0xff] << 16) ^ (s.sb[(s1 >> 8) & 0xff] << 8) ^ s.sb[s2 & 0xff] ^ rk[43];
}

// 128-bit big-endian counter + 64-bit increment.
__device__ __forceinline__ void ctr_add(const uint32_t (&base)[4], uint64_t j, uint32_t (&out)[4]) {
    uint64_t lo = ((uint64_t)base[2] << 32 | base[3]);
    uint64_t hi = ((uint64_t)base[0] << 32 | base[1]);
    const uint64_t nlo = lo + j;
    hi += (nlo < lo) ? 1u : 0u;
    out[0] = (uint32_t)(hi >> 32); out[1] = (uint32_t)hi;
    out[2] = (uint32_t)(nlo >> 32); out[3] = (uint32_t)nlo;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Mask keeping the first `bits` (MSB-first) of a word; 0 means the whole word.
__host__ __device__ constexpr uint32_t head_mask(int bits) {
    return bits == 0 ? 0xffffffffu : (0xffffffffu << ((32 - bits) & 31));
}

}  // namespace se
