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
#include "sha2_device.cuh"
#include "tables.h"

namespace se {

// ------------------------------------------------------------------ FMA-pipe integer ops
// `one` is a kernel parameter equal to 1 that ptxas cannot fold, so these stay
// IMADs and issue on the FMA pipe, leaving the ALU pipe (the path's limit:
// SHF/LOP3 of SHA-2) free.  See sha2_device.cuh and DESIGN.md §5.
__device__ __forceinline__ int iadd(int a, int b, uint32_t one) {
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}
__device__ __forceinline__ int isub(int a, int b, int m1) {       // a - b, m1 = -1 (opaque)
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(m1), "r"(a));
    return r;
}

// floor(v / 4) + c.  QHI: one IMAD.HI (v * 2^30 >> 32, signed) on the FMA
// pipe instead of LEA.HI on the ALU pipe (q30 = one << 30, opaque so ptxas
// keeps the multiply).  Round 1 measured it slower in both directions (C2
// masked protect / recover 182.7 / 183.9 vs 184.7 / 187.5 GB/s) with the
// SHA sigma shifts also on the FMA pipe; round 2, with those shifts back on
// the ALU pipe (SE_SHR_FMA 0), it helps the inverse and still hurts the
// forward transform (C4 recover 4.726 -> 4.664 ms, protect 4.676 -> 4.755):
// SE_LIFT_QHI_INV 1, SE_LIFT_QHI_FWD 0.
#ifndef SE_LIFT_QHI_FWD
#define SE_LIFT_QHI_FWD 0
#endif
#ifndef SE_LIFT_QHI_INV
#define SE_LIFT_QHI_INV 1
#endif
#ifndef SE_LIFT_LEA
#define SE_LIFT_LEA 2      // measured (C2 masked p / r GB/s): 0 182.7 / 187.2, 1 185.1 / 187.1, 2 185.1 / 188.7
#endif
template <bool QHI>
__device__ __forceinline__ int qfloor4(int v, int c, int q30) {
    if constexpr (QHI) {
        int r;
        asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(q30), "r"(c));
        return r;
    } else {
        (void)q30;
        return (v >> 2) + c;              // ptxas: one LEA.HI (shift and add) on the ALU pipe
    }
}

// a + (b >> 1): SE_LIFT_LEA >= 2 lets ptxas fuse it into one LEA.HI (ALU)
// instead of SHF (ALU) + IMAD (FMA)
__device__ __forceinline__ int add_half(int a, int b, uint32_t one) {
#if SE_LIFT_LEA >= 2
    (void)one;
    return a + (b >> 1);
#else
    return iadd(a, b >> 1, one);
#endif
}

// ------------------------------------------------------------------ lifting
// Forward 1-D lifting of n samples in place: output [s(0..n/2) | d(0..n/2)].
// Samples are NOT centered: lifting commutes exactly with adding a constant
// c to every sample (predict cancels it, update passes it through: both
// floors see an integer shift), so centering (C8) only moves the final LL
// band by -128 and is folded into the A-field offset (records) or applied to
// LL alone (dwt_fwd).
template <int N>
__device__ __forceinline__ void lift_fwd(int (&x)[N], uint32_t one, int m1) {
    constexpr int H = N / 2;
    int s[H], d[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
        if (2 * k + 2 < N) d[k] = isub(x[2 * k + 1], iadd(x[2 * k], x[2 * k + 2], one) >> 1, m1);   // Eq. 5.1
        else d[k] = isub(x[2 * k + 1], x[2 * k], m1);                 // x(N) = x(N-2)
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int dm1 = (k == 0) ? d[0] : d[k - 1];                   // d(-1) = d(0)
#if SE_LIFT_LEA || SE_LIFT_QHI_FWD
        s[k] = qfloor4<SE_LIFT_QHI_FWD != 0>(iadd(iadd(dm1, d[k], one), 2, one), x[2 * k], (int)(one << 30));   // Eq. 5.2 (+)
#else
        s[k] = iadd(x[2 * k], iadd(iadd(dm1, d[k], one), 2, one) >> 2, one);              // Eq. 5.2 (+)
#endif
    }
#pragma unroll
    for (int k = 0; k < H; ++k) { x[k] = s[k]; x[H + k] = d[k]; }
}

// Exact inverse: undo the update, then undo the predict.
template <int N>
__device__ __forceinline__ void lift_inv(int (&y)[N], uint32_t one, int m1) {
    constexpr int H = N / 2;
    int x[N];
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int dm1 = (k == 0) ? y[H] : y[H + k - 1];
        x[2 * k] = isub(y[k], qfloor4<SE_LIFT_QHI_INV != 0>(iadd(iadd(dm1, y[H + k], one), 2, one), 0, (int)(one << 30)), m1);
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        if (2 * k + 2 < N) x[2 * k + 1] = add_half(y[H + k], iadd(x[2 * k], x[2 * k + 2], one), one);
        else x[2 * k + 1] = iadd(y[H + k], x[2 * k], one);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) y[k] = x[k];
}

// One 2-D level on the top-left M x M region: rows, then columns (C5).
template <int M>
__device__ __forceinline__ void dwt2_level_fwd(int (&v)[8][8], uint32_t one, int m1) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int t[M];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = v[i][j];
        lift_fwd<M>(t, one, m1);
#pragma unroll
        for (int j = 0; j < M; ++j) v[i][j] = t[j];
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        int t[M];
#pragma unroll
        for (int i = 0; i < M; ++i) t[i] = v[i][j];
        lift_fwd<M>(t, one, m1);
#pragma unroll
        for (int i = 0; i < M; ++i) v[i][j] = t[i];
    }
}

template <int M>
__device__ __forceinline__ void dwt2_level_inv(int (&v)[8][8], uint32_t one, int m1) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
        int t[M];
#pragma unroll
        for (int i = 0; i < M; ++i) t[i] = v[i][j];
        lift_inv<M>(t, one, m1);
#pragma unroll
        for (int i = 0; i < M; ++i) v[i][j] = t[i];
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int t[M];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = v[i][j];
        lift_inv<M>(t, one, m1);
#pragma unroll
        for (int j = 0; j < M; ++j) v[i][j] = t[j];
    }
}

template <int L>
__device__ __forceinline__ void dwt8_fwd(int (&v)[8][8], uint32_t one) {
    const int m1 = -(int)one;
    dwt2_level_fwd<8>(v, one, m1);
    if (L >= 2) dwt2_level_fwd<4>(v, one, m1);
    if (L >= 3) dwt2_level_fwd<2>(v, one, m1);
}

template <int L>
__device__ __forceinline__ void dwt8_inv(int (&v)[8][8], uint32_t one) {
    const int m1 = -(int)one;
    if (L >= 3) dwt2_level_inv<2>(v, one, m1);
    if (L >= 2) dwt2_level_inv<4>(v, one, m1);
    dwt2_level_inv<8>(v, one, m1);
}

// ------------------------------------------------------------------ lean lifting
// The same transform written for issue-bound kernels (PUBLIC_PLAIN tile
// kernels, k_tile.cu): plain integer adds, so ptxas fuses the three-operand
// sums into IADD3 and each shift-and-add into one LEA.HI.
//   predict  x_o - floor((x_l + x_r) / 2) = x_o + floor((1 - x_l - x_r) / 2)
//   update   x_e + floor((d_l + d_r + 2) / 4)
//   inverse  x_e = s + floor((1 - d_l - d_r) / 4)   (= s - floor((d_l + d_r + 2) / 4))
//            x_o = d + floor((x_l + x_r) / 2)
// (floor via the arithmetic shift; -floor(m / 2^k) = floor((2^k - 1 - m) / 2^k)).
template <int N>
__device__ __forceinline__ void lift_fwd_lean(int (&x)[N]) {
    constexpr int H = N / 2;
    int s[H], d[H];
#pragma unroll
    for (int k = 0; k < H; ++k)
        d[k] = (2 * k + 2 < N) ? x[2 * k + 1] + ((1 - x[2 * k] - x[2 * k + 2]) >> 1) : x[2 * k + 1] - x[2 * k];
#pragma unroll
    for (int k = 0; k < H; ++k) s[k] = x[2 * k] + (((k == 0 ? d[0] : d[k - 1]) + d[k] + 2) >> 2);
#pragma unroll
    for (int k = 0; k < H; ++k) { x[k] = s[k]; x[H + k] = d[k]; }
}

#ifndef SE_INV_PRED_FMA
#define SE_INV_PRED_FMA 1
#endif
template <int N>
__device__ __forceinline__ void lift_inv_lean(int (&y)[N], uint32_t one) {
    constexpr int H = N / 2;
    int x[N];
#pragma unroll
    for (int k = 0; k < H; ++k) x[2 * k] = y[k] + ((1 - (k == 0 ? y[H] : y[H + k - 1]) - y[H + k]) >> 2);
#pragma unroll
    for (int k = 0; k < H; ++k) {
        if (2 * k + 2 < N) {
#if SE_INV_PRED_FMA
            // the two-operand sum as an IMAD (FMA pipe; recovery's ALU pipe is the busier)
            x[2 * k + 1] = y[H + k] + (iadd(x[2 * k], x[2 * k + 2], one) >> 1);
#else
            x[2 * k + 1] = y[H + k] + ((x[2 * k] + x[2 * k + 2]) >> 1);
#endif
        } else {
            x[2 * k + 1] = y[H + k] + x[2 * k];
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) y[k] = x[k];
}

// Mixed-pipe lean lifting (SE_LEAN_MIX bit 0: forward, bit 1: inverse): the
// sums move to the FMA pipe as IMADs by an opaque +-1 and each lift keeps one
// ALU op, the shift-and-add (LEA.HI).  Forward:
//   u   = 3 - x_l - x_r                (one IADD3; or, SE_MIX_FWD_PRED_LEAN 0, IMAD(x_l, -1, n_r)
//                                       with n_e = 3 - x_e by one IMAD per even sample)
//   d'  = x_o + (u >> 1) = d + 1       (LEA.HI; floor((3 - m) / 2) = 1 + floor((1 - m) / 2) = 1 - floor(m / 2))
//   s   = x_e + ((d'_l + d'_r) >> 2)   (IMAD + LEA.HI; d'_l + d'_r = d_l + d_r + 2)
// so every high-pass output carries +1 (d' = d + 1).  Lifting passes a
// constant offset of its inputs through the update and cancels it in the
// predict, so after dwt8_fwd_mix every band but the final LL holds v + 1
// (the caller folds the -1 into its field offsets); LL is exact.
// Inverse (exact values in and out):
//   m_d = 1 - d                        (IMAD; each d serves two updates)
//   x_e = s + ((1 - d_l - d_r) >> 2)   (IMAD(d_l, -1, m_r) + LEA.HI)
//   x_o = d + ((x_l + x_r) >> 1)       (IMAD + LEA.HI)
// Measured (C4 PUBLIC_PLAIN tile kernels, tools/gpu_r2_call37.sh): lean
// protect / recover 0.669 / 0.689 ms, mixed 0.627 / 0.653 ms (791 -> 839 GB/s
// round trip): SE_LEAN_MIX 3.
#ifndef SE_LEAN_MIX
#define SE_LEAN_MIX 3
#endif
__device__ __forceinline__ int imad(int a, int b, int c) {      // a * b + c on the FMA pipe (b opaque)
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// SE_MIX_FWD_PRED_LEAN 1: the forward predict as IADD3 + LEA.HI (two ALU ops,
// no n_e), the update mixed - fewer instructions, more ALU-pipe work.
// Measured (tools/gpu_r2_call51.sh, two passes): C4 PUBLIC_PLAIN protect
// 0.6259 -> 0.6237 ms, masked protect 4.659 -> 4.651 ms: 1.
#ifndef SE_MIX_FWD_PRED_LEAN
#define SE_MIX_FWD_PRED_LEAN 1
#endif
template <int N, bool PL = SE_MIX_FWD_PRED_LEAN != 0>
__device__ __forceinline__ void lift_fwd_mix(int (&x)[N], int m1) {
    constexpr int H = N / 2;
    int s[H], d[H];
    int n[H] = {};
    if constexpr (!PL) {
#pragma unroll
        for (int k = 1; k < H; ++k) n[k] = imad(x[2 * k], m1, 3);                // 3 - x_e (n[0] unused)
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        if (2 * k + 2 < N)
            d[k] = PL ? x[2 * k + 1] + ((3 - x[2 * k] - x[2 * k + 2]) >> 1)      // Eq. 5.1, +1
                      : x[2 * k + 1] + (imad(x[2 * k], m1, n[k + 1]) >> 1);
        else d[k] = x[2 * k + 1] - x[2 * k] + 1;                                 // x(N) = x(N-2), +1
    }
#pragma unroll
    for (int k = 0; k < H; ++k)                                                  // Eq. 5.2
        s[k] = k == 0 ? x[0] + (d[0] >> 1)                   // d(-1) = d(0): (2 d'_0) >> 2 = d'_0 >> 1, one LEA.HI
                      : x[2 * k] + (imad(d[k - 1], -m1, d[k]) >> 2);
#pragma unroll
    for (int k = 0; k < H; ++k) { x[k] = s[k]; x[H + k] = d[k]; }
}

template <int N>
__device__ __forceinline__ void lift_inv_mix(int (&y)[N], int m1) {
    constexpr int H = N / 2;
    int x[N], m[H] = {};
#pragma unroll
    for (int k = 1; k < H; ++k) m[k] = imad(y[H + k], m1, 1);                   // 1 - d (m[0] unused)
    // k = 0 (d(-1) = d(0)): floor((1 - 2 d) / 4) = floor(-d / 2), one IMAD (-d) and one LEA.HI
    x[0] = y[0] + (imad(y[H], m1, 0) >> 1);
#pragma unroll
    for (int k = 1; k < H; ++k) x[2 * k] = y[k] + (imad(y[H + k - 1], m1, m[k]) >> 2);
#pragma unroll
    for (int k = 0; k < H; ++k) {
        if (2 * k + 2 < N) x[2 * k + 1] = y[H + k] + (imad(x[2 * k], -m1, x[2 * k + 2]) >> 1);
        else x[2 * k + 1] = imad(x[2 * k], -m1, y[H + k]);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) y[k] = x[k];
}

template <int M, bool INV, int MIX = SE_LEAN_MIX>
__device__ __forceinline__ void dwt2_level_lean(int (&v)[8][8], uint32_t one) {
    // forward: rows then columns (C5); inverse: columns then rows
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
        const bool rows = (pass == 0) != INV;
#pragma unroll
        for (int a = 0; a < M; ++a) {
            int t[M];
#pragma unroll
            for (int b = 0; b < M; ++b) t[b] = rows ? v[a][b] : v[b][a];
            if (INV) {
                if constexpr ((MIX & 2) != 0) lift_inv_mix<M>(t, -(int)one);
                else lift_inv_lean<M>(t, one);
            } else {
                if constexpr ((MIX & 1) != 0) lift_fwd_mix<M, (MIX & 4) ? false : (SE_MIX_FWD_PRED_LEAN != 0)>(t, -(int)one);
                else lift_fwd_lean<M>(t);
            }
#pragma unroll
            for (int b = 0; b < M; ++b) {
                if (rows) v[a][b] = t[b];
                else v[b][a] = t[b];
            }
        }
    }
}

template <int L>
__device__ __forceinline__ void dwt8_fwd_lean(int (&v)[8][8], uint32_t one) {
    dwt2_level_lean<8, false>(v, one);
    if (L >= 2) dwt2_level_lean<4, false>(v, one);
    if (L >= 3) dwt2_level_lean<2, false>(v, one);
}

template <int L>
__device__ __forceinline__ void dwt8_inv_lean(int (&v)[8][8], uint32_t one) {
    if (L >= 3) dwt2_level_lean<2, true>(v, one);
    if (L >= 2) dwt2_level_lean<4, true>(v, one);
    dwt2_level_lean<8, true>(v, one);
}

// The mixed-pipe lifting on its own (the masked kernels, SE_MASK_MIX): the
// forward leaves +1 on every band but LL (see lift_fwd_mix).
// SE_MASK_PRED_IMAD 1: the masked kernels' forward predicts with IMAD sums
// (n_e = 3 - x_e precomputed) instead of IADD3 - ~80 fewer ALU-pipe ops per
// block, but measured equal (C4 protect 4.609 vs 4.611 ms, three passes,
// tools/gpu_r2_call62.sh), so 0.
#ifndef SE_MASK_PRED_IMAD
#define SE_MASK_PRED_IMAD 0
#endif
template <int L>
__device__ __forceinline__ void dwt8_fwd_mix(int (&v)[8][8], uint32_t one) {
    constexpr int MX = SE_MASK_PRED_IMAD ? 7 : 3;        // 7: the predicts' sums as IMADs too
    dwt2_level_lean<8, false, MX>(v, one);
    if (L >= 2) dwt2_level_lean<4, false, MX>(v, one);
    if (L >= 3) dwt2_level_lean<2, false, MX>(v, one);
}

template <int L>
__device__ __forceinline__ void dwt8_inv_mix(int (&v)[8][8], uint32_t one) {
    if (L >= 3) dwt2_level_lean<2, true, 3>(v, one);
    if (L >= 2) dwt2_level_lean<4, true, 3>(v, one);
    dwt2_level_lean<8, true, 3>(v, one);
}

// Any of 64 reconstructed samples outside [0, 255]?  Pairs as v_a + 2^16 v_b
// (IMAD, FMA pipe): for |v| < 2^15 (every sample the inverse can produce from
// <= 11-bit fields at L <= 3) the word has a bit of 0xff00ff00 set iff v_a or
// v_b is outside [0, 255] (a negative v_a sets bit 15), so half the ORs.
__device__ __forceinline__ bool out_of_range_pairs(const int (&v)[8][8], uint32_t one) {
    int orv = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2) orv |= imad(v[i][j + 1], (int)(one << 16), v[i][j]);
    return (orv & 0xff00ff00) != 0;
}

// ------------------------------------------------------------------ records
template <int L, int MODE = 0>
struct Rec {
    static constexpr int ABITS = (L == 1) ? 160 : (L == 2) ? 40 : 10;
    static constexpr int BBITS = (L == 1) ? 0 : (L == 2) ? (MODE ? 132 : 124) : (MODE ? 165 : 155);
    static constexpr int CBITS = 480;
    static constexpr int AW = (ABITS + 31) / 32;
    static constexpr int BW = BBITS ? (BBITS + 31) / 32 : 1;
    static constexpr int CW = 15;
    static constexpr int ABYTES = (ABITS + 7) / 8;     // bytes(A_b) in the hash (C15)
    static constexpr int BBYTES = (BBITS + 7) / 8;
};

// Place value v as a w-bit offset-binary field u = v + off (C9) at MSB-first
// bit `pos`.  Fields never overlap, so OR == ADD and a field inside one word
// is one multiply-add by an (opaque) power of two on the FMA pipe; a field
// straddling two words costs one shift on the ALU pipe.
template <int NW>
__device__ __forceinline__ void put_field(uint32_t (&r)[NW], int pos, int v, int off, int w, uint32_t one) {
    const int word = pos >> 5, end = (pos & 31) + w;
    const uint32_t u = (uint32_t)iadd(v, off, one);
    if (end <= 32) {
        uint32_t t;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(u), "r"(one << (32 - end)), "r"(r[word]));
        r[word] = t;
    } else {
        r[word] |= u >> (end - 32);
        uint32_t t;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(u), "r"(one << (64 - end)), "r"(r[word + 1]));
        r[word + 1] = t;
    }
}

// Inverse: v = field - off.  A field at the top of its word is one IMAD.HI
// (r * 2^w) >> 32 with the -off folded in as the addend; elsewhere the
// field is isolated with one LOP3 and shifted down by IMAD.HI.
template <int NW>
__device__ __forceinline__ int get_field(const uint32_t (&r)[NW], int pos, int off, int w, uint32_t one) {
    const int word = pos >> 5, start = pos & 31, end = start + w;
    int v;
    if (end <= 32) {
        const uint32_t masked = (start == 0) ? r[word] : (r[word] & (0xffffffffu >> start));
        if (end == 32) {
            v = isub((int)masked, off, -(int)one);
        } else {
            asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(masked), "r"(one << end), "r"(-off));
        }
    } else {
        const uint32_t u = ((r[word] << (end - 32)) | (r[word + 1] >> (64 - end))) & ((1u << w) - 1u);
        v = isub((int)u, off, -(int)one);
    }
    return v;
}

// Lean field placement (issue-bound kernels): v + off placed with one
// shift-add per field; the additions of constants chain and fold.
#ifndef SE_PACK_FMA
#define SE_PACK_FMA 0
#endif
template <int NW>
__device__ __forceinline__ void put_field_lean(uint32_t (&r)[NW], int pos, int v, int off, int w, uint32_t one) {
    const int word = pos >> 5, end = (pos & 31) + w;
    const uint32_t u = (uint32_t)(v + off);
    if (end <= 32) {
#if SE_PACK_FMA
        // u << k as an IMAD by an opaque power of two (FMA pipe); v * 2^k + (r + off * 2^k)
        uint32_t t;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(u), "r"(one << (32 - end)), "r"(r[word]));
        r[word] = t;
#else
        (void)one;
        r[word] += u << (32 - end);
#endif
    } else {
        r[word] += u >> (end - 32);
        r[word + 1] += u << (64 - end);
    }
}

// Lean field extraction: the caller has XORed every field's top bit in place
// (flip_top), so each field is the sign-extended w-bit value v = u - 2^(w-1)
// (offset binary, C9): one or two shifts.
#ifndef SE_EXTRACT_FMA
#define SE_EXTRACT_FMA 1
#endif
// SE_EXTRACT_HI 1: the sign-extending right shift as IMAD.HI.  Measured
// (tools/gpu_r2_call53.sh): C4 PUBLIC_PLAIN recover 0.637 -> 0.730 ms, so 0.
#ifndef SE_EXTRACT_HI
#define SE_EXTRACT_HI 0
#endif
template <int NW>
__device__ __forceinline__ int get_field_lean(const uint32_t (&r)[NW], int pos, int w, uint32_t one) {
    const int word = pos >> 5, start = pos & 31, end = start + w;
    uint32_t top;
    if (end <= 32) {
#if SE_EXTRACT_FMA
        // the left shift as an IMAD by an opaque power of two: the recovery
        // kernel's ALU pipe is the busier one (~83 %)
        if (start) asm("mul.lo.u32 %0, %1, %2;" : "=r"(top) : "r"(r[word]), "r"(one << start));
        else top = r[word];
#else
        (void)one;
        top = r[word] << start;
#endif
    } else {
        top = __funnelshift_l(r[word + 1], r[word], start);
    }
#if SE_EXTRACT_HI
    // the sign-extending right shift as IMAD.HI: (top * 2^w) >> 32 (FMA pipe)
    int v;
    asm("mul.hi.s32 %0, %1, %2;" : "=r"(v) : "r"(top), "r"(one << w));
    return v;
#else
    return (int)top >> (32 - w);
#endif
}

template <int NW>
__device__ __forceinline__ void flip_top(uint32_t (&r)[NW], int pos) {
    r[pos >> 5] ^= 0x80000000u >> (pos & 31);
}

// Visit every field of the three records in the canonical order (C10):
// A = LL_L; B = HL_l, LH_l, HH_l for l = L..2; C = HL1, LH1, HH1; row-major
// inside each band.  f(stream, pos, row, col, width) with (row, col) in the
// 8x8 dyadic block layout.  Widths (C22/C23): BLOCK8 HH_l (l >= 2) 11 bits,
// all else 10; FULL mode every B field 11 bits.
template <int L, int MODE = 0, typename F>
__device__ __forceinline__ void for_each_field(F&& f) {
    constexpr int sL = 8 >> L;
    constexpr int wb = MODE ? 11 : 10;
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
            for (int j = 0; j < s; ++j) { f(1, pos, i, s + j, wb); pos += wb; }   // HL
#pragma unroll
        for (int i = 0; i < s; ++i)
#pragma unroll
            for (int j = 0; j < s; ++j) { f(1, pos, s + i, j, wb); pos += wb; }   // LH
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

// ------------------------------------------------------------------ AES
static __device__ const uint32_t g_aes_te0[256] = SE_AES_TE0_INIT;

// Lane-replicated T-table in shared memory (64 KB, dynamic): row x is 256
// bytes — words 0..31 hold Te0[x] once per lane, words 32..63 Te2[x] =
// ror16(Te0[x]).  Lane l reads word l (or 32 + l) of whatever row its byte
// selects, so the 32 lanes of a warp always hit 32 distinct banks: one
// shared-memory wavefront per lookup instead of ~3.5 for random indices into
// a single table.  The row address (byte << 8 | lane column) is one PRMT.
// Te1 = ror8(Te0) and Te3 = ror8(Te2), and rotation distributes over XOR, so
// each output column needs a single rotation.  The S-box of the last round
// is byte 2 of Te0[x] = (2s, s, s, 3s).
constexpr int kAesLutBytes = 256 * 256;

__device__ __forceinline__ void aes_load_lut(uint32_t* lut, int tid, int nthreads) {
    uint4* l4 = reinterpret_cast<uint4*>(lut);
    for (int i = tid; i < 256 * 16; i += nthreads) {              // 16 x 16 B per row
        const uint32_t t = g_aes_te0[i >> 4];
        const uint32_t v = (i & 15) < 8 ? t : __funnelshift_r(t, t, 16);
        l4[i] = make_uint4(v, v, v, v);
    }
}

struct AesLane {
    const uint8_t* lut;   // shared-memory base of the table
    uint32_t c0, c2;      // this lane's byte column in the Te0 / Te2 halves
};

__device__ __forceinline__ AesLane aes_lane(const uint32_t* lut) {
    const uint32_t lane = threadIdx.x & 31;
    return AesLane{reinterpret_cast<const uint8_t*>(lut), lane * 4, 128 + lane * 4};
}

// table word for byte K of s (K = 3: most significant), column c
template <int K>
__device__ __forceinline__ uint32_t aes_lu(const AesLane& a, uint32_t s, uint32_t c) {
    const uint32_t addr = __byte_perm(s, c, 0x5504 | (K << 4));     // (byte K << 8) | c
    return *reinterpret_cast<const uint32_t*>(a.lut + addr);
}

// one output column of a middle round:
// Te0[sa.b3] ^ Te1[sb.b2] ^ Te2[sc.b1] ^ Te3[sd.b0] ^ k = Te0 ^ Te2 ^ ror8(Te0 ^ Te2) ^ k
__device__ __forceinline__ uint32_t aes_col(const AesLane& a, uint32_t sa, uint32_t sb, uint32_t sc, uint32_t sd,
                                            uint32_t k) {
    const uint32_t v = aes_lu<2>(a, sb, a.c0) ^ aes_lu<0>(a, sd, a.c2);
    return aes_lu<3>(a, sa, a.c0) ^ aes_lu<1>(a, sc, a.c2) ^ k ^ __funnelshift_r(v, v, 8);
}

// One AES-128 block (FIPS-197 §5.1), big-endian column words in/out; rk = 44
// round-key words.
__device__ __forceinline__ void aes128_block(const AesLane& a, const uint32_t* __restrict__ rk, uint32_t (&x)[4]) {
    uint32_t s0 = x[0] ^ rk[0], s1 = x[1] ^ rk[1], s2 = x[2] ^ rk[2], s3 = x[3] ^ rk[3];
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint32_t t0 = aes_col(a, s0, s1, s2, s3, rk[4 * r + 0]);
        const uint32_t t1 = aes_col(a, s1, s2, s3, s0, rk[4 * r + 1]);
        const uint32_t t2 = aes_col(a, s2, s3, s0, s1, rk[4 * r + 2]);
        const uint32_t t3 = aes_col(a, s3, s0, s1, s2, rk[4 * r + 3]);
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    // last round: SubBytes + ShiftRows + AddRoundKey; S[x] = byte 2 of Te0[x]
    const uint32_t s[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t hi = __byte_perm(aes_lu<3>(a, s[j], a.c0), aes_lu<2>(a, s[(j + 1) & 3], a.c0), 0x2600);
        const uint32_t lo = __byte_perm(aes_lu<1>(a, s[(j + 2) & 3], a.c0), aes_lu<0>(a, s[(j + 3) & 3], a.c0), 0x0026);
        x[j] = __byte_perm(lo, hi, 0x7610) ^ rk[40 + j];
    }
}

// The same table with its rotations stored too (128 KB: the first 64 KB as
// above, the second holding Te1[x] = ror8(Te0[x]) and Te3[x] = ror8(Te2[x])
// in the same row / lane positions, read at +64 KB by the same PRMT-built
// address): a middle-round column is 4 PRMT + 4 LDS + 2 LOP3 instead of
// 4 PRMT + 4 LDS + 3 LOP3 + 1 SHF.  Only the standalone cipher / keystream
// kernels use it (one CTA per SM).
constexpr int kAesLut4Bytes = 2 * kAesLutBytes;

__device__ __forceinline__ void aes_load_lut4(uint32_t* lut, int tid, int nthreads) {
    uint4* l4 = reinterpret_cast<uint4*>(lut);
    for (int i = tid; i < 2 * 256 * 16; i += nthreads) {          // two halves of 16 x 16 B per row
        const int h = i >> 12, j = i & 4095;
        const uint32_t t = g_aes_te0[j >> 4];
        uint32_t v = (j & 15) < 8 ? t : __funnelshift_r(t, t, 16);
        if (h) v = __funnelshift_r(v, v, 8);
        l4[i] = make_uint4(v, v, v, v);
    }
}

__device__ __forceinline__ uint32_t aes_col4(const AesLane& a, uint32_t sa, uint32_t sb, uint32_t sc, uint32_t sd,
                                             uint32_t k) {
    const uint32_t hi = aes_lu<3>(a, sa, a.c0) ^ aes_lu<1>(a, sc, a.c2) ^ k;
    const uint32_t t1 = *reinterpret_cast<const uint32_t*>(a.lut + kAesLutBytes + __byte_perm(sb, a.c0, 0x5524));
    const uint32_t t3 = *reinterpret_cast<const uint32_t*>(a.lut + kAesLutBytes + __byte_perm(sd, a.c2, 0x5504));
    return hi ^ t1 ^ t3;
}

__device__ __forceinline__ void aes128_block4(const AesLane& a, const uint32_t* __restrict__ rk, uint32_t (&x)[4]) {
    uint32_t s0 = x[0] ^ rk[0], s1 = x[1] ^ rk[1], s2 = x[2] ^ rk[2], s3 = x[3] ^ rk[3];
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint32_t t0 = aes_col4(a, s0, s1, s2, s3, rk[4 * r + 0]);
        const uint32_t t1 = aes_col4(a, s1, s2, s3, s0, rk[4 * r + 1]);
        const uint32_t t2 = aes_col4(a, s2, s3, s0, s1, rk[4 * r + 2]);
        const uint32_t t3 = aes_col4(a, s3, s0, s1, s2, rk[4 * r + 3]);
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint32_t s[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t hi = __byte_perm(aes_lu<3>(a, s[j], a.c0), aes_lu<2>(a, s[(j + 1) & 3], a.c0), 0x2600);
        const uint32_t lo = __byte_perm(aes_lu<1>(a, s[(j + 2) & 3], a.c0), aes_lu<0>(a, s[(j + 3) & 3], a.c0), 0x0026);
        x[j] = __byte_perm(lo, hi, 0x7610) ^ rk[40 + j];
    }
}

// Small T-tables (5 KB): te[0..3][256] (Te1..3 = byte rotations of Te0) + the
// S-box.  Random indices conflict in the shared-memory banks (~3.5 wavefronts
// per lookup), but the footprint is small: used for the keystream kernels
// that run concurrently with a fused kernel (programmatic launch), where the
// 64 KB lane table below measured 2.6 % slower on C2 protect.
static __device__ const uint8_t g_aes_sbox[256] = SE_AES_SBOX_INIT;

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

__device__ __forceinline__ void aes128_block(const AesSmem& s, const uint32_t* __restrict__ rk, uint32_t (&x)[4]) {
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
