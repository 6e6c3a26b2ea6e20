// sha2_device.cuh — SHA-256 / SHA-512 compression for the B and C masks
// (FIPS 180-4 §6.2.2 / §6.4.2), tuned for sm_100a integer pipes.
//
// The masks are ~85% of the path's instructions.  On
// sm_100 the shift / rotate / logic ops (SHF, LOP3, PRMT) issue only on the
// ALU pipe (16 lanes/clk/SMSP), while IMAD-class ops issue on the FMA pipe at
// the same rate.  Written naively, every add also lands on the ALU pipe
// (IADD3), so the ALU pipe is the bottleneck while the FMA pipe idles.  Here
// the adds are written as multiply-adds by an opaque 1 (a kernel parameter
// ptxas cannot fold): a 32-bit add is one IMAD, a 64-bit add is IMAD.WIDE.U32
// + IMAD, both on the FMA pipe — the ALU pipe keeps only the rotations and
// Boolean functions.
//
// Rounds run in a loop of 16-round unrolled bodies (message schedule in a
// 16-word register window, state roles rotated by index arithmetic), which
// keeps the hot code ~12 KB instead of ~100 KB fully unrolled: the fully
// unrolled kernel lost a third of its issue slots to instruction-fetch stalls.
#pragma once
#include <stdint.h>

#include "tables.h"

namespace se {

static __constant__ uint32_t c_sha256_k[64] = SE_SHA256_K_INIT;
static __constant__ uint64_t c_sha512_k[80] = SE_SHA512_K_INIT;

// ---------------------------------------------------------------- adds on the FMA pipe
__device__ __forceinline__ uint32_t fadd(uint32_t a, uint32_t b, uint32_t one) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}

struct W64 {
    uint32_t lo, hi;
};

__device__ __forceinline__ W64 w64(uint64_t v) { return W64{(uint32_t)v, (uint32_t)(v >> 32)}; }
__device__ __forceinline__ uint64_t u64(W64 v) { return (uint64_t)v.hi << 32 | v.lo; }

#ifndef SE_SHA512_ADD
#define SE_SHA512_ADD 2
#endif
// a + b (mod 2^64).
//   0: plain 64-bit add (ptxas: IADD3 + IADD3.X / IMAD.X)
//   1: IMAD.WIDE.U32 (a.lo * 1 + b) + IMAD: no ALU slot, but IMAD.WIDE takes
//      two FMA-pipe issue slots (measured, tools/intbench.cu)
//   2: add.cc on the low word (IADD3, ALU) + madc on the high word (IMAD.X,
//      FMA): one slot on each pipe
__device__ __forceinline__ W64 fadd64(W64 a, W64 b, uint32_t one) {
#if SE_SHA512_ADD == 1
    uint64_t t;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(a.lo), "r"(one), "l"(u64(b)));
    return W64{(uint32_t)t, fadd(a.hi, (uint32_t)(t >> 32), one)};
#elif SE_SHA512_ADD == 2
    W64 r;
    asm("add.cc.u32 %0, %2, %3;\n\tmadc.lo.u32 %1, %4, %5, %6;"
        : "=r"(r.lo), "=r"(r.hi) : "r"(a.lo), "r"(b.lo), "r"(a.hi), "r"(one), "r"(b.hi));
    return r;
#else
    (void)one;
    return w64(u64(a) + u64(b));
#endif
}

#ifndef SE_SHA512_SCHED_ADD
#define SE_SHA512_SCHED_ADD SE_SHA512_ADD
#endif
// the message-schedule adds, selectable separately (pipe balance tuning)
__device__ __forceinline__ W64 fadd64s(W64 a, W64 b, uint32_t one) {
#if SE_SHA512_SCHED_ADD == 1
    uint64_t t;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(a.lo), "r"(one), "l"(u64(b)));
    return W64{(uint32_t)t, fadd(a.hi, (uint32_t)(t >> 32), one)};
#else
    return fadd64(a, b, one);
#endif
}

__device__ __forceinline__ W64 xor3(W64 a, W64 b, W64 c) { return W64{a.lo ^ b.lo ^ c.lo, a.hi ^ b.hi ^ c.hi}; }

template <int N>
__device__ __forceinline__ W64 ror64(W64 v) {
    if constexpr (N < 32) return W64{__funnelshift_r(v.lo, v.hi, N), __funnelshift_r(v.hi, v.lo, N)};
    else
    return W64{__funnelshift_r(v.hi, v.lo, N - 32), __funnelshift_r(v.lo, v.hi, N - 32)};
}
#ifndef SE_SHR_FMA
#define SE_SHR_FMA 0
#endif
// SE_SHR_FMA 1: x >> n as IMAD.HI (x * 2^(32-n)).hi on the FMA pipe (2 issue
// slots there) instead of SHF on the ALU pipe.  Round 1 measured it ahead on
// C2 with the old kernels; re-measured in round 2 (tools/gpu_r2_call15.sh,
// variants A/B): C4 113.7 -> 114.3 GB/s and C2 88.9 -> 90.9 GB/s with the
// plain shift, so 0.
__device__ __forceinline__ uint32_t fshr(uint32_t x, int n, uint32_t one) {
#if SE_SHR_FMA
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(one << (32 - n)));
    return r;
#else
    (void)one;
    return x >> n;
#endif
}

#ifndef SE_ROT_WIDE
#define SE_ROT_WIDE 0
#endif
__device__ __forceinline__ void mulw(uint32_t x, uint32_t pw, uint32_t& lo, uint32_t& hi) {
    uint64_t r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "r"(pw));
    lo = (uint32_t)r;
    hi = (uint32_t)(r >> 32);
}

// rotr64(v, N) = t1 ^ t2 (disjoint pieces), two IMAD.WIDE
template <int N>
__device__ __forceinline__ void ror64w(W64 v, uint32_t one, W64& t1, W64& t2) {
    const uint32_t lo = N < 32 ? v.lo : v.hi, hi = N < 32 ? v.hi : v.lo;
    constexpr int n = N < 32 ? N : N - 32;
    uint32_t pl, ph, ql, qh;
    mulw(lo, one << (32 - n), pl, ph);               // ph = lo >> n, pl = lo << (32-n)
    mulw(hi, one << (32 - n), ql, qh);               // qh = hi >> n, ql = hi << (32-n)
    t1 = W64{ph, qh};
    t2 = W64{ql, pl};
}
__device__ __forceinline__ W64 x64(W64 a, W64 b) { return W64{a.lo ^ b.lo, a.hi ^ b.hi}; }

template <int N>
__device__ __forceinline__ W64 shr64(W64 v, uint32_t one) {   // N < 32
    return W64{__funnelshift_r(v.lo, v.hi, N), fshr(v.hi, N, one)};
}

__device__ __forceinline__ uint32_t ror32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

// ---------------------------------------------------------------- rotations on the FMA pipe
// x * 2^k as a 64-bit product is {hi: x >> (32-k), lo: x << k}: one IMAD.WIDE
// (FMA pipe, two issue slots) yields both pieces of a rotation, which enter
// the XOR tree separately.  Trades ~1 ALU op for ~4 FMA slots (SE_ROT_WIDE
// bit mask).  Measured on B200 (C2 protect, GB/s): off 182, schedule sigmas
// 166, all 149 — IMAD.WIDE costs more than its issue slots (latency, register
// pairs), so the default is off; kept for future re-tuning.
// rotr32(x, n) = a ^ b (disjoint pieces)
__device__ __forceinline__ void ror32w(uint32_t x, int n, uint32_t one, uint32_t& a, uint32_t& b) {
    mulw(x, one << (32 - n), b, a);                   // a = x >> n, b = x << (32-n)
}

// FIPS 180-4 §4.1.2 / §4.1.3 functions.  SE_ROT_WIDE bits: 1 SHA-512 sigma
// (schedule), 2 SHA-512 Sigma, 4 SHA-256 Sigma, 8 SHA-256 sigma: two of the
// three rotations through IMAD.WIDE.
__device__ __forceinline__ uint32_t Sig0_256(uint32_t a, uint32_t one) {
#if SE_ROT_WIDE & 4
    uint32_t p, q, r, t;
    ror32w(a, 2, one, p, q);
    ror32w(a, 13, one, r, t);
    return p ^ q ^ r ^ t ^ ror32(a, 22);
#else
    (void)one;
    return ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22);
#endif
}
__device__ __forceinline__ uint32_t Sig1_256(uint32_t e, uint32_t one) {
#if SE_ROT_WIDE & 4
    uint32_t p, q, r, t;
    ror32w(e, 6, one, p, q);
    ror32w(e, 11, one, r, t);
    return p ^ q ^ r ^ t ^ ror32(e, 25);
#else
    (void)one;
    return ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25);
#endif
}
__device__ __forceinline__ uint32_t sig0_256(uint32_t w, uint32_t one) {
#if SE_ROT_WIDE & 8
    uint32_t p, q, r, t;
    ror32w(w, 7, one, p, q);
    ror32w(w, 18, one, r, t);
    return p ^ q ^ r ^ t ^ fshr(w, 3, one);
#else
    return ror32(w, 7) ^ ror32(w, 18) ^ fshr(w, 3, one);
#endif
}
__device__ __forceinline__ uint32_t sig1_256(uint32_t w, uint32_t one) {
#if SE_ROT_WIDE & 8
    uint32_t p, q, r, t;
    ror32w(w, 17, one, p, q);
    ror32w(w, 19, one, r, t);
    return p ^ q ^ r ^ t ^ fshr(w, 10, one);
#else
    return ror32(w, 17) ^ ror32(w, 19) ^ fshr(w, 10, one);
#endif
}
template <int A, int B, int C, bool WIDE>
__device__ __forceinline__ W64 sig3_512(W64 v, uint32_t one) {       // ror A ^ ror B ^ ror C
    if constexpr (WIDE) {
        W64 p, q, r, t;
        ror64w<A>(v, one, p, q);
        ror64w<B>(v, one, r, t);
        return x64(x64(p, q), x64(x64(r, t), ror64<C>(v)));
    } else {
        return xor3(ror64<A>(v), ror64<B>(v), ror64<C>(v));
    }
}
template <int A, int B, int S, bool WIDE>
__device__ __forceinline__ W64 sig2s_512(W64 v, uint32_t one) {     // ror A ^ ror B ^ shr S
    if constexpr (WIDE) {
        W64 p, q, r, t;
        ror64w<A>(v, one, p, q);
        ror64w<B>(v, one, r, t);
        return x64(x64(p, q), x64(x64(r, t), shr64<S>(v, one)));
    } else {
        return xor3(ror64<A>(v), ror64<B>(v), shr64<S>(v, one));
    }
}


// ---------------------------------------------------------------- SHA-256

// One round on the state held in S[8] with role rotation: at round t the
// working variable i (a = 0 .. h = 7) lives in S[(i - t) & 7].
template <int T>
__device__ __forceinline__ void sha256_round(uint32_t (&S)[8], uint32_t kw, uint32_t one) {
    uint32_t& a = S[(0 - T) & 7];
    uint32_t& b = S[(1 - T) & 7];
    uint32_t& c = S[(2 - T) & 7];
    uint32_t& d = S[(3 - T) & 7];
    uint32_t& e = S[(4 - T) & 7];
    uint32_t& f = S[(5 - T) & 7];
    uint32_t& g = S[(6 - T) & 7];
    uint32_t& h = S[(7 - T) & 7];
    const uint32_t S1 = Sig1_256(e, one);
    const uint32_t ch = (e & f) ^ (~e & g);
    const uint32_t t1 = fadd(fadd(fadd(h, S1, one), ch, one), kw, one);
    const uint32_t S0 = Sig0_256(a, one);
    const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    d = fadd(d, t1, one);                  // new e
    h = fadd(fadd(t1, S0, one), mj, one);  // new a
}

template <int J>
__device__ __forceinline__ uint32_t sha256_sched(uint32_t (&W)[16], uint32_t one) {
    const uint32_t w2 = W[(J - 2) & 15], w15 = W[(J - 15) & 15];
    const uint32_t s1 = sig1_256(w2, one);
    const uint32_t s0 = sig0_256(w15, one);
    const uint32_t w = fadd(fadd(fadd(s1, W[(J - 7) & 15], one), s0, one), W[J & 15], one);
    W[J & 15] = w;
    return w;
}

template <int J>
__device__ __forceinline__ void sha256_msg_rounds(uint32_t (&S)[8], uint32_t (&W)[16], uint32_t one) {
    if constexpr (J < 16) {
        sha256_round<J>(S, fadd(W[J], c_sha256_k[J], one), one);
        sha256_msg_rounds<J + 1>(S, W, one);
    }
}

template <int J>
__device__ __forceinline__ void sha256_sched_rounds(uint32_t (&S)[8], uint32_t (&W)[16], const uint32_t* k,
                                                    uint32_t one) {
    if constexpr (J < 16) {
        const uint32_t w = sha256_sched<J>(W, one);
        sha256_round<J>(S, fadd(w, k[J], one), one);
        sha256_sched_rounds<J + 1>(S, W, k, one);
    }
}

// Loop body of the generic schedules: 8 rounds with a sliding 16-word window
// (half the code) or 16 rounds with rotating indices (no window moves).  The
// single-file protect kernels take 16 for their SHA-256 (SE_SHA256_BODY_P).
#ifndef SE_SHA_BODY
#define SE_SHA_BODY 8
#endif

template <int J>
__device__ __forceinline__ uint32_t& win32(uint32_t (&W)[16], uint32_t (&N)[8]) {
    if constexpr (J < 0) return W[16 + J];
    else return N[J];
}

template <int J>
__device__ __forceinline__ void sha256_sched8_rounds(uint32_t (&S)[8], uint32_t (&W)[16], uint32_t (&N)[8],
                                                     const uint32_t* k, uint32_t one) {
    if constexpr (J < 8) {
        const uint32_t w2 = win32<J - 2>(W, N), w15 = win32<J - 15>(W, N);
        const uint32_t s1 = sig1_256(w2, one);
        const uint32_t s0 = sig0_256(w15, one);
        N[J] = fadd(fadd(fadd(s1, win32<J - 7>(W, N), one), s0, one), win32<J - 16>(W, N), one);
        sha256_round<J>(S, fadd(N[J], k[J], one), one);
        sha256_sched8_rounds<J + 1>(S, W, N, k, one);
    }
}

// SHA-256 of one block whose words W[0..7] were consumed by the host
// midstate `st` (state after round 7); h0 = H(0).  Digest -> H.
template <int BODY = SE_SHA_BODY>
__device__ __forceinline__ void sha256_from_round8(const uint32_t (&st)[8], const uint32_t (&h0)[8],
                                                   uint32_t (&W)[16], uint32_t (&H)[8], uint32_t one) {
    // S[(i - 8) & 7] = S[i] holds variable i at round 8
    uint32_t S[8] = {st[0], st[1], st[2], st[3], st[4], st[5], st[6], st[7]};
    // rounds 8..15 use the message words directly
    sha256_round<8>(S, fadd(W[8], c_sha256_k[8], one), one);
    sha256_round<9>(S, fadd(W[9], c_sha256_k[9], one), one);
    sha256_round<10>(S, fadd(W[10], c_sha256_k[10], one), one);
    sha256_round<11>(S, fadd(W[11], c_sha256_k[11], one), one);
    sha256_round<12>(S, fadd(W[12], c_sha256_k[12], one), one);
    sha256_round<13>(S, fadd(W[13], c_sha256_k[13], one), one);
    sha256_round<14>(S, fadd(W[14], c_sha256_k[14], one), one);
    sha256_round<15>(S, fadd(W[15], c_sha256_k[15], one), one);
    if constexpr (BODY == 8) {
#pragma unroll 1
        for (int r = 16; r < 64; r += 8) {
            uint32_t N[8];
            sha256_sched8_rounds<0>(S, W, N, c_sha256_k + r, one);
#pragma unroll
            for (int i = 0; i < 8; ++i) { W[i] = W[8 + i]; W[8 + i] = N[i]; }
        }
    } else {
#pragma unroll 1
        for (int r = 16; r < 64; r += 16) sha256_sched_rounds<0>(S, W, c_sha256_k + r, one);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) H[i] = fadd(h0[i], S[i], one);   // 64 rounds: roles back in place
}

// ---------------------------------------------------------------- SHA-512

template <int T>
__device__ __forceinline__ void sha512_round(W64 (&S)[8], W64 kw, uint32_t one) {
    W64& a = S[(0 - T) & 7];
    W64& b = S[(1 - T) & 7];
    W64& c = S[(2 - T) & 7];
    W64& d = S[(3 - T) & 7];
    W64& e = S[(4 - T) & 7];
    W64& f = S[(5 - T) & 7];
    W64& g = S[(6 - T) & 7];
    W64& h = S[(7 - T) & 7];
    const W64 S1 = sig3_512<14, 18, 41, (SE_ROT_WIDE & 2) != 0>(e, one);
    const W64 ch = W64{(e.lo & f.lo) ^ (~e.lo & g.lo), (e.hi & f.hi) ^ (~e.hi & g.hi)};
    const W64 t1 = fadd64(fadd64(fadd64(h, S1, one), ch, one), kw, one);
    const W64 S0 = sig3_512<34, 39, 28, (SE_ROT_WIDE & 2) != 0>(a, one);
    const W64 mj = W64{(a.lo & b.lo) ^ (a.lo & c.lo) ^ (b.lo & c.lo), (a.hi & b.hi) ^ (a.hi & c.hi) ^ (b.hi & c.hi)};
    d = fadd64(d, t1, one);
    h = fadd64(fadd64(t1, S0, one), mj, one);
}

template <int J>
__device__ __forceinline__ W64 sha512_sched(W64 (&W)[16], uint32_t one) {
    const W64 w2 = W[(J - 2) & 15], w15 = W[(J - 15) & 15];
    const W64 s1 = sig2s_512<19, 61, 6, (SE_ROT_WIDE & 1) != 0>(w2, one);
    const W64 s0 = sig2s_512<1, 8, 7, (SE_ROT_WIDE & 1) != 0>(w15, one);
    const W64 w = fadd64(fadd64(fadd64(s1, W[(J - 7) & 15], one), s0, one), W[J & 15], one);
    W[J & 15] = w;
    return w;
}

template <int J>
__device__ __forceinline__ void sha512_sched_rounds(W64 (&S)[8], W64 (&W)[16], const uint64_t* k, uint32_t one) {
    if constexpr (J < 16) {
        const W64 w = sha512_sched<J>(W, one);
        sha512_round<J>(S, fadd64(w, w64(k[J]), one), one);
        sha512_sched_rounds<J + 1>(S, W, k, one);
    }
}

template <int T>
__device__ __forceinline__ void sha512_msg_rounds(W64 (&S)[8], W64 (&W)[16], uint32_t one) {
    if constexpr (T < 16) {
        sha512_round<T>(S, fadd64(W[T], w64(c_sha512_k[T]), one), one);
        sha512_msg_rounds<T + 1>(S, W, one);
    }
}

// 8-round loop body: W holds w(t-16..t-1), N receives w(t..t+7); at the end
// the window slides by 8 (16 register moves on the FMA pipe per 8 rounds).
// Half the code of a 16-round body, so the hot loop stays in the L0 I-cache.
template <int J>
__device__ __forceinline__ W64& win(W64 (&W)[16], W64 (&N)[8]) {
    if constexpr (J < 0) return W[16 + J];
    else return N[J];
}

template <int J>
__device__ __forceinline__ void sha512_sched8_rounds(W64 (&S)[8], W64 (&W)[16], W64 (&N)[8], const uint64_t* k,
                                                     uint32_t one) {
    if constexpr (J < 8) {
        const W64 w2 = win<J - 2>(W, N), w15 = win<J - 15>(W, N);
        const W64 s1 = sig2s_512<19, 61, 6, (SE_ROT_WIDE & 1) != 0>(w2, one);
        const W64 s0 = sig2s_512<1, 8, 7, (SE_ROT_WIDE & 1) != 0>(w15, one);
        N[J] = fadd64s(fadd64s(fadd64s(s1, win<J - 7>(W, N), one), s0, one), win<J - 16>(W, N), one);
        sha512_round<J>(S, fadd64(N[J], w64(k[J]), one), one);
        sha512_sched8_rounds<J + 1>(S, W, N, k, one);
    }
}

// SHA-512 of one block resuming at round R0 from state `st` (R0 = 0: st =
// H(0); R0 = 4: W[0..3] = K||IV consumed by the host midstate).  Digest -> H.
template <int R0>
__device__ __forceinline__ void sha512_from_round(const uint64_t (&st)[8], const uint64_t (&h0)[8],
                                                  W64 (&W)[16], uint64_t (&H)[8], uint32_t one) {
    // variable i at round R0 lives in S[(i - R0) & 7]
    W64 S[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) S[(i - R0) & 7] = w64(st[i]);
    sha512_msg_rounds<R0>(S, W, one);
#if SE_SHA_BODY == 8
#pragma unroll 1
    for (int r = 16; r < 80; r += 8) {
        W64 N[8];
        sha512_sched8_rounds<0>(S, W, N, c_sha512_k + r, one);
#pragma unroll
        for (int i = 0; i < 8; ++i) { W[i] = W[8 + i]; W[8 + i] = N[i]; }
    }
#else
#pragma unroll 1
    for (int r = 16; r < 80; r += 16) sha512_sched_rounds<0>(S, W, c_sha512_k + r, one);
#endif
    // after round 79 (80 rounds) variable i lives in S[(i - 80) & 7] = S[i]
#pragma unroll
    for (int i = 0; i < 8; ++i) H[i] = u64(fadd64(w64(h0[i]), S[i], one));
}

__device__ __forceinline__ void sha512_from_round4(const uint64_t (&st)[8], const uint64_t (&h0)[8],
                                                   W64 (&W)[16], uint64_t (&H)[8], uint32_t one) {
    sha512_from_round<4>(st, h0, W, H, one);
}

}  // namespace se
