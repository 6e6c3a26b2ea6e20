// sha2_spec.cuh — SHA-256 / SHA-512 for the B and C masks with the message
// schedule specialised to the framing (C15): only some message words depend
// on the block (the index b and the record bytes); K || IV, the padding and
// the length are the same for every block of a launch.  So is every schedule
// term built only from such words.  The host (se_api.cu, sched_consts*)
// evaluates, for t = 16..31, the block-independent part c_t of
//   W_t = s1(W_{t-2}) + W_{t-7} + s0(W_{t-15}) + W_{t-16}
// (the whole W_t when no term depends on the block) and K_t + W_t for every
// block-independent W_t; the device computes only the block-dependent terms.
// On the C-mask SHA-512 at L = 2 (message words 4, 5, 6 variable) this drops
// 20 of the 64 sigma evaluations and 9 round-constant additions; from t = 32
// on every word depends on the block and the generic 8-round loop takes over.
// Bit-exact by construction (same sums, regrouped; addition is mod 2^n).
#pragma once
#include <stdint.h>

#include "se_internal.h"
#include "sha2_device.cuh"

namespace se {

// unroll factor of the generic 8-round loop (rounds 32-79) after the
// specialised schedule; 1 keeps the hot loop in the instruction cache
// (measured, C2 masked protect / recover GB/s: 1 183.8 / 186.9, 2 ~172 /
// 183.5, 6 161.7 / 166.3 - the window moves it saves cost less than the
// instruction-fetch stalls of the longer body)
#ifndef SE_SHA512_TAIL_UNROLL
#define SE_SHA512_TAIL_UNROLL 1
#endif
constexpr int kSha512TailUnroll = SE_SHA512_TAIL_UNROLL;

template <uint64_t V, int T>
__device__ __forceinline__ constexpr bool var_t() { return (V >> T) & 1u; }

// ---------------------------------------------------------------- SHA-512

template <uint64_t V, int T>
__device__ __forceinline__ W64 w512(const W64 (&W)[16], const W64 (&N)[16]) {
    if constexpr (T < 16) return W[T];
    else return N[T - 16];
}

template <uint64_t V, int T>
__device__ __forceinline__ void sha512_spec_msg(W64 (&S)[8], const W64 (&W)[16], const SchedConst512& sc,
                                                uint32_t one) {
    if constexpr (T < 16) {
        const W64 kw = var_t<V, T>() ? fadd64(W[T], w64(c_sha512_k[T]), one) : w64(sc.kw[T]);
        sha512_round<T>(S, kw, one);
        sha512_spec_msg<V, T + 1>(S, W, sc, one);
    }
}

template <uint64_t V, int T>
__device__ __forceinline__ void sha512_spec_sched(W64 (&S)[8], const W64 (&W)[16], W64 (&N)[16],
                                                  const SchedConst512& sc, uint32_t one) {
    if constexpr (T < 32) {
        W64 w;
        if constexpr (!var_t<V, T>()) {
            w = w64(sc.c[T - 16]);
        } else {
            constexpr bool v2 = var_t<V, T - 2>(), v7 = var_t<V, T - 7>(), v15 = var_t<V, T - 15>(),
                           v16 = var_t<V, T - 16>();
            w = w64(sc.c[T - 16]);                           // block-independent terms (maybe 0)
            if constexpr (v2) w = fadd64(w, sig2s_512<19, 61, 6, (SE_ROT_WIDE & 1) != 0>(w512<V, T - 2>(W, N), one), one);
            if constexpr (v7) w = fadd64(w, w512<V, T - 7>(W, N), one);
            if constexpr (v15) w = fadd64(w, sig2s_512<1, 8, 7, (SE_ROT_WIDE & 1) != 0>(w512<V, T - 15>(W, N), one), one);
            if constexpr (v16) w = fadd64(w, w512<V, T - 16>(W, N), one);
        }
        N[T - 16] = w;
        const W64 kw = var_t<V, T>() ? fadd64(w, w64(c_sha512_k[T]), one) : w64(sc.kw[T]);
        sha512_round<T>(S, kw, one);
        sha512_spec_sched<V, T + 1>(S, W, N, sc, one);
    }
}

// SHA-512 of one block resuming at round R0 from state st (R0 = 4: W[0..3]
// = K||IV in the host midstate; R0 = 0: st = H(0)), schedule specialised for
// message-word mask MSG.  Digest -> H.
template <int R0, uint32_t MSG>
__device__ __forceinline__ void sha512_from_round_spec(const uint64_t (&st)[8], const uint64_t (&h0)[8],
                                                       const W64 (&W)[16], const SchedConst512& sc,
                                                       uint64_t (&H)[8], uint32_t one) {
    constexpr uint64_t V = sched_var(MSG);
    static_assert(((V >> 32) & 0xffffffffull) == 0xffffffffull, "t >= 32 must be block-dependent");
    W64 S[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) S[(i - R0) & 7] = w64(st[i]);
    sha512_spec_msg<V, R0>(S, W, sc, one);
    W64 N[16];                                               // W_16 .. W_31
    sha512_spec_sched<V, 16>(S, W, N, sc, one);
#pragma unroll (kSha512TailUnroll)
    for (int r = 32; r < 80; r += 8) {
        W64 M[8];
        sha512_sched8_rounds<0>(S, N, M, c_sha512_k + r, one);
#pragma unroll
        for (int i = 0; i < 8; ++i) { N[i] = N[8 + i]; N[8 + i] = M[i]; }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) H[i] = u64(fadd64(w64(h0[i]), S[i], one));
}

// ---------------------------------------------------------------- SHA-256

template <uint64_t V, int T>
__device__ __forceinline__ uint32_t w256(const uint32_t (&W)[16], const uint32_t (&N)[16]) {
    if constexpr (T < 16) return W[T];
    else return N[T - 16];
}

template <uint64_t V, int T>
__device__ __forceinline__ void sha256_spec_msg(uint32_t (&S)[8], const uint32_t (&W)[16], const SchedConst256& sc,
                                                uint32_t one) {
    if constexpr (T < 16) {
        const uint32_t kw = var_t<V, T>() ? fadd(W[T], c_sha256_k[T], one) : sc.kw[T];
        sha256_round<T>(S, kw, one);
        sha256_spec_msg<V, T + 1>(S, W, sc, one);
    }
}

template <uint64_t V, int T>
__device__ __forceinline__ void sha256_spec_sched(uint32_t (&S)[8], const uint32_t (&W)[16], uint32_t (&N)[16],
                                                  const SchedConst256& sc, uint32_t one) {
    if constexpr (T < 32) {
        uint32_t w;
        if constexpr (!var_t<V, T>()) {
            w = sc.c[T - 16];
        } else {
            w = sc.c[T - 16];
            if constexpr (var_t<V, T - 2>()) w = fadd(w, sig1_256(w256<V, T - 2>(W, N), one), one);
            if constexpr (var_t<V, T - 7>()) w = fadd(w, w256<V, T - 7>(W, N), one);
            if constexpr (var_t<V, T - 15>()) w = fadd(w, sig0_256(w256<V, T - 15>(W, N), one), one);
            if constexpr (var_t<V, T - 16>()) w = fadd(w, w256<V, T - 16>(W, N), one);
        }
        N[T - 16] = w;
        const uint32_t kw = var_t<V, T>() ? fadd(w, c_sha256_k[T], one) : sc.kw[T];
        sha256_round<T>(S, kw, one);
        sha256_spec_sched<V, T + 1>(S, W, N, sc, one);
    }
}

template <uint32_t MSG>
__device__ __forceinline__ void sha512_from_round4_spec(const uint64_t (&st)[8], const uint64_t (&h0)[8],
                                                        const W64 (&W)[16], const SchedConst512& sc,
                                                        uint64_t (&H)[8], uint32_t one) {
    sha512_from_round_spec<4, MSG>(st, h0, W, sc, H, one);
}

// SHA-256 resuming after round 7 (W[0..7] = K||IV in the host midstate).
template <uint32_t MSG>
__device__ __forceinline__ void sha256_from_round8_spec(const uint32_t (&st)[8], const uint32_t (&h0)[8],
                                                        const uint32_t (&W)[16], const SchedConst256& sc,
                                                        uint32_t (&H)[8], uint32_t one) {
    constexpr uint64_t V = sched_var(MSG);
    static_assert(((V >> 32) & 0xffffffffull) == 0xffffffffull, "t >= 32 must be block-dependent");
    uint32_t S[8] = {st[0], st[1], st[2], st[3], st[4], st[5], st[6], st[7]};
    sha256_spec_msg<V, 8>(S, W, sc, one);
    uint32_t N[16];
    sha256_spec_sched<V, 16>(S, W, N, sc, one);
#pragma unroll 1
    for (int r = 32; r < 64; r += 8) {
        uint32_t M[8];
        sha256_sched8_rounds<0>(S, N, M, c_sha256_k + r, one);
#pragma unroll
        for (int i = 0; i < 8; ++i) { N[i] = N[8 + i]; N[8 + i] = M[i]; }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) H[i] = fadd(h0[i], S[i], one);
}

}  // namespace se
