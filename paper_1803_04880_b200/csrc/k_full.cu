// k_full.cu — FULL-matrix mode (reading C1/C23).
//
// The paper transforms 8x8 blocks but notes the block size
// "can be changed"; FULL mode runs the same lifting (Eq. 5.1-5.2) over the
// whole W x R matrix, level by level, with whole-sample symmetric extension at
// each level's matrix borders, and stores the Mallat layout.  Fragments are
// then regrouped per 8x8 input footprint (4 / 12 / 48 coefficients at L = 2)
// and protected exactly like BLOCK8 records (fused_cta.cuh, MODE 1).
//
// Transform kernels: line-based (streaming) lifting.  A warp owns a column
// group and a segment of rows; each lane owns an 8-column chunk of every row.
// Rows stream through the lane in order: the horizontal lifting of a row runs
// in registers with the chunk-edge neighbours exchanged by warp shuffles, the
// vertical lifting keeps the few rows it needs (pending even / odd row and the
// previous detail row, per level) in registers and emits a finished row pair
// as soon as the next even row arrives; the low-low part of every level-l
// pair is the next row of level l + 1.  One pass over the input, no shared
// memory, no barriers: a global load of 8 bytes per lane per input row and
// 8-byte (4- / 2-byte at levels 2 / 3) Mallat stores per band.
//   Halos.  Every lifting step reads one neighbour of its level on each
// side, so after L levels an output depends on inputs within 2(2^L - 1)
// samples.  Warps overlap by HC chunks on each side (their edge lanes compute
// but do not store); segments process H rows before and after their output
// rows (H = 8 / 8 / 16: >= 2(2^L - 1), a multiple of 8, so the lifting phase
// of the segment equals the global one and rows go in blocks of 8 whose
// parities at every level are compile-time constants).  The first pair of a segment
// and the last one take the matrix-border rules (d(-1) = d(0), x(N) = x(N-2));
// exact at the matrix borders, elsewhere their error stays inside the halo.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>

#include "fused_cta.cuh"

namespace se {

constexpr unsigned kLanes = 0xffffffffu;
constexpr int kStreamThreads = 128, kStreamWarps = kStreamThreads / 32;

template <int L>
struct FStream {
    static constexpr int HC = L == 3 ? 2 : 1;                  // overlap chunks per warp side
    static constexpr int USE = 32 - 2 * HC;                    // chunks a warp stores
    static constexpr int H = L == 3 ? 16 : 8;                   // halo rows (>= 2(2^L - 1), multiple of 8)
};

struct StreamCtx {
    int one, m1;          // 1 and -1, opaque to ptxas (DwtParams::one): IMAD operands
    int W, R;
    int c0;               // first column of the lane's chunk (outside [0, W): a dummy lane)
    bool out_lane;        // lane stores (not an overlap lane, chunk inside the matrix)
    int A, B;             // output rows of the segment (global, multiples of 8)
    int row0, rows_out;   // the call's output window (local Mallat / byte offsets)
    int src0, src_rows;   // inverse: rows present in the local Mallat source
};

// Lifting steps.  SE_FULL_MIX bit 0 (forward) / bit 1 (inverse): the sums as
// IMADs by an opaque +-1 (FMA pipe), leaving one shift-and-add (LEA.HI, ALU
// pipe) per lift, exact values (tests/test_kernel_arith.py checks the
// identities: -floor(m / 2) = floor((1 - m) / 2), -floor((m + 2) / 4) =
// floor((1 - m) / 4)); otherwise plain adds and shifts, which ptxas already
// splits between IADD3 and IMAD.IADD.  Measured (C4-FULL round trip,
// tools/gpu_r2_call42.sh): plain 98.85, forward mixed 98.53, inverse mixed
// 98.77, both 98.45 GB/s — so 0.
#ifndef SE_FULL_MIX
#define SE_FULL_MIX 0
#endif
// L2 prefetch of the next 8 input rows by one lane in 16 (forward transform).
// Measured without it: C4-FULL protect 198.6 -> 196.9 GB/s, so 1.
#ifndef SE_FULL_PREFETCH
#define SE_FULL_PREFETCH 1
#endif
// SE_FULL_LEAN bit 0: the forward predict, bit 1: the inverse update as
// x + ((1 - a - b) >> k), one IADD3 and one LEA.HI, instead of a sum (which
// ptxas puts on the FMA pipe as IMAD.IADD), a shift and a subtraction.
// Measured (tools/gpu_r2_call65.sh, C4-FULL): bit 0 protect 198.6 -> 196.7
// GB/s (the forward transform is ALU-bound), bit 1 recover 197.4 -> 197.8: 2.
#ifndef SE_FULL_LEAN
#define SE_FULL_LEAN 2
#endif
__device__ __forceinline__ int fm_pred(int xo, int xl, int xr, const StreamCtx& c) {   // xo - floor((xl + xr) / 2)
#if SE_FULL_MIX & 1
    return xo + (imad(xl, c.m1, imad(xr, c.m1, 1)) >> 1);
#elif SE_FULL_LEAN & 1
    (void)c;
    return xo + ((1 - xl - xr) >> 1);                            // one IADD3 + one LEA.HI
#else
    (void)c;
    return xo - ((xl + xr) >> 1);
#endif
}
__device__ __forceinline__ int fm_upd(int xe, int dl, int dr, const StreamCtx& c) {    // xe + floor((dl + dr + 2) / 4)
#if SE_FULL_MIX & 1
    return xe + (imad(dl, c.one, imad(dr, c.one, 2)) >> 2);
#else
    (void)c;
    return xe + ((dl + dr + 2) >> 2);
#endif
}
__device__ __forceinline__ int fm_iupd(int sv, int dl, int dr, const StreamCtx& c) {   // sv - floor((dl + dr + 2) / 4)
#if SE_FULL_MIX & 2
    return sv + (imad(dl, c.m1, imad(dr, c.m1, 1)) >> 2);
#elif SE_FULL_LEAN & 2
    (void)c;
    return sv + ((1 - dl - dr) >> 2);                            // -floor((m + 2) / 4) = floor((1 - m) / 4)
#else
    (void)c;
    return sv - ((dl + dr + 2) >> 2);
#endif
}
__device__ __forceinline__ int fm_ipred(int d, int xl, int xr, const StreamCtx& c) {   // d + floor((xl + xr) / 2)
#if SE_FULL_MIX & 2
    return d + (imad(xl, c.one, xr) >> 1);
#else
    (void)c;
    return d + ((xl + xr) >> 1);
#endif
}

// Forward 1-D lifting of one level along a row: v holds NV samples of the
// level (columns gcol .. gcol + NV - 1 of a level row of Nl samples), even =
// s, odd = d on return.  Predict (Eq. 5.1) then update (Eq. 5.2, "+").
template <int NV>
__device__ __forceinline__ void hfwd(int (&v)[NV], int gcol, int Nl, const StreamCtx& c) {
    int xr = __shfl_down_sync(kLanes, v[0], 1);                // next chunk's first sample
    if (gcol + NV >= Nl) xr = v[NV - 2];                        // x(N) = x(N - 2)
#pragma unroll
    for (int m = 1; m < NV; m += 2) v[m] = fm_pred(v[m], v[m - 1], m + 1 < NV ? v[m + 1] : xr, c);
    int dl = __shfl_up_sync(kLanes, v[NV - 1], 1);             // previous chunk's last d
    if (gcol == 0) dl = v[1];                                   // d(-1) = d(0)
#pragma unroll
    for (int m = 0; m < NV; m += 2) v[m] = fm_upd(v[m], m ? v[m - 1] : dl, v[m + 1], c);
}

// Inverse of hfwd: undo the update, then the predict.
template <int NV>
__device__ __forceinline__ void hinv(int (&v)[NV], int gcol, int Nl, const StreamCtx& c) {
    int dl = __shfl_up_sync(kLanes, v[NV - 1], 1);
    if (gcol == 0) dl = v[1];
#pragma unroll
    for (int m = 0; m < NV; m += 2) v[m] = fm_iupd(v[m], m ? v[m - 1] : dl, v[m + 1], c);
    int xr = __shfl_down_sync(kLanes, v[0], 1);
    if (gcol + NV >= Nl) xr = v[NV - 2];
#pragma unroll
    for (int m = 1; m < NV; m += 2) v[m] = fm_ipred(v[m], v[m - 1], m + 1 < NV ? v[m + 1] : xr, c);
}

// NH int16 values (v[OFF], v[OFF + 2], ...) -> 2*NH bytes at g (aligned)
template <int NH, int OFF, int NV>
__device__ __forceinline__ void st_band(int16_t* g, const int (&v)[NV]) {
    if constexpr (NH == 4) {
        uint2 q;
        q.x = (uint32_t)(v[OFF] & 0xffff) | ((uint32_t)v[OFF + 2] << 16);
        q.y = (uint32_t)(v[OFF + 4] & 0xffff) | ((uint32_t)v[OFF + 6] << 16);
        *reinterpret_cast<uint2*>(g) = q;
    } else if constexpr (NH == 2) {
        *reinterpret_cast<uint32_t*>(g) = (uint32_t)(v[OFF] & 0xffff) | ((uint32_t)v[OFF + 2] << 16);
    } else {
        *g = (int16_t)v[OFF];
    }
}



// ---------------------------------------------------------------- forward

template <int NV>
struct FwdLine {          // vertical lifting state of one level
    int E[NV], O[NV], D[NV];
    int n;                // rows received in this segment
};
struct FwdState {
    FwdLine<8> l1;
    FwdLine<4> l2;
    FwdLine<2> l3;
    int kf;               // first input row of the segment
};
template <int l>
__device__ __forceinline__ auto& fline(FwdState& s) {
    if constexpr (l == 1) return s.l1;
    else if constexpr (l == 2) return s.l2;
    else return s.l3;
}

// QM: the level-l row index of the row being pushed, mod 2^(L - l + 1) — a
// compile-time constant (blocks of 8 input rows from a multiple of 8), so the
// even / odd roles of the rows are static and the registers get renamed
// instead of copied.  The LL row a level-l pair hands down has index k = q/2 - 1.
template <int L, int l, int QM>
__device__ __forceinline__ void fwd_push(FwdState& st, int (&x)[8 >> (l - 1)], int16_t* coef, const StreamCtx& c);

// A finished pair of level l (rows 2k, 2k+1 of the level): s row (vertical
// low) and d row.  Stores HL / LH / HH (and LL at l = L); LL feeds level l+1.
template <int L, int l, int QM>
__device__ __forceinline__ void fwd_emit(FwdState& st, int (&sv)[8 >> (l - 1)], const int (&d)[8 >> (l - 1)],
                                         int k, int16_t* coef, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1), NH = NV / 2;
    const int r_in = k << l;                                    // first input row of the pair
    if (c.out_lane && r_in >= c.A && r_in < c.B) {
        const int64_t top = k - (c.row0 >> l), bot = top + (c.rows_out >> l);
        const int colL = c.c0 >> l, colH = (c.W >> l) + colL;
        st_band<NH, 1>(coef + top * c.W + colH, sv);             // HL: vertical low, horizontal high
        st_band<NH, 0>(coef + bot * c.W + colL, d);              // LH
        st_band<NH, 1>(coef + bot * c.W + colH, d);              // HH
        if constexpr (l == L) {                                 // LL_L, centered (C8) here
            int ll[NV];
#pragma unroll
            for (int i = 0; i < NV; i += 2) ll[i] = sv[i] - 128;
            st_band<NH, 0>(coef + top * c.W + colL, ll);
        }
    }
    if constexpr (l < L) {
        int y[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) y[i] = sv[2 * i];
        fwd_push<L, l + 1, ((QM >> 1) - 1) & ((1 << (L - l)) - 1)>(st, y, coef, c);
    }
}

// Pair (E, O) completed by the next even row xn (x(N) = x(N-2) at the end: xn = E).
template <int L, int l, int QM>
__device__ __forceinline__ void fwd_pair(FwdState& st, const int (&xn)[8 >> (l - 1)], int16_t* coef,
                                         const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = fline<l>(st);
    int d[NV], sv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) d[i] = fm_pred(s.O[i], s.E[i], xn[i], c);
    if (s.n == 2) {                                             // first pair: d(-1) = d(0)
#pragma unroll
        for (int i = 0; i < NV; ++i) s.D[i] = d[i];
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) sv[i] = fm_upd(s.E[i], s.D[i], d[i], c);
#pragma unroll
    for (int i = 0; i < NV; ++i) s.D[i] = d[i];
    const int k = ((st.kf >> (l - 1)) + s.n - 2) >> 1;
    fwd_emit<L, l, QM>(st, sv, d, k, coef, c);
}

template <int L, int l, int QM>
__device__ __forceinline__ void fwd_push(FwdState& st, int (&x)[8 >> (l - 1)], int16_t* coef, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = fline<l>(st);
    hfwd<NV>(x, c.c0 >> (l - 1), c.W >> (l - 1), c);             // row pass of level l
    if constexpr ((QM & 1) == 0) {
        if (s.n >= 2) fwd_pair<L, l, QM>(st, x, coef, c);
#pragma unroll
        for (int i = 0; i < NV; ++i) s.E[i] = x[i];
    } else {
#pragma unroll
        for (int i = 0; i < NV; ++i) s.O[i] = x[i];
    }
    ++s.n;
}

template <int L, int l>
__device__ __forceinline__ void fwd_finish(FwdState& st, int16_t* coef, const StreamCtx& c) {
    auto& s = fline<l>(st);
    if (s.n >= 2) {                                             // pending pair (row counts are even)
        int e[8 >> (l - 1)];
#pragma unroll
        for (int i = 0; i < (8 >> (l - 1)); ++i) e[i] = s.E[i];
        fwd_pair<L, l, 0>(st, e, coef, c);                      // x(N) = x(N - 2)
    }
    if constexpr (l < L) fwd_finish<L, l + 1>(st, coef, c);
}

// 8 bytes of row r at columns c0..c0+7 as raw bytes.  The lifting runs on
// the uncentered bytes: shifting every sample by an even constant c shifts
// each s by c and leaves each d unchanged ((a + 2c) >> 1 = (a >> 1) + c in the
// predict; the update adds d's only), level after level, so the centering
// (C8, x = b - 128) is applied to LL_L alone (fwd_emit; the inverse adds it
// back on load).  Bytes past n read 0 (x = -128, C18); other bytes of rows
// outside the source window read 0x80 (x = 0; they only feed halo rows).
__device__ __forceinline__ uint2 fetch_row(const DwtParams& p, int r, int c0, bool col_ok) {
    const uint2 none = make_uint2(0x80808080u, 0x80808080u);
    if (!col_ok) return none;
    const uint64_t o = (uint64_t)r * p.width + c0;
    const bool have = r >= (int)p.src_row0 && r < (int)(p.src_row0 + p.src_rows);
    const uint8_t* src = p.in + (uint64_t)(r - (int)p.src_row0) * p.width + c0;
    if (o + 8 <= p.n_bytes) return have ? __ldg(reinterpret_cast<const uint2*>(src)) : none;
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int b = 0; b < 8; ++b)
        if (o + b < p.n_bytes) w[b >> 2] |= (have ? (uint32_t)src[b] : 0x80u) << (8 * (b & 3));
    return make_uint2(w[0], w[1]);
}

__device__ __forceinline__ void stream_ctx(StreamCtx& c, const DwtParams& p, int HC, int USE, int seg, int ncg,
                                           int& sg) {
    const int lane = threadIdx.x & 31;
    const int wid = (int)blockIdx.x * kStreamWarps + (int)(threadIdx.x >> 5);
    const int cg = wid % ncg;
    sg = wid / ncg;
    c.one = (int)p.one;
    c.m1 = -(int)p.one;
    c.W = (int)p.width;
    c.R = (int)p.rows;
    c.c0 = 8 * (cg * USE - HC + lane);
    c.out_lane = lane >= HC && lane < 32 - HC && c.c0 < c.W;
    c.row0 = (int)p.row0;
    c.rows_out = (int)p.rows_out;
    const int row_end = min((int)(p.row0 + p.rows_out), c.R);
    c.A = c.row0 + sg * seg;
    c.B = min(c.A + seg, row_end);
    c.src0 = (int)p.src_row0;
    c.src_rows = (int)p.src_rows;
}

template <int L, int J>
__device__ __forceinline__ void fwd_rows(FwdState& st, const uint2 (&q)[8], int16_t* coef, const StreamCtx& c) {
    if constexpr (J < 8) {
        int x[8];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            x[b] = (int)__byte_perm(q[J].x, 0u, 0x4440u + b);     // zero-extended byte (uncentered: see fwd_emit)
            x[4 + b] = (int)__byte_perm(q[J].y, 0u, 0x4440u + b);
        }
        fwd_push<L, 1, J & ((1 << L) - 1)>(st, x, coef, c);
        fwd_rows<L, J + 1>(st, q, coef, c);
    }
}

// Shared-memory carveout of the streaming transforms (no shared memory of
// their own): SE_FULL_CARVEOUT 0 leave the driver default, 1 maximum shared
// (as the footprint kernels around them), 2 maximum L1.  Measured
// (tools/gpu_r2_call57.sh, C4-FULL round trip): 0 99.0, 1 97.7 (the inverse
// transform loses its L1: recover 197.3 -> 192.8 GB/s), 2 99.0 GB/s: 0.
#ifndef SE_FULL_CARVEOUT
#define SE_FULL_CARVEOUT 0
#endif
static void full_carveout(const void* kernel) {
#if SE_FULL_CARVEOUT == 1
    carveout_max_once(kernel);
#elif SE_FULL_CARVEOUT == 2
    static thread_local const void* seen[8];
    static thread_local int n = 0;
    for (int i = 0; i < n; ++i)
        if (seen[i] == kernel) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxL1);
    if (n < 8) seen[n++] = kernel;
#else
    (void)kernel;
#endif
}

template <int L>
__global__ void __launch_bounds__(kStreamThreads) k_dwt_full_fwd(const __grid_constant__ DwtParams p, int seg,
                                                                 int ncg, int nseg) {
    using F = FStream<L>;
    StreamCtx c;
    int sg;
    stream_ctx(c, p, F::HC, F::USE, seg, ncg, sg);
    if (sg >= nseg) return;                                     // whole warp
    const int P0 = max(c.A - F::H, 0), P1 = min(c.B + F::H, c.R);
    const bool col_ok = c.c0 >= 0 && c.c0 < c.W;
    FwdState st;
    st.kf = P0;
    st.l1.n = 0;
    st.l2.n = 0;
    st.l3.n = 0;
    for (int r = P0; r < P1; r += 8) {                         // blocks of 8 rows
        uint2 q[8];
        const int lr = r - (int)p.src_row0;                     // local row in the source window
        if (col_ok && lr >= 0 && lr + 8 <= (int)p.src_rows && (uint64_t)(r + 7) * p.width + c.c0 + 8 <= p.n_bytes) {
            const uint8_t* src = p.in + (uint64_t)lr * p.width + c.c0;   // whole block present
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = __ldg(reinterpret_cast<const uint2*>(src + (uint64_t)j * p.width));
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = fetch_row(p, r + j, c.c0, col_ok);
        }
        if (SE_FULL_PREFETCH && r + 8 < P1 && col_ok && (threadIdx.x & 15) == 0) {   // next block -> L2
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int rr = r + 8 + j - (int)p.src_row0;
                if (rr >= 0 && rr < (int)p.src_rows)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.in + (uint64_t)rr * p.width + c.c0));
            }
        }
        fwd_rows<L, 0>(st, q, p.coef, c);
    }
    fwd_finish<L, 1>(st, p.coef, c);
}

// ---------------------------------------------------------------- inverse

template <int NV>
struct InvLine {
    int X[NV], D[NV];     // last even row rebuilt (x_2k) and d_k
    int n;                // pairs received in this segment
};
struct InvState {
    InvLine<8> l1;
    InvLine<4> l2;
    InvLine<2> l3;
    int kf;               // first input row of the segment
    uint32_t bad;         // footprint row flag (level 1 output)
};
template <int l>
__device__ __forceinline__ auto& iline(InvState& s) {
    if constexpr (l == 1) return s.l1;
    else if constexpr (l == 2) return s.l2;
    else return s.l3;
}

struct InvOut {
    const int16_t* coef;
    uint8_t* out;
    uint64_t n_bytes;
    se_report* report;
};

// One iteration's band rows, raw (8 output rows = 8 >> L top-level pairs):
// level l rows jb_l + t, t < 8 >> l, jb_l = (k0 << (L - l)) - (2^(L - l) - 1)
// (the rows the iteration's pairs emit), bands LL (top level only), HL, LH,
// HH.  All loads of an iteration are issued before its arithmetic.
struct InvPre {
    uint2 b1[4][4];
    uint2 b2[2][4];
    uint2 b3[1][4];
};
template <int l>
__device__ __forceinline__ auto& prow(InvPre& p) {
    if constexpr (l == 1) return p.b1;
    else if constexpr (l == 2) return p.b2;
    else return p.b3;
}

template <int l>
__device__ __forceinline__ uint2 ld_raw(const InvOut& o, const StreamCtx& c, int j, bool hr, bool hc) {
    const int sb0 = c.src0 >> l, sbn = c.src_rows >> l;
    if (c.c0 < 0 || c.c0 >= c.W || j < sb0 || j >= sb0 + sbn) return make_uint2(0, 0);
    const int16_t* g = o.coef + ((int64_t)(hr ? sbn : 0) + (j - sb0)) * c.W + (hc ? (c.W >> l) : 0) + (c.c0 >> l);
    if constexpr (l == 1) return __ldg(reinterpret_cast<const uint2*>(g));
    else if constexpr (l == 2) return make_uint2(__ldg(reinterpret_cast<const uint32_t*>(g)), 0u);
    else return make_uint2((uint32_t)(uint16_t)__ldg(g), 0u);
}

template <int NH>
__device__ __forceinline__ void unpack_band(uint2 q, int (&v)[NH]) {
    v[0] = (int)(int16_t)(q.x & 0xffff);
    if constexpr (NH >= 2) v[1] = (int)q.x >> 16;
    if constexpr (NH == 4) {
        v[2] = (int)(int16_t)(q.y & 0xffff);
        v[3] = (int)q.y >> 16;
    }
}

// every band row of the iteration inside the source window (and the lane's
// chunk inside the matrix): the loads need no tests
template <int L, int l>
__device__ __forceinline__ bool window_ok(const StreamCtx& c, int k0) {
    const int jb = (k0 << (L - l)) - ((1 << (L - l)) - 1);
    const int sb0 = c.src0 >> l, sbn = c.src_rows >> l;
    bool ok = jb >= sb0 && jb + (8 >> l) <= sb0 + sbn;
    if constexpr (l > 1) ok = ok && window_ok<L, l - 1>(c, k0);
    return ok;
}

template <int L, int l>
__device__ __forceinline__ void preload(InvPre& pre, const InvOut& o, const StreamCtx& c, int k0, bool fast) {
    constexpr int NR = 8 >> l;
    const int jb = (k0 << (L - l)) - ((1 << (L - l)) - 1);
    auto& b = prow<l>(pre);
    if (fast) {
        const int sb0 = c.src0 >> l, sbn = c.src_rows >> l;
        const int16_t* g0 = o.coef + (int64_t)(jb - sb0) * c.W + (c.c0 >> l);
        const int64_t hr = (int64_t)sbn * c.W;
        const int hc = c.W >> l;
#pragma unroll
        for (int t = 0; t < NR; ++t) {
#pragma unroll
            for (int band = (l == L ? 0 : 1); band < 4; ++band) {
                const int16_t* g = g0 + (int64_t)t * c.W + (band >= 2 ? hr : 0) + ((band & 1) ? hc : 0);
                if constexpr (l == 1) b[t][band] = __ldg(reinterpret_cast<const uint2*>(g));
                else if constexpr (l == 2) b[t][band] = make_uint2(__ldg(reinterpret_cast<const uint32_t*>(g)), 0u);
                else b[t][band] = make_uint2((uint32_t)(uint16_t)__ldg(g), 0u);
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < NR; ++t)
#pragma unroll
            for (int band = (l == L ? 0 : 1); band < 4; ++band)
                b[t][band] = ld_raw<l>(o, c, jb + t, band >= 2, band & 1);
    }
    if constexpr (l > 1) preload<L, l - 1>(pre, o, c, k0, fast);
}

template <int L, int l, int T>
__device__ __forceinline__ void inv_push(InvState& st, const int (&sr)[8 >> (l - 1)], const int (&dr)[8 >> (l - 1)],
                                         InvPre& pre, const InvOut& o, const StreamCtx& c);

// A row j of level l - 1's low-low band (or of the output, l = 1) rebuilt
// vertically at level l: undo the row pass, then hand it down.  T >= 0: the
// row's band data sit in pre (static index); T < 0: loaded here (finish).
template <int L, int l, int T>
__device__ __forceinline__ void inv_emit(InvState& st, int (&v)[8 >> (l - 1)], int j, InvPre& pre, const InvOut& o,
                                         const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    hinv<NV>(v, c.c0 >> (l - 1), c.W >> (l - 1), c);
    if constexpr (l == 1) {
        if (c.out_lane && j >= c.A && j < c.B) {
            uint32_t w[2] = {0, 0};
            int orv = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int b = v[i];                             // uncentered (LL_L + 128 on load)
                orv |= b;
                w[i >> 2] |= (uint32_t)(b & 0xff) << (8 * (i & 3));
            }
            if (orv & ~0xff) st.bad = 1;                        // a sample outside [0, 255]
            const uint64_t off = (uint64_t)j * c.W + c.c0;
            uint8_t* dst = o.out + (uint64_t)(j - c.row0) * c.W + c.c0;
            if (off + 8 <= o.n_bytes) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
            } else {
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    if (off + b < o.n_bytes) dst[b] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
            }
            if ((j & 7) == 7) {                                 // footprint row complete
                if (st.bad && o.report) {
                    const unsigned long long blk =
                        (unsigned long long)((j >> 3) - (c.row0 >> 3)) * (c.W >> 3) + (c.c0 >> 3);
                    atomicMin(reinterpret_cast<unsigned long long*>(&o.report->first_bad_block), blk);
                    atomicAdd(reinterpret_cast<unsigned long long*>(&o.report->bad_blocks), 1ull);
                }
                st.bad = 0;
            }
        }
    } else {
        // pair j of level l - 1: s row = (LL_{l-1}[j], HL_{l-1}[j]) interleaved, d row = (LH, HH)
        constexpr int NV2 = 2 * NV;
        int hl[NV], lh[NV], hh[NV];
        if constexpr (T >= 0) {
            auto& b = prow<l - 1>(pre);
            unpack_band<NV>(b[T][1], hl);
            unpack_band<NV>(b[T][2], lh);
            unpack_band<NV>(b[T][3], hh);
        } else {
            unpack_band<NV>(ld_raw<l - 1>(o, c, j, false, true), hl);
            unpack_band<NV>(ld_raw<l - 1>(o, c, j, true, false), lh);
            unpack_band<NV>(ld_raw<l - 1>(o, c, j, true, true), hh);
        }
        int sr[NV2], dr[NV2];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            sr[2 * i] = v[i];
            sr[2 * i + 1] = hl[i];
            dr[2 * i] = lh[i];
            dr[2 * i + 1] = hh[i];
        }
        inv_push<L, l - 1, T>(st, sr, dr, pre, o, c);
    }
}

// Pair k of level l arrives: x_2k = s_k - (d_{k-1} + d_k + 2) >> 2, then
// x_{2k-1} = d_{k-1} + (x_{2k-2} + x_2k) >> 1; rows leave in order.  Pair T
// of an iteration emits rows 2T and 2T + 1 of the next level's rows.
template <int L, int l, int T>
__device__ __forceinline__ void inv_push(InvState& st, const int (&sr)[8 >> (l - 1)], const int (&dr)[8 >> (l - 1)],
                                         InvPre& pre, const InvOut& o, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = iline<l>(st);
    const int k = (st.kf >> l) + s.n;
    if (s.n == 0) {                                             // first pair: d(-1) = d(0)
#pragma unroll
        for (int i = 0; i < NV; ++i) s.D[i] = dr[i];
    }
    int x[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i] = fm_iupd(sr[i], s.D[i], dr[i], c);
    if (s.n != 0) {
        int xo[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) xo[i] = fm_ipred(s.D[i], s.X[i], x[i], c);
        inv_emit<L, l, (T >= 0 ? 2 * T : -1)>(st, xo, 2 * k - 1, pre, o, c);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        s.X[i] = x[i];
        s.D[i] = dr[i];
    }
    ++s.n;
    inv_emit<L, l, (T >= 0 ? 2 * T + 1 : -1)>(st, x, 2 * k, pre, o, c);
}

// last odd row of each level: x_{2K+2} = x_2K (reflection; exact at the matrix bottom)
template <int L, int l>
__device__ __forceinline__ void inv_finish(InvState& st, InvPre& pre, const InvOut& o, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = iline<l>(st);
    if (s.n > 0) {
        int xo[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) xo[i] = s.D[i] + s.X[i];   // d + (2x >> 1)
        inv_emit<L, l, -1>(st, xo, 2 * ((st.kf >> l) + s.n - 1) + 1, pre, o, c);
    }
    if constexpr (l > 1) inv_finish<L, l - 1>(st, pre, o, c);
}

template <int L, int I>
__device__ __forceinline__ void inv_top(InvState& st, InvPre& pre, const InvOut& o, const StreamCtx& c) {
    if constexpr (I < (8 >> L)) {
        constexpr int NV = 8 >> (L - 1), NH = NV / 2;
        auto& b = prow<L>(pre);
        int ll[NH], hl[NH], lh[NH], hh[NH];
        unpack_band<NH>(b[I][0], ll);
#pragma unroll
        for (int i = 0; i < NH; ++i) ll[i] += 128;                // uncentered domain (see fetch_row)
        unpack_band<NH>(b[I][1], hl);
        unpack_band<NH>(b[I][2], lh);
        unpack_band<NH>(b[I][3], hh);
        int sr[NV], dr[NV];
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            sr[2 * i] = ll[i];
            sr[2 * i + 1] = hl[i];
            dr[2 * i] = lh[i];
            dr[2 * i + 1] = hh[i];
        }
        inv_push<L, L, I>(st, sr, dr, pre, o, c);
        inv_top<L, I + 1>(st, pre, o, c);
    }
}

template <int L>
__global__ void __launch_bounds__(kStreamThreads) k_dwt_full_inv(const __grid_constant__ DwtParams p,
                                                                 se_report* report, int seg, int ncg, int nseg) {
    using F = FStream<L>;
    StreamCtx c;
    int sg;
    stream_ctx(c, p, F::HC, F::USE, seg, ncg, sg);
    if (sg >= nseg) return;
    const int P0 = max(c.A - F::H, 0), P1 = min(c.B + F::H, c.R);
    InvOut o{p.coef, p.out, p.n_bytes, report};
    InvState st;
    st.kf = P0;
    st.l1.n = 0;
    st.l2.n = 0;
    st.l3.n = 0;
    st.bad = 0;
    InvPre pre;
    for (int k0 = P0 >> L; k0 < (P1 >> L); k0 += 8 >> L) {     // 8 output rows per iteration
        preload<L, L>(pre, o, c, k0, c.c0 >= 0 && c.c0 < c.W && window_ok<L, L>(c, k0));
        inv_top<L, 0>(st, pre, o, c);
    }
    inv_finish<L, L>(st, pre, o, c);
}

#ifndef SE_MIN_CTAS_FULL
#define SE_MIN_CTAS_FULL 4
#endif
template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS_FULL) k_protect_full(const __grid_constant__ FusedParams p) {
    protect_cta<L, MASK, 1>(p, blockIdx.x);
}

template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS_FULL) k_recover_full(const __grid_constant__ FusedParams p) {
    recover_cta<L, MASK, 1>(p, blockIdx.x);
}

// ---------------------------------------------------------------- launchers

// Launch shape: warps = column groups x row segments; segments of 256 rows,
// halved (down to 32) until the grid holds one full wave of warps (24 per
// SM at ~80 registers): shorter segments re-read relatively more halo rows
// (2H per segment).
static std::atomic<int> g_seg_override{0};     // se_full_segment_rows (tests): 0 = by size

template <int L>
static void stream_shape(const DwtParams& p, int& seg, int& ncg, int& nseg, unsigned& grid) {
    using F = FStream<L>;
    ncg = (int)((p.width / 8 + F::USE - 1) / F::USE);
    const uint64_t rows = std::min<uint64_t>(p.row0 + p.rows_out, p.rows) - p.row0;
    seg = 256;
    while (seg > 32 && (uint64_t)ncg * ((rows + seg - 1) / seg) < 148ull * 24) seg /= 2;
    if (const int o = g_seg_override.load(std::memory_order_relaxed)) seg = o;
    nseg = (int)((rows + seg - 1) / seg);
    grid = (unsigned)(((uint64_t)ncg * nseg + kStreamWarps - 1) / kStreamWarps);
}

template <int L>
static int full_fwd_l(const DwtParams& p, cudaStream_t s) {
    int seg, ncg, nseg;
    unsigned grid;
    stream_shape<L>(p, seg, ncg, nseg, grid);
    full_carveout((const void*)k_dwt_full_fwd<L>);
    if (grid) k_dwt_full_fwd<L><<<grid, kStreamThreads, 0, s>>>(p, seg, ncg, nseg);
    return (int)cudaGetLastError();
}

template <int L>
static int full_inv_l(const DwtParams& p, se_report* rep, cudaStream_t s) {
    int seg, ncg, nseg;
    unsigned grid;
    stream_shape<L>(p, seg, ncg, nseg, grid);
    full_carveout((const void*)k_dwt_full_inv<L>);
    if (grid) k_dwt_full_inv<L><<<grid, kStreamThreads, 0, s>>>(p, rep, seg, ncg, nseg);
    return (int)cudaGetLastError();
}

}  // namespace se

// Segment rows of the streaming FULL-mode transform (32, 64, 128 or 256;
// 0 = chosen by size, the default).  Test knob: the segment length decides
// which halo and window code runs, so the tests compare every length with the
// oracle.  Returns the previous value, or SE_EINVAL for another length.
extern "C" int se_full_segment_rows(int rows) {
    if (rows != 0 && rows != 32 && rows != 64 && rows != 128 && rows != 256) return SE_EINVAL;
    return se::g_seg_override.exchange(rows);
}

namespace se {

int launch_dwt_full_fwd(const DwtParams& p, uint32_t levels, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    note_launch();
    return levels == 1 ? full_fwd_l<1>(p, s) : levels == 2 ? full_fwd_l<2>(p, s) : full_fwd_l<3>(p, s);
}

int launch_dwt_full_inv(const DwtParams& p, uint32_t levels, se_report* report, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    note_launch();
    return levels == 1 ? full_inv_l<1>(p, report, s) : levels == 2 ? full_inv_l<2>(p, report, s)
                                                      : full_inv_l<3>(p, report, s);
}

template <int L>
static void prot_full_l(const FusedParams& p, bool mask, cudaStream_t s) {
    const unsigned g = (unsigned)((p.n_blocks + kBlocksPerCta - 1) / kBlocksPerCta);
    if (mask) launch_pdl(k_protect_full<L, true>, g, kBlocksPerCta, s, p);
    else launch_pdl(k_protect_full<L, false>, g, kBlocksPerCta, s, p);
}

template <int L>
static void rec_full_l(const FusedParams& p, bool mask, cudaStream_t s) {
    const unsigned g = (unsigned)((p.n_blocks + kBlocksPerCta - 1) / kBlocksPerCta);
    if (mask) launch_pdl(k_recover_full<L, true>, g, kBlocksPerCta, s, p);
    else launch_pdl(k_recover_full<L, false>, g, kBlocksPerCta, s, p);
}

int launch_protect_full(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) prot_full_l<1>(p, mask, s);
    else if (levels == 2) prot_full_l<2>(p, mask, s);
    else prot_full_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

int launch_recover_full(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) rec_full_l<1>(p, mask, s);
    else if (levels == 2) rec_full_l<2>(p, mask, s);
    else rec_full_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
