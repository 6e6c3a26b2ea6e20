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
// rows (H = 4 / 8 / 16: >= 2(2^L - 1), a multiple of 2^L so the lifting
// phase of the segment equals the global one).  The first pair of a segment
// and the last one take the matrix-border rules (d(-1) = d(0), x(N) = x(N-2));
// exact at the matrix borders, elsewhere their error stays inside the halo.
#include <cuda_runtime.h>

#include <algorithm>

#include "fused_cta.cuh"

namespace se {

constexpr unsigned kLanes = 0xffffffffu;
constexpr int kStreamThreads = 128, kStreamWarps = kStreamThreads / 32;

template <int L>
struct FStream {
    static constexpr int HC = L == 3 ? 2 : 1;                  // overlap chunks per warp side
    static constexpr int USE = 32 - 2 * HC;                    // chunks a warp stores
    static constexpr int H = L == 1 ? 4 : L == 2 ? 8 : 16;      // halo rows
};

// Forward 1-D lifting of one level along a row: v holds NV samples of the
// level (columns gcol .. gcol + NV - 1 of a level row of Nl samples), even =
// s, odd = d on return.  Predict (Eq. 5.1) then update (Eq. 5.2, "+").
template <int NV>
__device__ __forceinline__ void hfwd(int (&v)[NV], int gcol, int Nl) {
    int xr = __shfl_down_sync(kLanes, v[0], 1);                // next chunk's first sample
    if (gcol + NV >= Nl) xr = v[NV - 2];                        // x(N) = x(N - 2)
#pragma unroll
    for (int m = 1; m < NV; m += 2) v[m] -= (v[m - 1] + (m + 1 < NV ? v[m + 1] : xr)) >> 1;
    int dl = __shfl_up_sync(kLanes, v[NV - 1], 1);             // previous chunk's last d
    if (gcol == 0) dl = v[1];                                   // d(-1) = d(0)
#pragma unroll
    for (int m = 0; m < NV; m += 2) v[m] += ((m ? v[m - 1] : dl) + v[m + 1] + 2) >> 2;
}

// Inverse of hfwd: undo the update, then the predict.
template <int NV>
__device__ __forceinline__ void hinv(int (&v)[NV], int gcol, int Nl) {
    int dl = __shfl_up_sync(kLanes, v[NV - 1], 1);
    if (gcol == 0) dl = v[1];
#pragma unroll
    for (int m = 0; m < NV; m += 2) v[m] -= ((m ? v[m - 1] : dl) + v[m + 1] + 2) >> 2;
    int xr = __shfl_down_sync(kLanes, v[0], 1);
    if (gcol + NV >= Nl) xr = v[NV - 2];
#pragma unroll
    for (int m = 1; m < NV; m += 2) v[m] += (v[m - 1] + (m + 1 < NV ? v[m + 1] : xr)) >> 1;
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

template <int NH>
__device__ __forceinline__ void ld_band(const int16_t* g, int (&v)[NH]) {
    if constexpr (NH == 4) {
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(g));
        v[0] = (int)(int16_t)(q.x & 0xffff); v[1] = (int)q.x >> 16;
        v[2] = (int)(int16_t)(q.y & 0xffff); v[3] = (int)q.y >> 16;
    } else if constexpr (NH == 2) {
        const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(g));
        v[0] = (int)(int16_t)(q & 0xffff); v[1] = (int)q >> 16;
    } else {
        v[0] = __ldg(g);
    }
}

struct StreamCtx {
    int W, R;
    int c0;               // first column of the lane's chunk (outside [0, W): a dummy lane)
    bool out_lane;        // lane stores (not an overlap lane, chunk inside the matrix)
    int A, B;             // output rows of the segment (global, multiples of 8)
    int row0, rows_out;   // the call's output window (local Mallat / byte offsets)
    int src0, src_rows;   // inverse: rows present in the local Mallat source
};

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

template <int L, int l>
__device__ __forceinline__ void fwd_push(FwdState& st, int (&x)[8 >> (l - 1)], int16_t* coef, const StreamCtx& c);

// A finished pair of level l (rows 2k, 2k+1 of the level): s row (vertical
// low) and d row.  Stores HL / LH / HH (and LL at l = L); LL feeds level l+1.
template <int L, int l>
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
        if constexpr (l == L) st_band<NH, 0>(coef + top * c.W + colL, sv);   // LL_L
    }
    if constexpr (l < L) {
        int y[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) y[i] = sv[2 * i];
        fwd_push<L, l + 1>(st, y, coef, c);
    }
}

// Pair (E, O) completed by the next even row xn (x(N) = x(N-2) at the end: xn = E).
template <int L, int l>
__device__ __forceinline__ void fwd_pair(FwdState& st, const int (&xn)[8 >> (l - 1)], int16_t* coef,
                                         const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = fline<l>(st);
    int d[NV], sv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) d[i] = s.O[i] - ((s.E[i] + xn[i]) >> 1);
    const bool first = s.n == 2;                                // d(-1) = d(0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sv[i] = s.E[i] + (((first ? d[i] : s.D[i]) + d[i] + 2) >> 2);
#pragma unroll
    for (int i = 0; i < NV; ++i) s.D[i] = d[i];
    const int k = ((st.kf >> (l - 1)) + s.n - 2) >> 1;
    fwd_emit<L, l>(st, sv, d, k, coef, c);
}

template <int L, int l>
__device__ __forceinline__ void fwd_push(FwdState& st, int (&x)[8 >> (l - 1)], int16_t* coef, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = fline<l>(st);
    hfwd<NV>(x, c.c0 >> (l - 1), c.W >> (l - 1));             // row pass of level l
    if ((s.n & 1) == 0) {
        if (s.n >= 2) fwd_pair<L, l>(st, x, coef, c);
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
    if (s.n >= 2 && (s.n & 1) == 0) {
        int e[8 >> (l - 1)];
#pragma unroll
        for (int i = 0; i < (8 >> (l - 1)); ++i) e[i] = s.E[i];
        fwd_pair<L, l>(st, e, coef, c);                         // x(N) = x(N - 2)
    }
    if constexpr (l < L) fwd_finish<L, l + 1>(st, coef, c);
}

// 8 bytes of row r at columns c0..c0+7 as raw bytes: centering (C8) is
// applied by the caller (x = b - 128); bytes past n read 0 (-> -128, C18),
// other bytes of rows outside the source window read 0x80 (-> 0; they only
// feed halo rows).
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
    uint2 nxt = fetch_row(p, P0, c.c0, col_ok);
    for (int r = P0; r < P1; ++r) {
        const uint2 q = nxt;
        if (r + 1 < P1) nxt = fetch_row(p, r + 1, c.c0, col_ok);
        int x[8];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            x[b] = (int)((q.x >> (8 * b)) & 0xff) - 128;
            x[4 + b] = (int)((q.y >> (8 * b)) & 0xff) - 128;
        }
        fwd_push<L, 1>(st, x, p.coef, c);
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

template <int L, int l>
__device__ __forceinline__ void inv_push(InvState& st, const int (&sr)[8 >> (l - 1)],
                                         const int (&dr)[8 >> (l - 1)], const InvOut& o, const StreamCtx& c);

// band row j of level l (NH values at the lane's columns), 0 outside the source window
template <int l, int NH>
__device__ __forceinline__ void load_band(int (&v)[NH], const InvOut& o, const StreamCtx& c, int j, bool hr, bool hc) {
    const int sb0 = c.src0 >> l, sbn = c.src_rows >> l;
    if (c.c0 < 0 || c.c0 >= c.W || j < sb0 || j >= sb0 + sbn) {
#pragma unroll
        for (int i = 0; i < NH; ++i) v[i] = 0;
        return;
    }
    const int64_t row = (hr ? sbn : 0) + (j - sb0);
    const int col = (hc ? (c.W >> l) : 0) + (c.c0 >> l);
    ld_band<NH>(o.coef + row * c.W + col, v);
}

// A row j of level l - 1's low-low band (or of the output, l = 1) rebuilt
// vertically at level l: undo the row pass, then hand it down.
template <int L, int l>
__device__ __forceinline__ void inv_emit(InvState& st, int (&v)[8 >> (l - 1)], int j, const InvOut& o,
                                         const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    hinv<NV>(v, c.c0 >> (l - 1), c.W >> (l - 1));
    if constexpr (l == 1) {
        if (c.out_lane && j >= c.A && j < c.B) {
            uint32_t w[2] = {0, 0};
            int orv = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int b = v[i] + 128;
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
        load_band<l - 1, NV>(hl, o, c, j, false, true);
        load_band<l - 1, NV>(lh, o, c, j, true, false);
        load_band<l - 1, NV>(hh, o, c, j, true, true);
        int sr[NV2], dr[NV2];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            sr[2 * i] = v[i];
            sr[2 * i + 1] = hl[i];
            dr[2 * i] = lh[i];
            dr[2 * i + 1] = hh[i];
        }
        inv_push<L, l - 1>(st, sr, dr, o, c);
    }
}

// Pair k of level l arrives: x_2k = s_k - (d_{k-1} + d_k + 2) >> 2, then
// x_{2k-1} = d_{k-1} + (x_{2k-2} + x_2k) >> 1; rows leave in order.
template <int L, int l>
__device__ __forceinline__ void inv_push(InvState& st, const int (&sr)[8 >> (l - 1)],
                                         const int (&dr)[8 >> (l - 1)], const InvOut& o, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = iline<l>(st);
    const int k = (st.kf >> l) + s.n;
    int x[NV];
    const bool first = s.n == 0;                                // d(-1) = d(0)
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i] = sr[i] - (((first ? dr[i] : s.D[i]) + dr[i] + 2) >> 2);
    if (!first) {
        int xo[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) xo[i] = s.D[i] + ((s.X[i] + x[i]) >> 1);
        inv_emit<L, l>(st, xo, 2 * k - 1, o, c);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        s.X[i] = x[i];
        s.D[i] = dr[i];
    }
    ++s.n;
    inv_emit<L, l>(st, x, 2 * k, o, c);
}

// last odd row of each level: x_{2K+2} = x_2K (reflection; exact at the matrix bottom)
template <int L, int l>
__device__ __forceinline__ void inv_finish(InvState& st, const InvOut& o, const StreamCtx& c) {
    constexpr int NV = 8 >> (l - 1);
    auto& s = iline<l>(st);
    if (s.n > 0) {
        int xo[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) xo[i] = s.D[i] + s.X[i];   // d + (2x >> 1)
        inv_emit<L, l>(st, xo, 2 * ((st.kf >> l) + s.n - 1) + 1, o, c);
    }
    if constexpr (l > 1) inv_finish<L, l - 1>(st, o, c);
}

template <int L>
__global__ void __launch_bounds__(kStreamThreads) k_dwt_full_inv(const __grid_constant__ DwtParams p,
                                                                 se_report* report, int seg, int ncg, int nseg) {
    using F = FStream<L>;
    constexpr int NV = 8 >> (L - 1), NH = NV / 2;
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
    for (int k = P0 >> L; k < (P1 >> L); ++k) {
        int ll[NH], hl[NH], lh[NH], hh[NH];
        load_band<L, NH>(ll, o, c, k, false, false);
        load_band<L, NH>(hl, o, c, k, false, true);
        load_band<L, NH>(lh, o, c, k, true, false);
        load_band<L, NH>(hh, o, c, k, true, true);
        int sr[NV], dr[NV];
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            sr[2 * i] = ll[i];
            sr[2 * i + 1] = hl[i];
            dr[2 * i] = lh[i];
            dr[2 * i + 1] = hh[i];
        }
        inv_push<L, L>(st, sr, dr, o, c);
    }
    inv_finish<L, L>(st, o, c);
}

template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, 4) k_protect_full(const __grid_constant__ FusedParams p) {
    protect_cta<L, MASK, 1>(p, blockIdx.x);
}

template <int L, bool MASK>
__global__ void __launch_bounds__(kBlocksPerCta, 4) k_recover_full(const __grid_constant__ FusedParams p) {
    recover_cta<L, MASK, 1>(p, blockIdx.x);
}

// ---------------------------------------------------------------- launchers

// Launch shape: warps = column groups x row segments; segments of 256 rows,
// halved (down to 32) until the grid holds enough warps to fill the SMs.
template <int L>
static void stream_shape(const DwtParams& p, int& seg, int& ncg, int& nseg, unsigned& grid) {
    using F = FStream<L>;
    ncg = (int)((p.width / 8 + F::USE - 1) / F::USE);
    const uint64_t rows = std::min<uint64_t>(p.row0 + p.rows_out, p.rows) - p.row0;
    seg = 256;
    while (seg > 32 && (uint64_t)ncg * ((rows + seg - 1) / seg) < 148ull * 48) seg /= 2;
    nseg = (int)((rows + seg - 1) / seg);
    grid = (unsigned)(((uint64_t)ncg * nseg + kStreamWarps - 1) / kStreamWarps);
}

template <int L>
static int full_fwd_l(const DwtParams& p, cudaStream_t s) {
    int seg, ncg, nseg;
    unsigned grid;
    stream_shape<L>(p, seg, ncg, nseg, grid);
    if (grid) k_dwt_full_fwd<L><<<grid, kStreamThreads, 0, s>>>(p, seg, ncg, nseg);
    return (int)cudaGetLastError();
}

template <int L>
static int full_inv_l(const DwtParams& p, se_report* rep, cudaStream_t s) {
    int seg, ncg, nseg;
    unsigned grid;
    stream_shape<L>(p, seg, ncg, nseg, grid);
    if (grid) k_dwt_full_inv<L><<<grid, kStreamThreads, 0, s>>>(p, rep, seg, ncg, nseg);
    return (int)cudaGetLastError();
}

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
