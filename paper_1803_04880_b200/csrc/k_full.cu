// k_full.cu — FULL-matrix mode (reading C1/C23).
//
// The paper transforms 8x8 blocks but notes the block size
// "can be changed"; FULL mode runs the same lifting (Eq. 5.1-5.2) over the
// whole W x R matrix, level by level, with whole-sample symmetric extension at
// each level's matrix borders, and stores the Mallat layout.  Fragments are
// then regrouped per 8x8 input footprint (4 / 12 / 48 coefficients at L = 2)
// and protected exactly like BLOCK8 records (fused_cta.cuh, MODE 1).
//
// Transform kernels: one CTA per 64 x 128 output tile.  The tile is loaded
// into shared memory with a halo of H = 2(2^L - 1) samples (rounded up to a
// multiple of 2^L so the lifting phase of the tile grid equals the global
// one): every 1-D lifting pass consumes 2 samples of its level on each side,
// so after L levels the tile interior is exact while the halo absorbs the
// error of the cut.  Lifting runs in place on the interleaved grid (level l
// touches every 2^(l-1)-th sample; even positions hold s, odd hold d), one
// shared-memory sweep per predict / update step; neighbours beyond the
// matrix border are reflected per level, neighbours beyond the halo are never
// read for interior outputs.  Coefficients move between the interleaved grid
// and the Mallat layout band by band, so global reads and writes are row
// segments (coalesced).
#include <cuda_runtime.h>

#include "fused_cta.cuh"

namespace se {

constexpr int kTileR = 64, kTileC = 128, kFullThreads = 512;

template <int L>
struct FullTile {
    static constexpr int H = L == 1 ? 4 : L == 2 ? 8 : 16;   // >= 2(2^L - 1), multiple of 2^L and of 4
    static constexpr int SR = kTileR + 2 * H, SC = kTileC + 2 * H;
    // the grid sits inside a margin of 2 s_max samples before and s_max + 1
    // after it (s_max = 2^(L-1)), so a lifting chunk's edge loads (forward
    // m = -2..8, inverse m = -1..9) never leave shared memory and need no
    // bounds test (values there only feed halo outputs)
    static constexpr int S_MAX = 1 << (L - 1), PAD_LO = 2 * S_MAX, PAD_HI = S_MAX + 1;
    static constexpr int P = (SC + PAD_LO + PAD_HI) | 1;      // odd pitch: row / column chunks in distinct banks
    static constexpr int ROWS = SR + PAD_LO + PAD_HI;
    static constexpr int OFF = PAD_LO * P + PAD_LO;           // grid origin inside the buffer
    static constexpr size_t smem = (size_t)ROWS * P * sizeof(int);
};

// One lifting pass of level spacing s along one direction of the tile
// (DIR 0: along rows, DIR 1: along columns), predict and update together.
// The active samples of a line are cut into chunks of 8 (4 even, 4 odd); a
// thread loads its chunk plus the samples the chunk edges need (forward:
// m = -2..8, so d(-1) of the previous chunk is recomputed from raw samples;
// inverse: m = -1..9), all threads load before any stores (one barrier), and
// the lifting runs in registers.  Consecutive threads take consecutive lines,
// which the odd row pitch puts in distinct banks.  Matrix borders: whole-sample
// symmetric extension per level (x(N) = x(N-2), d(-1) = d(0)); samples beyond
// the tile edge read 0 — they only feed halo outputs, which the halo of
// 2(2^L - 1) samples keeps away from the tile interior.
template <int L, int DIR, int s, bool INV>
__device__ __forceinline__ void lift_pass(int* g, int R0, int C0, int R, int W) {
    using T = FullTile<L>;
    constexpr int span = DIR == 0 ? T::SC : T::SR;            // along
    constexpr int nA = (DIR == 0 ? T::SR : T::SC) / s;         // active lines
    constexpr int nC = span / (8 * s);                         // chunks per line
    static_assert(span % (8 * s) == 0, "tile span must hold whole chunks");
    constexpr int items = nA * nC;
    constexpr int iters = (items + kFullThreads - 1) / kFullThreads;
    constexpr int step = DIR == 0 ? s : s * T::P;              // smem distance between active samples
    constexpr int m0 = INV ? -1 : -2;                          // first loaded sample
    const int O = DIR == 0 ? C0 : R0, N = DIR == 0 ? W : R;    // along: global origin, extent
    const int Oa = DIR == 0 ? R0 : C0, Na = DIR == 0 ? R : W;  // across
    static_assert(INV ? (s <= T::PAD_LO && s + 1 <= T::PAD_HI) : (2 * s <= T::PAD_LO && 1 <= T::PAD_HI),
                  "margin must cover the chunk edge loads");
    int v[iters][11];
#pragma unroll
    for (int it = 0; it < iters; ++it) {
        const int idx = threadIdx.x + it * kFullThreads;
        const int a = (idx % nA) * s, j0 = (idx / nA) * 8 * s;
        const int base = DIR == 0 ? a * T::P + j0 : j0 * T::P + a;
        const bool live = (items % kFullThreads == 0 || it + 1 < iters) || idx < items;
#pragma unroll
        for (int q = 0; q < 11; ++q) v[it][q] = live ? g[base + (q + m0) * step] : 0;   // margin: no bounds test
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < iters; ++it) {
        const int idx = threadIdx.x + it * kFullThreads;
        if (idx >= items) continue;
        const int a = (idx % nA) * s, j0 = (idx / nA) * 8 * s;
        const int ga = Oa + a;
        if (ga < 0 || ga >= Na) continue;                      // line outside the matrix
        const int base = DIR == 0 ? a * T::P + j0 : j0 * T::P + a;
        const int G0 = O + j0;                                 // global coordinate of m = 0
        int* x = v[it] - m0;                                   // x[m], m = m0 .. m0 + 10
        if (G0 - 2 * s >= 0 && G0 + 8 * s < N) {
            // interior chunk (every tile but those on the matrix border): no reflection, no store test
            if constexpr (!INV) {
#pragma unroll
                for (int m = -1; m <= 7; m += 2) x[m] -= (x[m - 1] + x[m + 1]) >> 1;
#pragma unroll
                for (int m = 0; m <= 6; m += 2) x[m] += (x[m - 1] + x[m + 1] + 2) >> 2;
            } else {
#pragma unroll
                for (int m = 0; m <= 8; m += 2) x[m] -= (x[m - 1] + x[m + 1] + 2) >> 2;
#pragma unroll
                for (int m = 1; m <= 7; m += 2) x[m] += (x[m - 1] + x[m + 1]) >> 1;
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) g[base + m * step] = x[m];
            continue;
        }
        if constexpr (!INV) {
            // predict (Eq. 5.1) at odd m = -1, 1, 3, 5, 7; right neighbour reflected at the border
#pragma unroll
            for (int m = -1; m <= 7; m += 2) {
                const int Gm = G0 + m * s;
                const int r = (Gm + s >= N) ? x[m - 1] : x[m + 1];
                x[m] -= (x[m - 1] + r) >> 1;
            }
            // update (Eq. 5.2, "+") at even m = 0, 2, 4, 6; d(-1) = d(0) at the left border
#pragma unroll
            for (int m = 0; m <= 6; m += 2) {
                const int Gm = G0 + m * s;
                const int l = (Gm == 0) ? x[m + 1] : x[m - 1];
                x[m] += (l + x[m + 1] + 2) >> 2;
            }
        } else {
            // undo update at even m = 0 .. 8, then undo predict at odd m = 1 .. 7
#pragma unroll
            for (int m = 0; m <= 8; m += 2) {
                const int Gm = G0 + m * s;
                const int l = (Gm == 0) ? x[m + 1] : x[m - 1];
                x[m] -= (l + x[m + 1] + 2) >> 2;
            }
#pragma unroll
            for (int m = 1; m <= 7; m += 2) {
                const int Gm = G0 + m * s;
                const int r = (Gm + s >= N) ? x[m - 1] : x[m + 1];
                x[m] += (x[m - 1] + r) >> 1;
            }
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int Gm = G0 + m * s;
            if (Gm >= 0 && Gm < N) g[base + m * step] = x[m];
        }
    }
    __syncthreads();
}

// Zero the margin around the grid (keeps the unused edge arithmetic defined).
template <int L>
__device__ __forceinline__ void zero_margin(int* buf) {
    using T = FullTile<L>;
    constexpr int top = T::PAD_LO * T::P, bot0 = (T::PAD_LO + T::SR) * T::P;
    constexpr int side = T::P - T::SC;                          // margin columns per grid row
    for (int i = threadIdx.x; i < top + T::PAD_LO; i += kFullThreads) buf[i] = 0;   // + row 0's left margin
    for (int i = threadIdx.x; i < T::ROWS * T::P - bot0; i += kFullThreads) buf[bot0 + i] = 0;
    for (int i = threadIdx.x; i < T::SR * side; i += kFullThreads) {
        const int r = i / side, c = i % side;                   // columns [SC, P) then wrap to [0, PAD_LO)
        const int col = T::PAD_LO + T::SC + c;                  // right margin + left margin of the next row
        buf[(T::PAD_LO + r) * T::P + col] = 0;
    }
}

// All levels, forward (l = 1..L: rows then columns) / inverse (l = L..1:
// columns then rows); the spacing s = 2^(l-1) is a compile-time constant.
template <int L, int l>
__device__ __forceinline__ void fwd_levels(int* g, int R0, int C0, int R, int W) {
    if constexpr (l <= L) {
        lift_pass<L, 0, 1 << (l - 1), false>(g, R0, C0, R, W);
        lift_pass<L, 1, 1 << (l - 1), false>(g, R0, C0, R, W);
        fwd_levels<L, l + 1>(g, R0, C0, R, W);
    }
}
template <int L, int l>
__device__ __forceinline__ void inv_levels(int* g, int R0, int C0, int R, int W) {
    if constexpr (l >= 1) {
        lift_pass<L, 1, 1 << (l - 1), true>(g, R0, C0, R, W);
        lift_pass<L, 0, 1 << (l - 1), true>(g, R0, C0, R, W);
        inv_levels<L, l - 1>(g, R0, C0, R, W);
    }
}

// Visit the Mallat band rectangles covered by a tile region: for level l and
// band (0 LL (l == L only), 1 HL, 2 LH, 3 HH), grid offset (pr, pc) of the
// band's samples inside each 2^l x 2^l cell and Mallat origin.
template <int L, typename F>
__device__ __forceinline__ void for_each_band(F&& f) {
#pragma unroll
    for (int l = 1; l <= L; ++l)
#pragma unroll
        for (int band = (l == L ? 0 : 1); band < 4; ++band) f(l, band);
}

template <int L>
__global__ void __launch_bounds__(kFullThreads) k_dwt_full_fwd(const __grid_constant__ DwtParams p) {
    using T = FullTile<L>;
    extern __shared__ int g_buf[];
    int* g = g_buf + T::OFF;                                    // grid origin inside the margin
    zero_margin<L>(g_buf);
    const int W = (int)p.width, R = (int)p.rows;
    const int row0 = (int)p.row0, row_end = min((int)(p.row0 + p.rows_out), R);
    const int s0 = (int)p.src_row0, s1 = (int)(p.src_row0 + p.src_rows);
    const int tr0 = row0 + (int)blockIdx.y * kTileR, tc0 = (int)blockIdx.x * kTileC;
    const int R0 = tr0 - T::H, C0 = tc0 - T::H;
    // load tile + halo, 4 bytes per access, centered (C8), zero fill past n
    // (C18); rows the caller did not provide (beyond a stripe's halo) read 0
    constexpr int WPR = T::SC / 4;
    for (int idx = threadIdx.x; idx < T::SR * WPR; idx += kFullThreads) {
        const int i = idx / WPR, w = idx % WPR;
        const int gr = R0 + i, gc = C0 + 4 * w;
        int v0 = 0, v1 = 0, v2 = 0, v3 = 0;
        if (gr >= 0 && gr < R && gc >= 0 && gc < W) {            // whole word inside (W % 8 == 0)
            const uint64_t o = (uint64_t)gr * W + gc;
            const bool have = gr >= s0 && gr < s1;
            if (have && o + 4 <= p.n_bytes) {
                const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(p.in + (uint64_t)(gr - s0) * W + gc));
                v0 = (int)(q & 0xff) - 128; v1 = (int)((q >> 8) & 0xff) - 128;
                v2 = (int)((q >> 16) & 0xff) - 128; v3 = (int)(q >> 24) - 128;
            } else {
                int t[4];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    t[b] = (o + b >= p.n_bytes) ? -128 : have ? (int)p.in[(uint64_t)(gr - s0) * W + gc + b] - 128 : 0;
                v0 = t[0]; v1 = t[1]; v2 = t[2]; v3 = t[3];
            }
        }
        int* d = g + i * T::P + 4 * w;
        d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3;
    }
    __syncthreads();
    fwd_levels<L, 1>(g, R0, C0, R, W);
    // write the tile interior band by band in Mallat layout
    for_each_band<L>([&](int l, int band) {
        const int hr = band >= 2, hc = band & 1, half = 1 << (l - 1);
        const int br = kTileR >> l, bc = kTileC >> l;          // band rectangle of this tile
        const int64_t mr0 = (hr ? ((int64_t)p.rows_out >> l) : 0) + ((tr0 - row0) >> l);   // local Mallat rows
        const int mc0 = (hc ? (W >> l) : 0) + (tc0 >> l);
        for (int idx = threadIdx.x; idx < br * bc; idx += kFullThreads) {
            const int bi = idx / bc, bj = idx % bc;
            const int gr = tr0 + (bi << l) + (hr ? half : 0);
            const int gc = tc0 + (bj << l) + (hc ? half : 0);
            if (gr >= row_end || gc >= W) continue;
            const int v = g[(gr - R0) * T::P + (gc - C0)];
            p.coef[(uint64_t)(mr0 + bi) * W + (mc0 + bj)] = (int16_t)v;
        }
    });
}

template <int L>
__global__ void __launch_bounds__(kFullThreads) k_dwt_full_inv(const __grid_constant__ DwtParams p,
                                                               se_report* report) {
    using T = FullTile<L>;
    extern __shared__ int g_buf[];
    int* g = g_buf + T::OFF;                                    // grid origin inside the margin
    zero_margin<L>(g_buf);
    __shared__ unsigned int s_badmask[(kTileR / 8) * (kTileC / 8) / 32];
    const int W = (int)p.width, R = (int)p.rows;
    const int row0 = (int)p.row0, row_end = min((int)(p.row0 + p.rows_out), R);
    const int tr0 = row0 + (int)blockIdx.y * kTileR, tc0 = (int)blockIdx.x * kTileC;
    const int R0 = tr0 - T::H, C0 = tc0 - T::H;
    for (int i = threadIdx.x; i < (kTileR / 8) * (kTileC / 8) / 32; i += kFullThreads) s_badmask[i] = 0;
    // gather tile + halo from the Mallat layout into the interleaved grid, band by band
    for_each_band<L>([&](int l, int band) {
        const int hr = band >= 2, hc = band & 1, half = 1 << (l - 1);
        // band samples whose grid position falls in [R0, R0+SR) x [C0, C0+SC)
        const int b_r0 = (R0 - (hr ? half : 0) + ((1 << l) - 1)) >> l;   // ceil, R0 may be negative
        const int b_c0 = (C0 - (hc ? half : 0) + ((1 << l) - 1)) >> l;
        const int nbr = (T::SR >> l) + 1, nbc = (T::SC >> l) + 1;
        // the source window holds band rows [src_row0 >> l, (src_row0 + src_rows) >> l)
        const int sb0 = (int)(p.src_row0 >> l), sbn = (int)(p.src_rows >> l);
        // rows of band samples inside the tile grid and the source window, then columns
        const int r_lo = max(max(b_r0, 0), sb0), r_hi = min(min(b_r0 + nbr, R >> l), sb0 + sbn);
        const int c_lo = max(b_c0, 0), c_hi = min(b_c0 + nbc, W >> l);
        const int nr = max(r_hi - r_lo, 0), nc = max(c_hi - c_lo, 0);
        const int16_t* src = p.coef + (hc ? (W >> l) : 0);
        const int64_t mrow0 = (hr ? sbn : 0) - sb0;
#pragma unroll 4
        for (int idx = threadIdx.x; idx < nr * nc; idx += kFullThreads) {
            const int bi = r_lo + idx / nc, bj = c_lo + idx % nc;
            const int gr = (bi << l) + (hr ? half : 0), gc = (bj << l) + (hc ? half : 0);
            if (gr >= R0 + T::SR || gc >= C0 + T::SC) continue;
            g[(gr - R0) * T::P + (gc - C0)] = __ldg(src + (uint64_t)(mrow0 + bi) * W + bj);
        }
    });
    __syncthreads();
    inv_levels<L, L>(g, R0, C0, R, W);
    // write bytes (+128), 4 per store; flag footprints with samples outside [0, 255]
    constexpr int WPR = kTileC / 4;
    for (int idx = threadIdx.x; idx < kTileR * WPR; idx += kFullThreads) {
        const int i = idx / WPR, w = idx % WPR;
        const int gr = tr0 + i, gc = tc0 + 4 * w;
        if (gr >= row_end || gc >= W) continue;
        const int* src = g + (i + T::H) * T::P + (4 * w + T::H);
        const int v0 = src[0] + 128, v1 = src[1] + 128, v2 = src[2] + 128, v3 = src[3] + 128;
        if ((v0 | v1 | v2 | v3) & ~0xff) {
            const int fp = (i / 8) * (kTileC / 8) + (4 * w) / 8;
            atomicOr(&s_badmask[fp / 32], 1u << (fp % 32));
        }
        const uint64_t o = (uint64_t)gr * W + gc;
        uint8_t* dst = p.out + (uint64_t)(gr - row0) * W + gc;
        if (o + 4 <= p.n_bytes) {
            *reinterpret_cast<uint32_t*>(dst) = (uint32_t)(v0 & 0xff) | (uint32_t)(v1 & 0xff) << 8 |
                                                (uint32_t)(v2 & 0xff) << 16 | (uint32_t)(v3 & 0xff) << 24;
        } else {
            const int vv[4] = {v0, v1, v2, v3};
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (o + b < p.n_bytes) dst[b] = (uint8_t)vv[b];
        }
    }
    if (report) {
        __syncthreads();
        const int nfp = (kTileR / 8) * (kTileC / 8);
        for (int fp = threadIdx.x; fp < nfp; fp += kFullThreads) {
            if (s_badmask[fp / 32] & (1u << (fp % 32))) {
                const int64_t fbr = tr0 / 8 + fp / (kTileC / 8), fbc = tc0 / 8 + fp % (kTileC / 8);
                if (fbr < row_end / 8 && fbc < W / 8) {                   // block index local to row0
                    const unsigned long long b = (unsigned long long)((fbr - row0 / 8) * (W / 8) + fbc);
                    atomicMin(reinterpret_cast<unsigned long long*>(&report->first_bad_block), b);
                    atomicAdd(reinterpret_cast<unsigned long long*>(&report->bad_blocks), 1ull);
                }
            }
        }
    }
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

template <int L>
static int full_fwd_l(const DwtParams& p, cudaStream_t s) {
    using T = FullTile<L>;
    cudaFuncSetAttribute(k_dwt_full_fwd<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::smem);
    const dim3 grid((unsigned)((p.width + kTileC - 1) / kTileC), (unsigned)((p.rows_out + kTileR - 1) / kTileR));
    k_dwt_full_fwd<L><<<grid, kFullThreads, T::smem, s>>>(p);
    return (int)cudaGetLastError();
}

template <int L>
static int full_inv_l(const DwtParams& p, se_report* rep, cudaStream_t s) {
    using T = FullTile<L>;
    cudaFuncSetAttribute(k_dwt_full_inv<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::smem);
    const dim3 grid((unsigned)((p.width + kTileC - 1) / kTileC), (unsigned)((p.rows_out + kTileR - 1) / kTileR));
    k_dwt_full_inv<L><<<grid, kFullThreads, T::smem, s>>>(p, rep);
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
