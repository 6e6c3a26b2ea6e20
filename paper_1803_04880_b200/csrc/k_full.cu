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
    static constexpr int H = L == 1 ? 2 : L == 2 ? 8 : 16;   // >= 2(2^L - 1), multiple of 2^L
    static constexpr int SR = kTileR + 2 * H, SC = kTileC + 2 * H;
    static constexpr size_t smem = (size_t)SR * SC * sizeof(int);
};

// One lifting step over the tile grid along one direction.
//   DIR 0: rows (neighbours at j +- s), DIR 1: columns (i +- s)
//   STEP 0: predict (odd level positions), 1: update (even positions),
//   INV: the inverse step (undo update = STEP 1, undo predict = STEP 0)
template <int L, int DIR, int STEP, bool INV, int s>
__device__ __forceinline__ void lift_sweep(int* g, int64_t R0, int64_t C0, int64_t R, int64_t W) {
    using T = FullTile<L>;
    // positions: along DIR, index ≡ (STEP == 0 ? s : 0) mod 2s; across DIR, ≡ 0 mod s
    const int nA = DIR == 0 ? T::SR / s : T::SC / s;             // across
    const int nL = DIR == 0 ? T::SC / (2 * s) : T::SR / (2 * s); // along (one parity)
    const int64_t N = DIR == 0 ? W : R;                           // signal extent (samples of level 1)
    const int64_t O = DIR == 0 ? C0 : R0;
    const int64_t Oa = DIR == 0 ? R0 : C0, Na = DIR == 0 ? R : W;
    const int span = DIR == 0 ? T::SC : T::SR;
    for (int idx = threadIdx.x; idx < nA * nL; idx += blockDim.x) {
        // consecutive threads: along a row (DIR 0) or across columns (DIR 1),
        // so a warp's shared-memory accesses fall in distinct banks
        const int a = (DIR == 0 ? idx / nL : idx % nA) * s;                        // across coordinate
        const int k = (DIR == 0 ? idx % nL : idx / nA) * 2 * s + (STEP == 0 ? s : 0);   // along coordinate
        const int64_t ga = Oa + a, gk = O + k;
        if (ga < 0 || ga >= Na || gk < 0 || gk >= N) continue;    // outside the matrix
        int lo = k - s, hi = k + s;
        if (STEP == 0) {                               // odd position: neighbours are even samples
            if (gk + s >= N) hi = k - s;               // x(N) = x(N-2)
        } else {                                       // even position: neighbours are d's
            if (gk - s < 0) lo = k + s;                // d(-1) = d(0)
        }
        if (lo < 0 || hi >= span) continue;            // halo edge: output not needed
        auto at = [&](int kk) -> int& { return DIR == 0 ? g[a * T::SC + kk] : g[kk * T::SC + a]; };
        int& x = at(k);
        const int nb = at(lo) + at(hi);
        if (STEP == 0) x = INV ? x + (nb >> 1) : x - (nb >> 1);            // Eq. 5.1
        else x = INV ? x - ((nb + 2) >> 2) : x + ((nb + 2) >> 2);          // Eq. 5.2 (+)
    }
}

// All levels, forward (l = 1..L) / inverse (l = L..1); the sample spacing
// s = 2^(l-1) is a compile-time constant so the sweep index arithmetic folds.
template <int L, int l>
__device__ __forceinline__ void fwd_levels(int* g, int64_t R0, int64_t C0, int64_t R, int64_t W) {
    if constexpr (l <= L) {
        constexpr int s = 1 << (l - 1);
        lift_sweep<L, 0, 0, false, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 0, 1, false, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 1, 0, false, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 1, 1, false, s>(g, R0, C0, R, W); __syncthreads();
        fwd_levels<L, l + 1>(g, R0, C0, R, W);
    }
}
template <int L, int l>
__device__ __forceinline__ void inv_levels(int* g, int64_t R0, int64_t C0, int64_t R, int64_t W) {
    if constexpr (l >= 1) {
        constexpr int s = 1 << (l - 1);
        lift_sweep<L, 1, 1, true, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 1, 0, true, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 0, 1, true, s>(g, R0, C0, R, W); __syncthreads();
        lift_sweep<L, 0, 0, true, s>(g, R0, C0, R, W); __syncthreads();
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
    extern __shared__ int g[];
    const int64_t W = p.width, R = p.rows;
    const int64_t row0 = (int64_t)p.row0, row_end = min((int64_t)(p.row0 + p.rows_out), R);
    const int64_t s0 = (int64_t)p.src_row0, s1 = (int64_t)(p.src_row0 + p.src_rows);
    const int64_t tr0 = row0 + (int64_t)blockIdx.y * kTileR, tc0 = (int64_t)blockIdx.x * kTileC;
    const int64_t R0 = tr0 - T::H, C0 = tc0 - T::H;
    // load tile + halo, centered (C8), zero fill past n (C18); rows the caller
    // did not provide (beyond a stripe's halo) only feed outputs not written
    for (int idx = threadIdx.x; idx < T::SR * T::SC; idx += blockDim.x) {
        const int i = idx / T::SC, j = idx % T::SC;
        const int64_t gr = R0 + i, gc = C0 + j;
        int v = 0;
        if (gr >= 0 && gr < R && gc >= 0 && gc < W) {
            const uint64_t o = (uint64_t)gr * W + gc;
            if (o >= p.n_bytes) v = -128;                                   // zero fill (C18)
            else if (gr >= s0 && gr < s1) v = (int)p.in[(uint64_t)(gr - s0) * W + gc] - 128;
        }
        g[idx] = v;
    }
    __syncthreads();
    fwd_levels<L, 1>(g, R0, C0, R, W);
    // write the tile interior band by band in Mallat layout
    for_each_band<L>([&](int l, int band) {
        const int hr = band >= 2, hc = band & 1, half = 1 << (l - 1);
        const int br = kTileR >> l, bc = kTileC >> l;        // band rectangle of this tile
        const int64_t mr0 = (hr ? ((int64_t)p.rows_out >> l) : 0) + ((tr0 - row0) >> l);   // local Mallat rows
        const int64_t mc0 = (hc ? (W >> l) : 0) + (tc0 >> l);
        for (int idx = threadIdx.x; idx < br * bc; idx += blockDim.x) {
            const int bi = idx / bc, bj = idx % bc;
            const int64_t gr = tr0 + ((int64_t)bi << l) + (hr ? half : 0);
            const int64_t gc = tc0 + ((int64_t)bj << l) + (hc ? half : 0);
            if (gr >= row_end || gc >= W) continue;
            const int v = g[(gr - R0) * T::SC + (gc - C0)];
            p.coef[(uint64_t)(mr0 + bi) * W + (mc0 + bj)] = (int16_t)v;
        }
    });
}

template <int L>
__global__ void __launch_bounds__(kFullThreads) k_dwt_full_inv(const __grid_constant__ DwtParams p,
                                                               se_report* report) {
    using T = FullTile<L>;
    extern __shared__ int g[];
    __shared__ unsigned int s_badmask[(kTileR / 8) * (kTileC / 8) / 32];
    const int64_t W = p.width, R = p.rows;
    const int64_t row0 = (int64_t)p.row0, row_end = min((int64_t)(p.row0 + p.rows_out), R);
    const int64_t tr0 = row0 + (int64_t)blockIdx.y * kTileR, tc0 = (int64_t)blockIdx.x * kTileC;
    const int64_t R0 = tr0 - T::H, C0 = tc0 - T::H;
    for (int i = threadIdx.x; i < (kTileR / 8) * (kTileC / 8) / 32; i += blockDim.x) s_badmask[i] = 0;
    // gather tile + halo from the Mallat layout into the interleaved grid, band by band
    for_each_band<L>([&](int l, int band) {
        const int hr = band >= 2, hc = band & 1, half = 1 << (l - 1);
        // band samples whose grid position falls in [R0, R0+SR) x [C0, C0+SC)
        const int64_t b_r0 = (R0 - (hr ? half : 0) + ((1 << l) - 1)) >> l;   // ceil, R0 may be negative
        const int64_t b_c0 = (C0 - (hc ? half : 0) + ((1 << l) - 1)) >> l;
        const int nbr = (T::SR >> l) + 1, nbc = (T::SC >> l) + 1;
        // the source window holds band rows [src_row0 >> l, (src_row0 + src_rows) >> l)
        const int64_t sb0 = (int64_t)p.src_row0 >> l, sbn = (int64_t)p.src_rows >> l;
        for (int idx = threadIdx.x; idx < nbr * nbc; idx += blockDim.x) {
            const int64_t bi = b_r0 + idx / nbc, bj = b_c0 + idx % nbc;
            if (bi < 0 || bj < 0 || bi >= (R >> l) || bj >= (W >> l)) continue;
            if (bi < sb0 || bi >= sb0 + sbn) continue;            // beyond a stripe's halo: unused
            const int64_t gr = (bi << l) + (hr ? half : 0), gc = (bj << l) + (hc ? half : 0);
            if (gr < R0 || gr >= R0 + T::SR || gc < C0 || gc >= C0 + T::SC) continue;
            const int64_t mr = (hr ? sbn : 0) + (bi - sb0), mc = (hc ? (W >> l) : 0) + bj;
            g[(gr - R0) * T::SC + (gc - C0)] = p.coef[(uint64_t)mr * W + mc];
        }
    });
    __syncthreads();
    inv_levels<L, L>(g, R0, C0, R, W);
    // write bytes (+128), flag footprints with samples outside [0, 255]
    for (int idx = threadIdx.x; idx < kTileR * kTileC; idx += blockDim.x) {
        const int i = idx / kTileC, j = idx % kTileC;
        const int64_t gr = tr0 + i, gc = tc0 + j;
        if (gr >= row_end || gc >= W) continue;
        const int v = g[(i + T::H) * T::SC + (j + T::H)] + 128;
        if (v & ~0xff) {
            const int fp = (i / 8) * (kTileC / 8) + (j / 8);
            atomicOr(&s_badmask[fp / 32], 1u << (fp % 32));
        }
        const uint64_t o = (uint64_t)gr * W + gc;
        if (o < p.n_bytes) p.out[(uint64_t)(gr - row0) * W + gc] = (uint8_t)v;
    }
    if (report) {
        __syncthreads();
        const int nfp = (kTileR / 8) * (kTileC / 8);
        for (int fp = threadIdx.x; fp < nfp; fp += blockDim.x) {
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
