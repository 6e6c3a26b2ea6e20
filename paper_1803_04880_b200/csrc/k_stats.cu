// k_stats.cu — security-battery sums (NEXT row f2).
//
// One HBM pass over x and y: 256-bin histograms of both (per-warp private
// shared-memory counters, flushed once per CTA), the moments behind r_xy
// (Eq. 5.8), the bit difference popcount(x ^ y) (Dif, KS), the adjacent-pair
// sums of y read as a W-wide matrix (h / v / d correlation) and, optionally,
// the joint histogram for NMI (global atomics: 65536 bins, little contention).
// Every sum is an exact integer, so the device result must equal the oracle's
// bit for bit; the metrics are computed from the sums on the host.
#include <cuda_runtime.h>

#include "se_internal.h"

namespace se {

constexpr int kStatsThreads = 256;
constexpr int kStatsWarps = kStatsThreads / 32;

struct StatsParams {
    const uint8_t* x;     // nullable
    const uint8_t* y;
    uint64_t n;
    uint32_t width;
    se_stats* out;
    uint32_t* joint;      // nullable
};

__device__ __forceinline__ void warp_sum(unsigned long long& v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
}

__global__ void __launch_bounds__(kStatsThreads) k_stats(const __grid_constant__ StatsParams p) {
    __shared__ uint32_t hx[kStatsWarps][256], hy[kStatsWarps][256];
    __shared__ unsigned long long red[24];
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < kStatsWarps * 256; i += kStatsThreads) {
        (&hx[0][0])[i] = 0;
        (&hy[0][0])[i] = 0;
    }
    if (threadIdx.x < 24) red[threadIdx.x] = 0;
    __syncthreads();
    // per-thread accumulators: 0 sx 1 sy 2 sxx 3 syy 4 sxy 5 diff, 6.. adj[3][6]
    unsigned long long acc[24];
#pragma unroll
    for (int k = 0; k < 24; ++k) acc[k] = 0;
    const uint64_t W = p.width, n = p.n;
    const uint64_t segs_per_row = (W + 15) / 16;                 // 16-byte row segments
    const uint64_t n_segs = (n + W - 1) / W * segs_per_row;
    const uint64_t stride = (uint64_t)gridDim.x * kStatsThreads;
    for (uint64_t sg = (uint64_t)blockIdx.x * kStatsThreads + threadIdx.x; sg < n_segs; sg += stride) {
      const uint64_t row = sg / segs_per_row, c0 = (sg - row * segs_per_row) * 16;
      const uint64_t i0 = row * W + c0;
      const uint64_t i1 = min(min(i0 + 16, row * W + W), n);
      for (uint64_t i = i0; i < i1; ++i) {
        const uint32_t y = p.y[i];
        atomicAdd(&hy[warp][y], 1u);
        acc[1] += y;
        acc[3] += y * y;
        if (p.x) {
            const uint32_t x = p.x[i];
            atomicAdd(&hx[warp][x], 1u);
            acc[0] += x;
            acc[2] += x * x;
            acc[4] += x * y;
            acc[5] += __popc(x ^ y);
            if (p.joint) atomicAdd(&p.joint[x * 256 + y], 1u);
        }
        const uint64_t col = i - row * W;
        const bool right = col + 1 < W && i + 1 < n;
        const bool down = i + W < n;
        const bool diag = col + 1 < W && i + W + 1 < n;
        uint32_t b[3] = {0, 0, 0};
        const bool has[3] = {right, down, diag};
        if (right) b[0] = p.y[i + 1];
        if (down) b[1] = p.y[i + W];
        if (diag) b[2] = p.y[i + W + 1];
#pragma unroll
        for (int d = 0; d < 3; ++d)
            if (has[d]) {
                acc[6 + 6 * d + 0] += 1;
                acc[6 + 6 * d + 1] += y;
                acc[6 + 6 * d + 2] += b[d];
                acc[6 + 6 * d + 3] += y * y;
                acc[6 + 6 * d + 4] += b[d] * b[d];
                acc[6 + 6 * d + 5] += y * b[d];
            }
      }
    }
#pragma unroll
    for (int k = 0; k < 24; ++k) {
        warp_sum(acc[k]);
        if ((threadIdx.x & 31) == 0 && acc[k]) atomicAdd(&red[k], acc[k]);
    }
    __syncthreads();
    unsigned long long* o = reinterpret_cast<unsigned long long*>(p.out);
    // se_stats layout: n, hist_x[256], hist_y[256], sx, sy, sxx, syy, sxy, diff_bits, adj[18]
    for (int v = threadIdx.x; v < 256; v += kStatsThreads) {
        uint32_t sx = 0, sy = 0;
#pragma unroll
        for (int w = 0; w < kStatsWarps; ++w) { sx += hx[w][v]; sy += hy[w][v]; }
        if (sx) atomicAdd(&o[1 + v], (unsigned long long)sx);
        if (sy) atomicAdd(&o[1 + 256 + v], (unsigned long long)sy);
    }
    if (threadIdx.x < 24 && red[threadIdx.x]) atomicAdd(&o[1 + 512 + threadIdx.x], red[threadIdx.x]);
}

__global__ void k_stats_count(se_stats* s, uint64_t n) { s->n += n; }

int launch_stats(const void* x, const void* y, uint64_t n, uint32_t width, se_stats* out, uint32_t* joint,
                 void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    StatsParams p = {(const uint8_t*)x, (const uint8_t*)y, n, width, out, joint};
    const uint64_t want = (n + kStatsThreads - 1) / kStatsThreads;
    const unsigned grid = (unsigned)(want < (uint64_t)sms * 8 ? want : (uint64_t)sms * 8);
    cudaStream_t s = (cudaStream_t)stream;
    k_stats<<<grid, kStatsThreads, 0, s>>>(p);
    k_stats_count<<<1, 1, 0, s>>>(out, n);
    note_launch();
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
