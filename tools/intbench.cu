// intbench.cu — integer pipe microbenchmark for the roofline denominator
// (DESIGN.md §5): per-SM lane-op throughput of the SASS classes the SHA-2 /
// lifting code is made of, and whether ALU-pipe and FMA-pipe ops co-issue.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intbench intbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
constexpr int ITERS = 4096;

__device__ unsigned long long g_cycles[3 * 4096];   // per CTA: SM id, start, end (clock64)

template <int OP>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t seed, uint32_t one) {
    __syncthreads();
    const long long c0 = clock64();
    uint32_t x[CHAINS], y[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { x[c] = seed + threadIdx.x * 7 + c; y[c] = seed ^ (c * 0x9e3779b9u); }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (OP == 0) {          // SHF.R.W (funnel shift)
                asm volatile("shf.r.wrap.b32 %0, %0, %1, 13;" : "+r"(x[c]) : "r"(y[c]));
            } else if (OP == 1) {   // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(one));
            } else if (OP == 2) {   // IADD3 (two dependent adds fuse into IADD3)
                asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[c]) : "r"(y[c]), "r"(one));
            } else if (OP == 3) {   // IMAD
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(one), "r"(y[c]));
            } else if (OP == 4) {   // IMAD.WIDE.U32
                uint64_t w;
                asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(x[c]), "r"(one), "l"((uint64_t)y[c] << 32 | x[c]));
                x[c] = (uint32_t)w ^ (uint32_t)(w >> 32);
            } else if (OP == 5) {   // alternate SHF and IMAD on independent chains
                if (c & 1) asm volatile("shf.r.wrap.b32 %0, %0, %1, 13;" : "+r"(x[c]) : "r"(y[c]));
                else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(one), "r"(y[c]));
            } else if (OP == 6) {   // IMAD.HI.U32 (x >> k as a multiply)
                asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(one));
                x[c] += y[c];
            } else if (OP == 7) {   // PRMT
                asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(x[c]) : "r"(y[c]));
            } else if (OP == 8) {   // issue rate: LOP3 | IMAD | FFMA | LOP3 ... on independent chains
                if (c % 4 == 0 || c % 4 == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(one));
                else if (c % 4 == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(one), "r"(y[c]));
                else asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(x[c]) : "r"(y[c]));
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_cycles[3 * blockIdx.x] = sm;
        g_cycles[3 * blockIdx.x + 1] = (unsigned long long)c0;
        g_cycles[3 * blockIdx.x + 2] = (unsigned long long)clock64();
    }
}

template <int OP>
float run(uint32_t* d, int grid, const char* name, int sms, float ops_per_chain_iter) {
    k<OP><<<grid, 256>>>(d, 1, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 20; ++w) k<OP><<<grid, 256>>>(d, 1, 1);      // warm the clocks up
    cudaEventRecord(a);
    k<OP><<<grid, 256>>>(d, 1, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    static unsigned long long cyc[3 * 4096];
    const int nc = grid < 4096 ? grid : 4096;
    cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * 3 * nc);
    // per SM: its CTAs' lane ops over its busy window (first start .. last end,
    // clock64 is the SM's own cycle counter); averaged over SMs
    static unsigned long long lo[1024], hi[1024], cnt[1024];
    for (int i = 0; i < 1024; ++i) { lo[i] = ~0ull; hi[i] = 0; cnt[i] = 0; }
    for (int i = 0; i < nc; ++i) {
        const unsigned sm = (unsigned)cyc[3 * i] & 1023u;
        if (cyc[3 * i + 1] < lo[sm]) lo[sm] = cyc[3 * i + 1];
        if (cyc[3 * i + 2] > hi[sm]) hi[sm] = cyc[3 * i + 2];
        ++cnt[sm];
    }
    double sum_rate = 0;
    int nsm = 0;
    for (int i = 0; i < 1024; ++i)
        if (cnt[i]) { sum_rate += (double)cnt[i] * 256 * ITERS * CHAINS * ops_per_chain_iter / (double)(hi[i] - lo[i]); ++nsm; }
    double lane_ops = (double)grid * 256 * ITERS * CHAINS * ops_per_chain_iter;
    double per_s = lane_ops / (ms / 1e3);
    const double per_clk_sm = sum_rate / nsm;
    printf("{\"op\": \"%s\", \"ms\": %.4f, \"Tlane_ops_per_s\": %.3f, \"lane_ops_per_clk_per_sm\": %.2f, "
           "\"lane_ops_per_clk_per_sm_at_max_clock\": %.2f, \"effective_mhz\": %.0f}\n",
           name, ms, per_s / 1e12, per_clk_sm, per_s / sms / (clk_khz * 1e3), per_s / sms / per_clk_sm / 1e6);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int grid = sms * 8;
    uint32_t* d;
    cudaMalloc(&d, (size_t)grid * 256 * 4);
    run<0>(d, grid, "SHF.R.W", sms, 1);
    run<1>(d, grid, "LOP3", sms, 1);
    run<2>(d, grid, "IADD3", sms, 1);
    run<3>(d, grid, "IMAD", sms, 1);
    run<4>(d, grid, "IMAD.WIDE.U32(+LOP3)", sms, 1);
    run<5>(d, grid, "SHF|IMAD alternating", sms, 1);
    run<6>(d, grid, "IMAD.HI(+IADD)", sms, 1);
    run<7>(d, grid, "PRMT", sms, 1);
    run<8>(d, grid, "issue: LOP3|IMAD|LOP3|FFMA", sms, 1);
    printf("{\"sms\": %d}\n", sms);
    return 0;
}
