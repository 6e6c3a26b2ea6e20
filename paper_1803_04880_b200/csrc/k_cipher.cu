// k_cipher.cu — AES-128-CTR over an arbitrary byte range (cipher_encrypt /
// cipher_decrypt, row a6 as a standalone op and the paper's full-encryption
// comparator).  Lane-replicated T-table in 64 KB of
// dynamic shared memory (conflict-free lookups, se_device.cuh); one 16-byte
// counter block per thread per iteration, 128-bit coalesced loads/stores,
// grid sized to whole waves of the 148 SMs (2 CTAs of 1024 threads per SM).
#include <cuda_runtime.h>

#include "se_device.cuh"

namespace se {

#ifndef SE_LANE_THREADS
#define SE_LANE_THREADS 1024
#endif
constexpr int kLaneThreads = SE_LANE_THREADS;       // CTA size of the lane-table cipher (one 64 KB table per CTA)
// Keystream next to a fused kernel (grid-stride).  Wide: 256-thread CTAs, up
// to 8 per SM.  Narrow (SE_KS_NARROW=1 honours CipherParams::narrow, set by
// the masked protect): one 128-thread CTA per SM, so all 5 fused CTAs of
// every SM start at once beside it.  Measured on C2 (three A/B rounds):
// protect 186.3 vs 184.4 GB/s, but the recover that follows 186.0 vs 188.4 —
// round trip 93.1 vs 93.2, so off.
#ifndef SE_KS_NARROW
#define SE_KS_NARROW 0
#endif
constexpr int kKsThreads = 256, kKsNarrowThreads = 128;
constexpr int kKsNarrowCtasPerSm = 1;

// p.in == nullptr: write the keystream itself (used by the fused kernels,
// which then XOR it into the private fragment, see fused_cta.cuh).
// LANE: the 64 KB lane-replicated table (standalone cipher), else the 5 KB
// tables (keystream next to a running fused kernel).
#ifdef SE_TRACE
// diagnostic builds (tools/cta_trace.py): per CTA of the last keystream launch,
// SM id and %globaltimer at entry and exit
constexpr int kKsTraceMax = 4096;
__device__ unsigned long long g_trace_ks[3 * kKsTraceMax];
extern "C" int se_trace_ks_read(unsigned long long* host, int n_ctas) {
    if (n_ctas > kKsTraceMax) n_ctas = kKsTraceMax;
    return (int)cudaMemcpyFromSymbol(host, g_trace_ks, sizeof(unsigned long long) * 3 * n_ctas);
}
#endif

// SE_LUT4 1: the lane-table kernels use the 128 KB table with stored
// rotations (se_device.cuh aes_load_lut4), one CTA per SM.  Measured
// (tools/gpu_r2_call52.sh, two passes): AES-CTR comparator 788 -> 801 GB/s
// (the kernel is shared-memory-wavefront bound as much as ALU bound), C4
// masked 115.24 -> 115.36 GB/s, C5 107.53 -> 107.67 GB/s: 1.
#ifndef SE_CARVEOUT_MAX
#define SE_CARVEOUT_MAX 1      // as k_block8.cu: maximum shared-memory carveout
#endif
#ifndef SE_LUT4
#define SE_LUT4 1
#endif
constexpr int kLaneLutBytes = SE_LUT4 ? kAesLut4Bytes : kAesLutBytes;

template <bool LANE, int NT>
__global__ void __launch_bounds__(NT) k_cipher_ctr(const __grid_constant__ CipherParams p) {
#ifdef SE_TRACE
    unsigned long long tr0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
#endif
    // a dependent kernel launched with programmatic stream serialization may
    // start now; it waits (griddepcontrol.wait) before reading our output
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.report && blockIdx.x == 0 && threadIdx.x == 0) {
        p.report->first_bad_block = -1;
        p.report->bad_blocks = 0;
    }
    extern __shared__ __align__(16) uint32_t lut[];
    __shared__ AesSmem small;
    if constexpr (LANE) {
        if constexpr (SE_LUT4) aes_load_lut4(lut, threadIdx.x, NT);
        else aes_load_lut(lut, threadIdx.x, NT);
    } else {
        aes_load_tables(small, threadIdx.x, NT);
    }
    __syncthreads();
    const AesLane lane = aes_lane(lut);
    const uint64_t nblk = (p.n + 15) / 16;
    const uint64_t stride = (uint64_t)gridDim.x * NT;
    for (uint64_t j = (uint64_t)blockIdx.x * NT + threadIdx.x; j < nblk; j += stride) {
        uint32_t x[4];
        ctr_add(p.ctr, j, x);
        if constexpr (LANE && SE_LUT4) aes128_block4(lane, p.rk, x);
        else if constexpr (LANE) aes128_block(lane, p.rk, x);
        else aes128_block(small, p.rk, x);
        const uint64_t off = j * 16;
        if (p.cta_ablocks) {                  // scatter: keystream only, whole AES blocks (se_api.cu checks)
            const uint64_t cta = j / p.cta_ablocks, b0 = cta * kBlocksPerCta;
            const uint64_t br = b0 / p.bpr, bc = b0 - br * p.bpr;
            uint8_t* dst = p.out + 8 * br * (uint64_t)p.width + 8 * bc + 16 * (j - cta * p.cta_ablocks);
            *reinterpret_cast<uint4*>(dst) = make_uint4(bswap32(x[0]), bswap32(x[1]), bswap32(x[2]), bswap32(x[3]));
            continue;
        }
        if (off + 16 <= p.n) {
            const uint4 q = p.in ? __ldg(reinterpret_cast<const uint4*>(p.in + off)) : make_uint4(0, 0, 0, 0);
            uint4 r;
            r.x = q.x ^ bswap32(x[0]);
            r.y = q.y ^ bswap32(x[1]);
            r.z = q.z ^ bswap32(x[2]);
            r.w = q.w ^ bswap32(x[3]);
            *reinterpret_cast<uint4*>(p.out + off) = r;
        } else {
            for (uint64_t k = off; k < p.n; ++k) {
                const uint32_t w = x[(k - off) / 4];
                p.out[k] = (p.in ? p.in[k] : 0) ^ (uint8_t)(w >> (24 - 8 * ((k - off) % 4)));
            }
        }
    }
#ifdef SE_TRACE
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < kKsTraceMax) {
        unsigned long long tr1;
        unsigned sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace_ks[3 * blockIdx.x] = sm;
        g_trace_ks[3 * blockIdx.x + 1] = tr0;
        g_trace_ks[3 * blockIdx.x + 2] = tr1;
    }
#endif
}


// Keystream of every file's A stream in a batch (fragment_protect_batch):
// one thread per 16-byte counter block over all CTAs of the launch (a CTA's A
// slice is exactly ABITS counter blocks), written into each file's own A'
// buffer; the fused batch kernel follows with programmatic serialization and
// XORs its records in (no scratch).  Each warp owns one contiguous range of
// counter blocks, 32 per step: it finds the job of its first block once (a
// 32-ary search, 3 dependent loads at 10,000 jobs) and then only steps the
// job pointer forward as the range crosses file boundaries (round 2 did a
// 14-load binary search per warp and step: C5 3.13 ms, long-scoreboard bound).
#ifndef SE_BATCH_KS_RANGE
#define SE_BATCH_KS_RANGE 1
#endif
template <int ABITS>
__device__ __forceinline__ void batch_ks_block(const BatchParams& bp, const AesLane& lane, uint32_t jl, uint64_t idx) {
    const uint64_t cta = idx / ABITS, t = idx - cta * ABITS;
    const se_job& job = bp.jobs[jl];
    const uint64_t rows = ((job.n_bytes + job.width - 1) / job.width + 7) / 8 * 8;
    const uint64_t a_bytes = (rows / 8 * (job.width / 8) * ABITS + 7) / 8;
    const uint64_t lcta = cta - job.cta_begin;
    const uint64_t off = (lcta * ABITS + t) * 16;
    if (off >= a_bytes) return;
    uint8_t* dst = job.a + off;
    if (bp.base.ks_in_out) {        // recover: into the CTA's own output region, where it qualifies
        if (!batch_ks_out_cta(job.n_bytes, job.width, lcta, ABITS)) return;
        const uint64_t bpr = job.width / 8, b0 = lcta * kBlocksPerCta, br = b0 / bpr, bc = b0 - br * bpr;
        dst = job.out + 8 * br * (uint64_t)job.width + 8 * bc + 16 * t;
    }
    const JobDerived& dv = *reinterpret_cast<const JobDerived*>(job.derived);
    uint32_t x[4];
    ctr_add(dv.ctr, lcta * ABITS + t, x);
    if constexpr (SE_LUT4) aes128_block4(lane, bp.base.rk, x);
    else aes128_block(lane, bp.base.rk, x);
    if (off + 16 <= a_bytes || bp.base.ks_in_out) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(bswap32(x[0]), bswap32(x[1]), bswap32(x[2]), bswap32(x[3]));
    } else {
        for (uint64_t k = 0; k < a_bytes - off; ++k) dst[k] = (uint8_t)(x[k / 4] >> (24 - 8 * (k % 4)));
    }
}

// largest job j with cta_begin <= cta (jobs sorted; jobs[0].cta_begin == 0), by the whole warp
__device__ __forceinline__ uint32_t batch_job_of(const BatchParams& bp, uint64_t cta) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = 0, n = bp.n_jobs;                       // answer in [lo, lo + n)
    while (n > 1) {
        const uint32_t step = (n + 31) / 32;
        const uint32_t idx = lo + lane * step;
        const bool le = lane * step < n && bp.jobs[idx].cta_begin <= cta;
        const uint32_t m = __ballot_sync(0xffffffffu, le);
        const uint32_t k = 31 - __clz(m);
        lo += k * step;
        n = min(step, n - k * step);
    }
    return lo;
}

template <int ABITS>
__global__ void __launch_bounds__(kLaneThreads) k_batch_keystream(const __grid_constant__ BatchParams bp) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(16) uint32_t lut[];
    if constexpr (SE_LUT4) aes_load_lut4(lut, threadIdx.x, kLaneThreads);   // lane-replicated table (as k_cipher_ctr)
    else aes_load_lut(lut, threadIdx.x, kLaneThreads);
    __syncthreads();
    const AesLane lane = aes_lane(lut);
    const uint64_t total = bp.total_ctas * (uint64_t)ABITS;
#if SE_BATCH_KS_RANGE
    const uint32_t ln = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kLaneThreads / 32);
    const uint64_t gw = (uint64_t)blockIdx.x * (kLaneThreads / 32) + (threadIdx.x >> 5);
    const uint64_t per = ((total + nwarps - 1) / nwarps + 31) / 32 * 32;
    const uint64_t i0 = gw * per, i1 = min(total, i0 + per);
    if (i0 >= i1) return;
    uint32_t j = batch_job_of(bp, i0 / ABITS);
    uint64_t nb = j + 1 < bp.n_jobs ? bp.jobs[j + 1].cta_begin : ~0ull;   // first CTA of the next job
    for (uint64_t base = i0; base < i1; base += 32) {
        const uint64_t idx = base + ln;
        const uint64_t cta = idx / ABITS;
        uint32_t jl = j;
        uint64_t nbl = nb;
        while (cta >= nbl) {                                // crossed into a later file (rare)
            ++jl;
            nbl = jl + 1 < bp.n_jobs ? bp.jobs[jl + 1].cta_begin : ~0ull;
        }
        if (idx < i1) batch_ks_block<ABITS>(bp, lane, jl, idx);
        j = __shfl_sync(0xffffffffu, jl, 31);
        nb = ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(nbl >> 32), 31) << 32) |
             __shfl_sync(0xffffffffu, (uint32_t)nbl, 31);
    }
#else
    const uint64_t stride = (uint64_t)gridDim.x * kLaneThreads;
    for (uint64_t idx = (uint64_t)blockIdx.x * kLaneThreads + threadIdx.x; idx < total; idx += stride) {
        const uint64_t cta = idx / ABITS;
        uint32_t lo = 0, hi = bp.n_jobs - 1;                   // largest job with cta_begin <= cta
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) / 2;
            if (bp.jobs[mid].cta_begin <= cta) lo = mid;
            else hi = mid - 1;
        }
        batch_ks_block<ABITS>(bp, lane, lo, idx);
    }
#endif
}

// 64 KB of dynamic shared memory needs an opt-in, once per kernel and device
template <auto Kernel>
static void allow_lut() {
    static thread_local int done = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (done == dev) return;
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLaneLutBytes);
#if SE_CARVEOUT_MAX
    cudaFuncSetAttribute(Kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
#endif
    done = dev;
}

// Standalone cipher: 3 CTAs x 64 KB lane tables per SM.  Keystream for a
// fused kernel that runs concurrently (programmatic launch): 5 KB tables.
constexpr int kCipherCtasPerSm = 3;
constexpr int kKeystreamCtasPerSm = 8;


int launch_batch_keystream(const BatchParams& bp, uint32_t a_bits, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t total = bp.total_ctas * (uint64_t)a_bits;
    const uint64_t want = (total + kLaneThreads - 1) / kLaneThreads;
    const int lane_ctas = SE_LUT4 ? 1 : kCipherCtasPerSm < 2048 / kLaneThreads ? kCipherCtasPerSm : 2048 / kLaneThreads;
    const uint64_t cap = (uint64_t)sms * lane_ctas;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    cudaStream_t s = (cudaStream_t)stream;
    if (grid == 0) return 0;
    if (a_bits == 40) {
        allow_lut<k_batch_keystream<40>>();
        k_batch_keystream<40><<<grid, kLaneThreads, kLaneLutBytes, s>>>(bp);
    } else if (a_bits == 160) {
        allow_lut<k_batch_keystream<160>>();
        k_batch_keystream<160><<<grid, kLaneThreads, kLaneLutBytes, s>>>(bp);
    } else {
        allow_lut<k_batch_keystream<10>>();
        k_batch_keystream<10><<<grid, kLaneThreads, kLaneLutBytes, s>>>(bp);
    }
    note_launch();
    return (int)cudaGetLastError();
}

int launch_cipher_ctr(const CipherParams& p, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t nblk = (p.n + 15) / 16;
    const bool lane = p.in != nullptr || p.lane_lut;
    const bool narrow = SE_KS_NARROW && !lane && p.narrow;
    // lane table next to a fused kernel (p.narrow): one 128-thread CTA per SM,
    // whose 4 warps fit beside the fused kernel's 5 CTAs (registers), so no
    // SM holds back fused CTAs while the keystream runs
    const bool lane_narrow = lane && p.in == nullptr && p.narrow;
    const int nt = lane_narrow ? kKsNarrowThreads : lane ? kLaneThreads : narrow ? kKsNarrowThreads : kKsThreads;
    const uint64_t want = (nblk + nt - 1) / nt;
    // lane table: 64 KB per CTA -> at most 3 CTAs per SM, and 2048 threads per SM
    const int lane_ctas = SE_LUT4 ? 1 : kCipherCtasPerSm < 2048 / kLaneThreads ? kCipherCtasPerSm : 2048 / kLaneThreads;
    const uint64_t cap = (uint64_t)sms * (lane_narrow ? 1 : lane ? lane_ctas : narrow ? kKsNarrowCtasPerSm
                                                                                       : kKeystreamCtasPerSm);
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    if (grid == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (lane_narrow) {
        allow_lut<k_cipher_ctr<true, kKsNarrowThreads>>();
        k_cipher_ctr<true, kKsNarrowThreads><<<grid, kKsNarrowThreads, kLaneLutBytes, s>>>(p);
    } else if (lane) {
        allow_lut<k_cipher_ctr<true, kLaneThreads>>();
        k_cipher_ctr<true, kLaneThreads><<<grid, kLaneThreads, kLaneLutBytes, s>>>(p);
    } else if (narrow) {
        k_cipher_ctr<false, kKsNarrowThreads><<<grid, kKsNarrowThreads, 0, s>>>(p);
    } else {
        k_cipher_ctr<false, kKsThreads><<<grid, kKsThreads, 0, s>>>(p);
    }
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
