// k_block8.cu — fused BLOCK8 protect / recover kernels and the transform-only
// kernels (rows a1-a10 of SURVEY.md §8.1), sm_100a.
//
// Mapping: one thread owns one 8x8 block end to end; one CTA owns 128
// consecutive blocks (row-major block order).  Per CTA the fragment streams
// are contiguous and 16-byte aligned (A' 16*a_bits B, B' 16*b_bits B, C'
// 7680 B), so each CTA assembles its records in shared memory and writes
// them with 128-bit coalesced stores; the A stream of the CTA is exactly
// a_bits AES blocks, so the AES-CTR keystream for it is computed by the CTA
// itself, fused with the LL-band extraction: the private fragment never
// leaves the SM in plaintext and is never re-read from HBM.
//
// Loads: each thread issues 8 x 64-bit loads (one per block row); a warp's
// 32 consecutive blocks cover 256 contiguous bytes per row instruction.
#include <cuda_runtime.h>

#include "fused_cta.cuh"

#ifndef SE_MIN_CTAS
#define SE_MIN_CTAS 5      // resident 128-thread CTAs per SM the register budget must allow (96 regs)
#endif
// PUBLIC_PLAIN kernels (no SHA) are latency-bound: more resident warps pay
// (protect fits 72 registers without spills; recover holds more records)
#ifndef SE_MIN_CTAS_PLAIN_P
#define SE_MIN_CTAS_PLAIN_P 7
#endif
#ifndef SE_MIN_CTAS_PLAIN_R
#define SE_MIN_CTAS_PLAIN_R 6
#endif
#ifndef SE_MIN_CTAS_BATCH
#define SE_MIN_CTAS_BATCH 5
#endif
// batch kernels with the launch-constant SHA-512 schedule: its constants
// depend on K || IV, so fragment_batch_plan derives them per file
#ifndef SE_BATCH_SPEC
#define SE_BATCH_SPEC 1
#endif

namespace se {

// ---------------------------------------------------------------- kernels

// Blocks (threads) per CTA of the single-file kernels.  Finer CTAs spread
// a file more evenly over the SMs (C2: 1536 CTAs of 128 leave each SM 10 or 11
// of them, ~10 % idle at the end; 64-block CTAs halve that).  The CTA's
// stream slices must stay whole 16-byte units: L = 3 (155-bit B records)
// keeps 128.
#ifndef SE_BPC
#define SE_BPC 128
#endif
template <int L>
__host__ __device__ constexpr int bpc_for() { return L == 3 ? kBlocksPerCta : SE_BPC; }
// resident CTAs per SM the masked kernels' register budget must allow
#ifndef SE_MINB_MASK
#define SE_MINB_MASK(bpc) (SE_MIN_CTAS * kBlocksPerCta / (bpc))
#endif

// SE_TRACE (diagnostic builds only, tools/cta_trace.py): per CTA, the SM id
// and %globaltimer at entry and exit, read back with se_trace_read.
#ifdef SE_TRACE
constexpr int kTraceMax = 1 << 16;
__device__ unsigned long long g_trace[3 * kTraceMax];
struct CtaTrace {
    unsigned long long t0;
    __device__ CtaTrace() {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    __device__ ~CtaTrace() {
        __syncthreads();
        if (threadIdx.x == 0 && blockIdx.x < kTraceMax) {
            unsigned long long t1;
            unsigned sm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_trace[3 * blockIdx.x] = sm;
            g_trace[3 * blockIdx.x + 1] = t0;
            g_trace[3 * blockIdx.x + 2] = t1;
        }
    }
};
#define SE_CTA_TRACE CtaTrace trace_;
#else
#define SE_CTA_TRACE
#endif

template <int L, bool MASK>
__global__ void __launch_bounds__(bpc_for<L>(), MASK ? SE_MINB_MASK(bpc_for<L>()) : SE_MIN_CTAS_PLAIN_P * kBlocksPerCta / bpc_for<L>())
k_protect_block8(const __grid_constant__ FusedParams p) {
    SE_CTA_TRACE
    protect_cta<L, MASK, 0, bpc_for<L>(), true, SE_SHA256_BODY_P>(p, blockIdx.x);
}

template <int L, bool MASK>
__global__ void __launch_bounds__(bpc_for<L>(), MASK ? SE_MINB_MASK(bpc_for<L>()) : SE_MIN_CTAS_PLAIN_R * kBlocksPerCta / bpc_for<L>())
k_recover_block8(const __grid_constant__ FusedParams p) {
    SE_CTA_TRACE
    recover_cta<L, MASK, 0, bpc_for<L>(), true, SE_SPEC_REC256 != 0>(p, blockIdx.x);
}

// Many independent files in one launch (C5; SURVEY §8.6 "sharded by file").
// A unit is one CTA's worth of a file (128 blocks; a file's last unit may be
// partial).  Job parameters are assembled in shared memory (the per-job
// counter base and SHA midstates were derived on the host by
// fragment_batch_plan) and the same CTA body runs on them.
//
// One CTA per unit.  Measured and dropped (C5, tools/gpu_r2_call46.sh /
// call47.sh): persistent CTAs, 5 per SM, that find the job once per range and
// then only step the job pointer — contiguous per-CTA ranges 98.9 GB/s,
// grid-strided chunks of 2 / 4 / 8 / 16 units 98.9 / 99.8 / 100.6 / 101.2,
// against 107.7 for one CTA per unit.

template <int L>
__device__ __forceinline__ void batch_job_params(FusedParams& sp, const BatchParams& bp, uint32_t jb) {
    using R = Rec<L>;
    const se_job& job = bp.jobs[jb];
    const JobDerived& dv = *reinterpret_cast<const JobDerived*>(job.derived);
    const uint32_t t = threadIdx.x;
    if (t == 0) {
        sp.in = job.in;
        sp.out = job.out;
        sp.a = job.a; sp.b = job.b; sp.c = job.c;
        sp.report = bp.reports ? bp.reports + jb : nullptr;
        sp.n_bytes = job.n_bytes;
        sp.width = job.width;
        sp.bpr = job.width / 8;
        const uint64_t rows = ((job.n_bytes + job.width - 1) / job.width + 7) / 8 * 8;
        sp.n_blocks = rows / 8 * sp.bpr;
        sp.block_offset = job.block_offset;
        sp.a_bytes = (sp.n_blocks * R::ABITS + 7) / 8;
        sp.b_bytes = (sp.n_blocks * R::BBITS + 7) / 8;
        sp.c_bytes = (sp.n_blocks * R::CBITS + 7) / 8;
    } else if (t >= 32 && t < 36) {
        sp.ctr[t - 32] = dv.ctr[t - 32];
    } else if (t >= 36 && t < 44) {
        sp.kiv[t - 36] = dv.kiv[t - 36];
    } else if (t >= 44 && t < 52) {
        sp.mid256[t - 44] = dv.mid256[t - 44];
    } else if (t >= 52 && t < 60) {
        sp.mid512[t - 52] = dv.mid512[t - 52];
    }
    if (SE_BATCH_SPEC && t >= 64) {                  // this file's C-mask schedule constants
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&dv.s512);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&sp.s512);
        for (uint32_t i = t - 64; i < sizeof(SchedConst512) / 4; i += kBlocksPerCta - 64) dst[i] = src[i];
    }
}

// largest job j with cta_begin <= unit (jobs sorted, jobs[0].cta_begin == 0),
// by one warp: 32 ways, one candidate per lane (3 dependent passes at 10,000
// jobs).  SE_BATCH_SEARCH_WAYS 128 (4 candidates per lane, 2 passes) measured
// slower on C5: 106.7 vs 107.8 GB/s (tools/gpu_r2_call49.sh).
#ifndef SE_BATCH_SEARCH_WAYS
#define SE_BATCH_SEARCH_WAYS 32
#endif
__device__ __forceinline__ uint32_t batch_find_job(const BatchParams& bp, uint64_t unit) {
    constexpr uint32_t Q = SE_BATCH_SEARCH_WAYS / 32;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = 0, n = bp.n_jobs;                   // answer in [lo, lo + n)
    while (n > 1) {
        const uint32_t step = (n + 32 * Q - 1) / (32 * Q);
        uint32_t trues = 0;                           // candidates c = lane * Q + q, sorted: a prefix is true
#pragma unroll
        for (uint32_t q = 0; q < Q; ++q) {
            const uint32_t c = lane * Q + q;
            const bool le = c * step < n && bp.jobs[lo + c * step].cta_begin <= unit;
            trues += __popc(__ballot_sync(0xffffffffu, le));
        }
        const uint32_t k = trues - 1;                 // candidate 0 always true
        lo += k * step;
        n = min(step, n - k * step);
    }
    return lo;
}

template <int L, bool MASK, bool RECOVER>
__global__ void __launch_bounds__(kBlocksPerCta, SE_MIN_CTAS_BATCH)
k_batch_block8(const __grid_constant__ BatchParams bp) {
    __shared__ FusedParams sp;
    __shared__ uint32_t s_job;
    using R = Rec<L>;
    // job table / report init written by earlier work; with the keystream kernel
    // right before (protect, base.ks_in_a: a normal launch, so everything
    // earlier is complete) only its keystream is waited for, at the copy-out
    // (recover with base.ks_in_out likewise: report init and jobs precede the
    // keystream kernel; qualifying CTAs wait for their keystream before use)
    if (!bp.base.ks_in_a && !bp.base.ks_in_out) asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t x = blockIdx.x;
    if (threadIdx.x < 32) {
        const uint32_t jb = batch_find_job(bp, x);
        if (threadIdx.x == 0) s_job = jb;
    }
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&bp.base);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&sp);
        for (uint32_t i = threadIdx.x; i < sizeof(FusedParams) / 4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const se_job& job = bp.jobs[s_job];
    batch_job_params<L>(sp, bp, s_job);
    if (bp.base.ks_in_out && threadIdx.x == 0)         // this CTA's keystream parked in its output region, or not
        sp.ks_in_out = batch_ks_out_cta(job.n_bytes, job.width, x - job.cta_begin, R::ABITS) ? 1u : 0u;
    __syncthreads();
    const uint64_t cta = x - job.cta_begin;
    if (RECOVER) recover_cta<L, MASK, 0, kBlocksPerCta, SE_BATCH_SPEC != 0>(sp, cta);
    else protect_cta<L, MASK, 0, kBlocksPerCta, SE_BATCH_SPEC != 0>(sp, cta);
}

__global__ void k_report_init(se_report* r, uint32_t n) {
    asm volatile("griddepcontrol.launch_dependents;");
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { r[i].first_bad_block = -1; r[i].bad_blocks = 0; }
}

int launch_report_init(se_report* r, uint32_t n, void* stream) {
    carveout_max_once((const void*)k_report_init);
    k_report_init<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(r, n);
    note_launch();
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- transform only

template <int L>
__global__ void __launch_bounds__(kBlocksPerCta) k_dwt_fwd_block8(const __grid_constant__ DwtParams p) {
    const uint64_t blk = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (blk >= p.n_blocks) return;
    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
    int v[8][8];
    load_block(p.in, p.n_bytes, p.width, br, bc, v);
    dwt8_fwd<L>(v, p.one);
#pragma unroll
    for (int i = 0; i < (8 >> L); ++i)
#pragma unroll
        for (int j = 0; j < (8 >> L); ++j) v[i][j] -= 128;     // centering (C8) lands on LL_L only
    int16_t* base = p.coef + 8 * br * (uint64_t)p.width + 8 * bc;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint4 q;
        q.x = (uint32_t)(v[i][0] & 0xffff) | ((uint32_t)v[i][1] << 16);
        q.y = (uint32_t)(v[i][2] & 0xffff) | ((uint32_t)v[i][3] << 16);
        q.z = (uint32_t)(v[i][4] & 0xffff) | ((uint32_t)v[i][5] << 16);
        q.w = (uint32_t)(v[i][6] & 0xffff) | ((uint32_t)v[i][7] << 16);
        *reinterpret_cast<uint4*>(base + (uint64_t)i * p.width) = q;
    }
}

template <int L>
__global__ void __launch_bounds__(kBlocksPerCta) k_dwt_inv_block8(const __grid_constant__ DwtParams p) {
    const uint64_t blk = (uint64_t)blockIdx.x * kBlocksPerCta + threadIdx.x;
    if (blk >= p.n_blocks) return;
    const uint64_t br = blk / p.bpr, bc = blk - br * p.bpr;
    const int16_t* base = p.coef + 8 * br * (uint64_t)p.width + 8 * bc;
    int v[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)i * p.width));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[i][2 * k] = (int)(int16_t)(w[k] & 0xffff);
            v[i][2 * k + 1] = (int)(int16_t)(w[k] >> 16);
        }
    }
#pragma unroll
    for (int i = 0; i < (8 >> L); ++i)
#pragma unroll
        for (int j = 0; j < (8 >> L); ++j) v[i][j] += 128;
    dwt8_inv<L>(v, p.one);
    store_block(p.out, p.n_bytes, p.width, br, bc, v);
}

// ---------------------------------------------------------------- launchers

#ifdef SE_TRACE
extern "C" int se_trace_read(unsigned long long* host, int n_ctas) {
    if (n_ctas > kTraceMax) n_ctas = kTraceMax;
    return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * 3 * n_ctas);
}
#endif

// Launch with programmatic stream serialization: the kernel may start while
// the preceding keystream kernel (k_cipher_ctr) still runs; it synchronises
// with griddepcontrol.wait where it needs the keystream (fused_cta.cuh).
// SE_CARVEOUT_MAX 1: ask for the maximum shared-memory carveout on the fused
// kernels (and the lane-table keystream kernels, k_cipher.cu), so kernels
// that follow each other on a stream never need an L1 / shared-memory
// reconfiguration of the SMs between them.  Measured (tools/gpu_r2_call55.sh,
// two passes): C2 93.0 -> 93.3, C3 110.5 -> 111.3, C4 115.61 -> 115.79 GB/s: 1.
#ifndef SE_CARVEOUT_MAX
#define SE_CARVEOUT_MAX 1
#endif
void carveout_max_once(const void* kernel) {
#if SE_CARVEOUT_MAX
    static thread_local const void* seen[128];
    static thread_local int n_seen = 0, seen_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != seen_dev) { n_seen = 0; seen_dev = dev; }
    for (int i = 0; i < n_seen; ++i)
        if (seen[i] == kernel) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (n_seen < 128) seen[n_seen++] = kernel;
#else
    (void)kernel;
#endif
}

template <typename P>
static void carveout_once(void (*kernel)(P)) {
    carveout_max_once((const void*)kernel);
}

template <typename P>
void launch_pdl(void (*kernel)(P), unsigned grid, unsigned block, cudaStream_t s, const P& p) {
    carveout_once(kernel);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, p);
}
template void launch_pdl<FusedParams>(void (*)(FusedParams), unsigned, unsigned, cudaStream_t, const FusedParams&);
template void launch_pdl<DctParams>(void (*)(DctParams), unsigned, unsigned, cudaStream_t, const DctParams&);

static unsigned grid_for(uint64_t n_blocks, int bpc = kBlocksPerCta) {
    return (unsigned)((n_blocks + bpc - 1) / bpc);
}

template <int L>
static void protect_l(const FusedParams& p, bool mask, cudaStream_t s) {
    constexpr int B = bpc_for<L>();
    if (mask) launch_pdl(k_protect_block8<L, true>, grid_for(p.n_blocks, B), B, s, p);
    else launch_pdl(k_protect_block8<L, false>, grid_for(p.n_blocks, B), B, s, p);
}
template <int L>
static void recover_l(const FusedParams& p, bool mask, cudaStream_t s) {
    constexpr int B = bpc_for<L>();
    if (mask) launch_pdl(k_recover_block8<L, true>, grid_for(p.n_blocks, B), B, s, p);
    else launch_pdl(k_recover_block8<L, false>, grid_for(p.n_blocks, B), B, s, p);
}

int launch_protect_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) protect_l<1>(p, mask, s);
    else if (levels == 2) protect_l<2>(p, mask, s);
    else protect_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

int launch_recover_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (levels == 1) recover_l<1>(p, mask, s);
    else if (levels == 2) recover_l<2>(p, mask, s);
    else recover_l<3>(p, mask, s);
    note_launch();
    return (int)cudaGetLastError();
}

template <int L, bool RECOVER>
static void batch_l(const BatchParams& bp, uint64_t ctas, bool mask, cudaStream_t s) {
    if (mask) launch_pdl(k_batch_block8<L, true, RECOVER>, (unsigned)ctas, kBlocksPerCta, s, bp);
    else launch_pdl(k_batch_block8<L, false, RECOVER>, (unsigned)ctas, kBlocksPerCta, s, bp);
}

int launch_batch_block8(const BatchParams& bp, uint64_t total_ctas, uint32_t levels, bool mask, bool recover,
                        void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (recover && bp.reports && !bp.reports_ready) {
        carveout_max_once((const void*)k_report_init);
        k_report_init<<<(bp.n_jobs + 255) / 256, 256, 0, s>>>(bp.reports, bp.n_jobs);
        note_launch();
    }
    if (total_ctas == 0) return (int)cudaGetLastError();
    if (recover) {
        if (levels == 1) batch_l<1, true>(bp, total_ctas, mask, s);
        else if (levels == 2) batch_l<2, true>(bp, total_ctas, mask, s);
        else batch_l<3, true>(bp, total_ctas, mask, s);
    } else {
        if (levels == 1) batch_l<1, false>(bp, total_ctas, mask, s);
        else if (levels == 2) batch_l<2, false>(bp, total_ctas, mask, s);
        else batch_l<3, false>(bp, total_ctas, mask, s);
    }
    note_launch();
    return (int)cudaGetLastError();
}

int launch_dwt_fwd_block8(const DwtParams& p, uint32_t levels, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = grid_for(p.n_blocks);
    if (levels == 1) k_dwt_fwd_block8<1><<<g, kBlocksPerCta, 0, s>>>(p);
    else if (levels == 2) k_dwt_fwd_block8<2><<<g, kBlocksPerCta, 0, s>>>(p);
    else k_dwt_fwd_block8<3><<<g, kBlocksPerCta, 0, s>>>(p);
    note_launch();
    return (int)cudaGetLastError();
}

int launch_dwt_inv_block8(const DwtParams& p, uint32_t levels, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = grid_for(p.n_blocks);
    if (levels == 1) k_dwt_inv_block8<1><<<g, kBlocksPerCta, 0, s>>>(p);
    else if (levels == 2) k_dwt_inv_block8<2><<<g, kBlocksPerCta, 0, s>>>(p);
    else k_dwt_inv_block8<3><<<g, kBlocksPerCta, 0, s>>>(p);
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace se
