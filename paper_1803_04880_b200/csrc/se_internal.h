// se_internal.h — kernel parameter blocks and launcher prototypes shared by
// the host API (se_api.cu) and the kernel translation units.  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/se.h"
#include "../../include/se_dct.h"

// NVTX ranges around every public entry point (host side: the range covers
// argument checks and the enqueue of the call's kernels / copies), so
// profilers show library calls on the timeline and `ncu --nvtx
// --nvtx-include "fragment_protect/"` selects one call's kernels.  Header-only
// NVTX3: no cost beyond a predicted branch when no tool is attached.
#ifndef SE_NVTX
#define SE_NVTX 1
#endif
#if SE_NVTX
#include <nvtx3/nvToolsExt.h>
namespace se {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace se
#define SE_RANGE(name) ::se::NvtxRange se_nvtx_range_(name)
#else
#define SE_RANGE(name) ((void)0)
#endif

namespace se {

constexpr int kBlocksPerCta = 128;   // one thread per 8x8 block, 128 blocks per CTA


// ---- message-schedule specialisation of the B / C mask hashes (sha2_spec.cuh)
// bit t set: schedule word W_t depends on the block (t < 64)
__host__ __device__ constexpr uint64_t sched_var(uint32_t msg_mask) {
    uint64_t v = msg_mask;
    for (int t = 16; t < 64; ++t)
        if (((v >> (t - 2)) | (v >> (t - 7)) | (v >> (t - 15)) | (v >> (t - 16))) & 1u) v |= 1ull << t;
    return v;
}
// block-dependent message words: SHA-512 over K||IV||be64(b)||record (64-bit
// words: b is word 4, record bytes from byte 40), SHA-256 over the same
// framing (32-bit words: b is words 8, 9)
__host__ __device__ constexpr uint32_t msg_var512(int rec_bytes) {
    uint32_t m = 1u << 4;
    for (int w = 5; w <= (40 + rec_bytes - 1) / 8; ++w) m |= 1u << w;
    return m;
}
__host__ __device__ constexpr uint32_t msg_var256(int rec_bytes) {
    uint32_t m = (1u << 8) | (1u << 9);
    for (int w = 10; w <= (40 + rec_bytes - 1) / 4; ++w) m |= 1u << w;
    return m;
}
// block-independent schedule data of one launch (host-computed):
// c[t-16] for t = 16..31 = W_t if block-independent, else the sum of its
// block-independent terms; kw[t] = K_t + W_t for block-independent W_t, t < 32
struct SchedConst512 {
    uint64_t c[16];
    uint64_t kw[32];
};
struct SchedConst256 {
    uint32_t c[16];
    uint32_t kw[32];
};

// Everything a fused protect/recover launch needs (passed by value; lives in
// the constant bank, so round keys and midstates are uniform operands).
struct FusedParams {
    const uint8_t* in;        // protect: input bytes; recover: unused
    uint8_t* out;             // recover: output bytes
    uint8_t* a;               // A' stream
    uint8_t* b;               // B' stream
    uint8_t* c;               // C' stream
    se_report* report;        // recover only, nullable
    int16_t* ws;              // FULL mode: R x W Mallat coefficient workspace
    uint64_t rows;            // R (FULL mode)
    uint64_t n_bytes;
    uint64_t n_blocks;
    uint64_t block_offset;    // global index of local block 0 (hash nonce, C16)
    uint64_t a_bytes, b_bytes, c_bytes;
    uint64_t n_tiles;         // k_tile.cu: tiles of the launch
    uint64_t fast_tiles;      // k_tile.cu: leading tiles moved by bulk copies (the rest: per-thread path)
    uint32_t width;
    uint32_t bpr;             // 8x8 blocks per block-row = width / 8
    uint32_t one;             // = 1, opaque to ptxas: adds become IMADs (sha2_device.cuh)
    uint32_t bpr_magic;       // k_tile.cu: ceil(2^20 / bpr) (block row of a tile-local block)
    uint32_t ks_in_a;         // per-CTA protect: A' already holds the keystream (k_cipher_ctr before)
    uint32_t ks_in_out;       // per-CTA recover, keystream written by k_cipher_ctr just before: 1 = each
                              // CTA's A slice at the start of its own output region (scatter mode),
                              // 2 = the whole A stream at the start of out (FULL mode: out is written
                              // only by the inverse transform afterwards)
    uint32_t ctr[4];          // IV + block_offset*a_bits/128, big-endian words
    uint32_t rk[44];          // AES-128 round keys, big-endian words
    uint32_t kiv[8];          // K || IV as big-endian words (SHA W0..W7)
    uint32_t mid256[8];       // SHA-256 state after rounds 0..7 over K||IV
    uint32_t h256[8];         // SHA-256 H(0)
    uint64_t mid512[8];       // SHA-512 state after rounds 0..3 over K||IV
    uint64_t h512[8];         // SHA-512 H(0)
    SchedConst512 s512;       // C-mask schedule constants (single-file / FULL kernels)
    SchedConst256 s256;       // B-mask schedule constants
};

// Batch recover, keystream parked in the output (k_batch_keystream with
// base.ks_in_out): CTA `cta` of a job qualifies when its first row run is a
// whole 1024-byte row segment inside the file that holds the CTA's A slice.
__host__ __device__ inline bool batch_ks_out_cta(uint64_t n_bytes, uint32_t width, uint64_t cta, uint32_t a_bits) {
    if (width % 1024 != 0 || a_bits * kBlocksPerCta / 8 > 1024) return false;
    const uint64_t bpr = width / 8, b0 = cta * kBlocksPerCta, br = b0 / bpr, bc = b0 - br * bpr;
    return 8 * br * (uint64_t)width + 8 * bc + a_bits * kBlocksPerCta / 8 <= n_bytes;
}

// Library-private layout of se_job.derived[] (filled by fragment_batch_plan).
struct JobDerived {
    uint32_t ctr[4];          // IV + block_offset*a_bits/128
    uint32_t kiv[8];          // K || IV words
    uint32_t mid256[8];       // SHA-256 midstate over K||IV
    uint64_t mid512[8];       // SHA-512 midstate over K||IV
    SchedConst512 s512;       // C-mask schedule constants of this file's K||IV (sha2_spec.cuh)
};
static_assert(sizeof(JobDerived) <= sizeof(((se_job*)0)->derived), "se_job.derived too small");

struct BatchParams {
    const se_job* jobs;       // device array, sorted by cta_begin
    se_report* reports;       // recover: one per job, nullable
    uint64_t total_ctas;
    uint32_t n_jobs;
    uint32_t reports_ready;   // recover: reports already initialised (no init kernel in the launcher)
    FusedParams base;         // shared fields: rk, h256, h512, one
};

struct CipherParams {
    const uint8_t* in;
    uint8_t* out;
    uint64_t n;
    uint32_t ctr[4];          // IV + ctr_block_offset
    uint32_t rk[44];
    uint32_t lane_lut;        // keystream (in == nullptr) with the 64 KB lane table
    uint32_t narrow;          // keystream: one 128-thread CTA per SM (k_cipher.cu)
    se_report* report;        // nullable: initialised to {-1, 0} by this kernel (the fused recover
                              // kernel that follows updates it only after griddepcontrol.wait)
    // scatter mode (cta_ablocks != 0): AES block j goes to the output region of
    // recover CTA i = j / cta_ablocks (128 blocks per CTA): out + 8*br*W + 8*bc
    // of its first 8x8 block (br, bc), + 16 * (j % cta_ablocks)
    uint32_t cta_ablocks;
    uint32_t bpr;
    uint32_t width;
};

struct DwtParams {
    const uint8_t* in;
    uint8_t* out;
    int16_t* coef;
    uint64_t n_bytes;         // of the whole file
    uint64_t n_blocks;
    uint32_t width;
    uint32_t bpr;
    uint32_t rows;            // R of the whole matrix (border reflection)
    uint32_t one;             // = 1, opaque to ptxas (see FusedParams::one)
    // FULL-mode row window (whole file: 0, R, 0, R).  Output rows
    // [row0, row0 + rows_out): Mallat bands of these rows only (forward) or
    // these bytes (inverse), at local offsets.  Source rows [src_row0,
    // src_row0 + src_rows): input bytes at in[(r - src_row0) * W] (forward) or
    // the local Mallat layout of their coefficients in coef (inverse).
    uint64_t row0, rows_out, src_row0, src_rows;
};

// Chapter 4 DCT 8x8 SE (row f3, k_dct.cu).  One thread per 8x8 block
// position (all channels), 128 positions per CTA.
struct DctParams {
    const uint8_t* in;        // protect: image; recover: Fragment 2 (P')
    uint8_t* out;             // protect: Fragment 2; recover: rebuilt image
    uint8_t* a;               // Fragment 1 stream (protect: holds the keystream on entry)
    const uint8_t* ks;        // recover: keystream of Fragment 1 (scratch)
    float* coef;              // dct_select: records x 6; dct8_forward/inverse: coefficient image
    uint64_t n_pos;           // block positions (W/8)*(H/8)
    uint64_t a_bytes;
    uint64_t block_offset;    // global record index of record 0 (KEYED nonce)
    uint32_t width;           // pixels per row
    uint32_t bpr;             // block positions per block row = width / 8
    uint32_t one;             // = 1, opaque to ptxas (sha2_device.cuh)
    uint32_t pad_;
    uint32_t kiv[8];          // K || IV words (KEYED)
    uint64_t mid512[8];       // SHA-512 state after rounds 0..3 over K||IV (KEYED)
    uint64_t h512[8];         // SHA-512 H(0)
    SchedConst512 s512;       // level-2 mask schedule constants (sha2_spec.cuh)
    uint32_t ctr[4];          // Fragment-1 AES-CTR: IV + block_offset*66/128 (fused AES)
    uint32_t rk[44];          // AES-128 round keys
};
// whether the DCT kernel of `op` (0 protect, 1 recover) runs the AES of
// Fragment 1 itself (k_dct.cu) instead of a keystream kernel before it
bool dct_fused_aes(int op, uint32_t level, uint64_t n_pos);
// message words of the level-2 hash that depend on the record: unkeyed rec9
// (words 0, 1), keyed K||IV||be64(r)||rec9 (words 4, 5, 6)
constexpr uint32_t kDctMsgUnkeyed = 0x3u;
constexpr uint32_t kDctMsgKeyed = 0x70u;
void dct_sched_consts(DctParams& p, bool keyed);

// host helpers shared by the API translation units (se_api.cu)
void cipher_setup(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block, CipherParams& cp);
void sha512_kiv(const uint8_t key[16], const uint8_t iv[16], uint32_t kiv[8], uint64_t mid[8], uint64_t h0[8]);
// options of the shared protect / recover implementation (se_api.cu)
struct ImplOpts {
    bool mapped = false;          // BLOCK8 buffers in page-locked host memory (se_host.cu): per-CTA kernels
    bool report_ready = false;    // recover: the report is already {-1, 0}
    void* ws = nullptr;           // FULL mode: caller workspace (fragment_workspace_size)
    uint64_t ws_bytes = 0;
};
constexpr uint64_t kMaxBlocks = 1ull << 32;     // 8x8 blocks per call (256 GiB)
int protect_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in, void* d_a,
                 void* d_b, void* d_c, const ImplOpts& o, void* stream);
int recover_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a, const void* d_b,
                 const void* d_c, void* d_out, se_report* d_report, const ImplOpts& o, void* stream);

// launchers (return cudaError_t as int)
int launch_protect_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream);
int launch_recover_block8(const FusedParams& p, uint32_t levels, bool mask, void* stream);
// persistent warp-specialised single-file kernels (k_tile.cu)
int launch_tile_block8(const FusedParams& p, uint32_t levels, bool mask, bool recover, void* stream);
int launch_batch_block8(const BatchParams& bp, uint64_t total_ctas, uint32_t levels, bool mask, bool recover,
                        void* stream);
int launch_batch_keystream(const BatchParams& bp, uint32_t a_bits, void* stream);   // into each job's A'
int launch_dwt_fwd_block8(const DwtParams& p, uint32_t levels, void* stream);
// the maximum shared-memory carveout for a kernel, once per device (k_block8.cu, SE_CARVEOUT_MAX)
void carveout_max_once(const void* kernel);
int launch_report_init(se_report* r, uint32_t n, void* stream);   // {-1, 0} x n
// FULL mode (row a11): whole-matrix transform kernels and the footprint CTA kernels
int launch_dwt_full_fwd(const DwtParams& p, uint32_t levels, void* stream);
int launch_dwt_full_inv(const DwtParams& p, uint32_t levels, se_report* report, void* stream);
int launch_protect_full(const FusedParams& p, uint32_t levels, bool mask, void* stream);
int launch_recover_full(const FusedParams& p, uint32_t levels, bool mask, void* stream);
int launch_dwt_inv_block8(const DwtParams& p, uint32_t levels, void* stream);
int launch_cipher_ctr(const CipherParams& p, void* stream);

int launch_dct(const DctParams& p, uint32_t channels, uint32_t level, bool keyed, int op, void* stream);  // op 0 protect, 1 recover, 2 select, 3 dct8 fwd, 4 dct8 inv

int launch_stats(const void* x, const void* y, uint64_t n, uint32_t width, se_stats* out, uint32_t* joint,
                 void* stream);

void note_launch();
template <typename P>
void launch_pdl(void (*kernel)(P), unsigned grid, unsigned block, cudaStream_t s, const P& p);

}  // namespace se
