// se_api.cu — host side of libse.so: the C ABI declared in include/se.h.
//
// Validates geometry, derives everything that is the same
// for every block once on the host — AES-128 key schedule (FIPS-197 §5.2),
// the CTR start counter (C13), and the SHA-256 / SHA-512 midstates over the
// constant message prefix K||IV (C15) — and launches the fused kernels on the
// caller's stream.  No device allocation, no synchronisation on the hot path:
// FULL mode takes a caller-owned workspace (fragment_workspace_size).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>

#include "se_internal.h"
#include "../../include/se_container.h"
#include "tables.h"

namespace se {

static thread_local uint64_t t_launches = 0;
void note_launch() { ++t_launches; }

static const uint8_t kSbox[256] = SE_AES_SBOX_INIT;
static const uint32_t kK256[64] = SE_SHA256_K_INIT;
static const uint32_t kH256[8] = SE_SHA256_H0_INIT;
static const uint64_t kK512[80] = SE_SHA512_K_INIT;
static const uint64_t kH512[8] = SE_SHA512_H0_INIT;

static uint32_t be32(const uint8_t* p) {
    return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | p[3];
}

// FIPS-197 §5.2 KeyExpansion (Nk = 4, Nr = 10), big-endian words.
static void key_expansion(const uint8_t key[16], uint32_t rk[44]) {
    for (int i = 0; i < 4; ++i) rk[i] = be32(key + 4 * i);
    uint32_t rcon = 0x01;
    for (int i = 4; i < 44; ++i) {
        uint32_t t = rk[i - 1];
        if (i % 4 == 0) {
            t = (t << 8) | (t >> 24);                                        // RotWord
            t = (uint32_t)kSbox[t >> 24] << 24 | (uint32_t)kSbox[(t >> 16) & 0xff] << 16 |
                (uint32_t)kSbox[(t >> 8) & 0xff] << 8 | kSbox[t & 0xff];     // SubWord
            t ^= rcon << 24;
            rcon = ((rcon << 1) ^ ((rcon & 0x80) ? 0x1b : 0)) & 0xff;
        }
        rk[i] = rk[i - 4] ^ t;
    }
}

static uint32_t ror32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
static uint64_t ror64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

// SHA-256 rounds 0..7 over W0..W7 = K||IV (FIPS 180-4 §6.2.2 step 3).
static void sha256_mid(const uint32_t w[8], uint32_t st[8]) {
    uint32_t a = kH256[0], b = kH256[1], c = kH256[2], d = kH256[3];
    uint32_t e = kH256[4], f = kH256[5], g = kH256[6], h = kH256[7];
    for (int t = 0; t < 8; ++t) {
        const uint32_t t1 = h + (ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25)) + ((e & f) ^ (~e & g)) + kK256[t] + w[t];
        const uint32_t t2 = (ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// SHA-512 rounds 0..3 over W0..W3 = K||IV (FIPS 180-4 §6.4.2 step 3).
static void sha512_mid(const uint64_t w[4], uint64_t st[8]) {
    uint64_t a = kH512[0], b = kH512[1], c = kH512[2], d = kH512[3];
    uint64_t e = kH512[4], f = kH512[5], g = kH512[6], h = kH512[7];
    for (int t = 0; t < 4; ++t) {
        const uint64_t t1 = h + (ror64(e, 14) ^ ror64(e, 18) ^ ror64(e, 41)) + ((e & f) ^ (~e & g)) + kK512[t] + w[t];
        const uint64_t t2 = (ror64(a, 28) ^ ror64(a, 34) ^ ror64(a, 39)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// 128-bit big-endian IV + j (SP 800-38A counter), as 4 big-endian words.
static void ctr_base(const uint8_t iv[16], uint64_t j, uint32_t out[4]) {
    uint64_t hi = (uint64_t)be32(iv) << 32 | be32(iv + 4);
    uint64_t lo = (uint64_t)be32(iv + 8) << 32 | be32(iv + 12);
    const uint64_t nlo = lo + j;
    if (nlo < lo) ++hi;
    out[0] = (uint32_t)(hi >> 32); out[1] = (uint32_t)hi;
    out[2] = (uint32_t)(nlo >> 32); out[3] = (uint32_t)nlo;
}

void cipher_setup(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block, CipherParams& cp) {
    ctr_base(iv, ctr_block, cp.ctr);
    key_expansion(key, cp.rk);
}

void sha512_kiv(const uint8_t key[16], const uint8_t iv[16], uint32_t kiv[8], uint64_t mid[8], uint64_t h0[8]) {
    for (int i = 0; i < 4; ++i) { kiv[i] = be32(key + 4 * i); kiv[4 + i] = be32(iv + 4 * i); }
    uint64_t w[4];
    for (int i = 0; i < 4; ++i) w[i] = (uint64_t)kiv[2 * i] << 32 | kiv[2 * i + 1];
    sha512_mid(w, mid);
    memcpy(h0, kH512, sizeof kH512);
}

static void record_bits(uint32_t L, uint32_t mode, uint32_t bits[3]) {
    // BLOCK8 (C21, C22) / FULL (C23): A, B, C bits per block
    if (L == 1) { bits[0] = 160; bits[1] = 0; bits[2] = 480; return; }
    if (L == 2) { bits[0] = 40; bits[1] = mode ? 132 : 124; bits[2] = 480; return; }
    bits[0] = 10; bits[1] = mode ? 165 : 155; bits[2] = 480;
}

static int check_geom(const se_geom* g) {
    if (!g) return SE_EINVAL;
    if (g->width == 0 || g->width % 8) return SE_EINVAL;
    if (g->levels < 1 || g->levels > 3) return SE_EINVAL;
    if (g->mode > SE_MODE_FULL) return SE_EINVAL;
    if (g->flags & ~(uint32_t)(SE_FLAG_PUBLIC_PLAIN | SE_FLAG_HOST_MAPPED)) return SE_EINVAL;
    return SE_OK;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// FIPS 180-4 §4.1.2 / §4.1.3 small sigmas
static uint32_t s0_256(uint32_t x) { return ror32(x, 7) ^ ror32(x, 18) ^ (x >> 3); }
static uint32_t s1_256(uint32_t x) { return ror32(x, 17) ^ ror32(x, 19) ^ (x >> 10); }
static uint64_t s0_512(uint64_t x) { return ror64(x, 1) ^ ror64(x, 8) ^ (x >> 7); }
static uint64_t s1_512(uint64_t x) { return ror64(x, 19) ^ ror64(x, 61) ^ (x >> 6); }

// Block-independent schedule data (sha2_spec.cuh) for message words w[16]
// whose block-dependent words (mask) are ignored.
template <typename T, typename S0, typename S1>
static void sched_consts(uint32_t mask, const T w[16], const T* K, S0 s0, S1 s1, T c[16], T kw[32]) {
    const uint64_t V = sched_var(mask);
    auto var = [&](int t) { return ((V >> t) & 1u) != 0; };
    T W[32];
    for (int t = 0; t < 16; ++t) W[t] = var(t) ? 0 : w[t];
    for (int t = 16; t < 32; ++t) {
        T part = 0;
        if (!var(t - 2)) part += s1(W[t - 2]);
        if (!var(t - 7)) part += W[t - 7];
        if (!var(t - 15)) part += s0(W[t - 15]);
        if (!var(t - 16)) part += W[t - 16];
        W[t] = var(t) ? 0 : part;
        c[t - 16] = part;                        // == W_t when no term depends on the block
    }
    for (int t = 0; t < 32; ++t) kw[t] = var(t) ? 0 : (T)(K[t] + W[t]);
}

// level-2 DCT mask (k_dct.cu): the 9-byte record alone, or K||IV||be64(r)||rec9
void dct_sched_consts(DctParams& p, bool keyed) {
    uint64_t w[16] = {0};
    if (keyed) {
        for (int i = 0; i < 4; ++i) w[i] = (uint64_t)p.kiv[2 * i] << 32 | p.kiv[2 * i + 1];
        w[6] = 0x80ull << 48;                    // pad at byte 49 (a record word; kept for clarity)
        w[15] = 49 * 8;
        sched_consts<uint64_t>(kDctMsgKeyed, w, kK512, s0_512, s1_512, p.s512.c, p.s512.kw);
    } else {
        w[15] = 9 * 8;
        sched_consts<uint64_t>(kDctMsgUnkeyed, w, kK512, s0_512, s1_512, p.s512.c, p.s512.kw);
    }
}

static void fill_sched(FusedParams& p, const se_layout& lay) {
    const int L = lay.b_bits == 0 ? 1 : 2;       // L = 1: the C mask hashes A; else B', B from A
    // SHA-512 of the C mask: K||IV||be64(b)||record, record = B' (L >= 2) or A (L = 1)
    const int sb = (int)((L == 1 ? lay.a_bits : lay.b_bits) + 7) / 8;
    uint64_t w5[16] = {0};
    for (int i = 0; i < 4; ++i) w5[i] = (uint64_t)p.kiv[2 * i] << 32 | p.kiv[2 * i + 1];
    w5[(40 + sb) / 8] |= 0x80ull << (56 - 8 * ((40 + sb) % 8));         // FIPS 180-4 §5.1.2
    w5[15] = (uint64_t)(40 + sb) * 8;
    sched_consts<uint64_t>(msg_var512(sb), w5, kK512, s0_512, s1_512, p.s512.c, p.s512.kw);
    if (lay.b_bits) {                            // SHA-256 of the B mask: K||IV||be64(b)||A
        const int ab = (int)(lay.a_bits + 7) / 8;
        uint32_t w2[16] = {0};
        for (int i = 0; i < 8; ++i) w2[i] = p.kiv[i];
        w2[(40 + ab) / 4] |= 0x80u << (24 - 8 * ((40 + ab) % 4));      // FIPS 180-4 §5.1.1
        w2[15] = (uint32_t)(40 + ab) * 8;
        sched_consts<uint32_t>(msg_var256(ab), w2, kK256, s0_256, s1_256, p.s256.c, p.s256.kw);
    }
}

static void fill_fused(FusedParams& p, const se_geom* g, const se_layout& lay, const uint8_t key[16],
                       const uint8_t iv[16]) {
    memset(&p, 0, sizeof p);
    p.n_bytes = g->n_bytes;
    p.n_blocks = lay.n_blocks;
    p.block_offset = g->block_offset;
    p.a_bytes = lay.a_bytes; p.b_bytes = lay.b_bytes; p.c_bytes = lay.c_bytes;
    p.width = g->width;
    p.bpr = g->width / 8;
    p.one = 1;
    ctr_base(iv, g->block_offset * lay.a_bits / 128, p.ctr);
    key_expansion(key, p.rk);
    for (int i = 0; i < 4; ++i) { p.kiv[i] = be32(key + 4 * i); p.kiv[4 + i] = be32(iv + 4 * i); }
    sha256_mid(p.kiv, p.mid256);
    memcpy(p.h256, kH256, sizeof kH256);
    uint64_t w[4];
    for (int i = 0; i < 4; ++i) w[i] = (uint64_t)p.kiv[2 * i] << 32 | p.kiv[2 * i + 1];
    sha512_mid(w, p.mid512);
    memcpy(p.h512, kH512, sizeof kH512);
    fill_sched(p, lay);
}

}  // namespace se

using namespace se;

extern "C" {

const char* se_strerror(int s) {
    switch (s) {
        case SE_OK: return "ok";
        case SE_EINVAL: return "invalid argument";
        case SE_EALIGN: return "device pointer not 16-byte aligned";
        case SE_ECUDA: return "CUDA error";
        case SE_ENOTSUP: return "not supported";
        case SE_EFORMAT: return "bad container format";
        case SE_EINTEGRITY: return "container stream digest mismatch";
        default: return "unknown status";
    }
}

uint64_t se_launch_count(int reset) {
    const uint64_t v = t_launches;
    if (reset) t_launches = 0;
    return v;
}

int fragment_layout(const se_geom* g, se_layout* out) {
    int rc = check_geom(g);
    if (rc) return rc;
    if (!out) return SE_EINVAL;
    uint32_t bits[3];
    record_bits(g->levels, g->mode, bits);
    const uint64_t R = ((g->n_bytes + g->width - 1) / g->width + 7) / 8 * 8;
    const uint64_t nb = (R / 8) * (g->width / 8);
    out->rows = R;
    out->n_blocks = nb;
    out->a_bits = bits[0]; out->b_bits = bits[1]; out->c_bits = bits[2];
    out->a_bytes = (nb * bits[0] + 7) / 8;
    out->b_bytes = (nb * bits[1] + 7) / 8;
    out->c_bytes = (nb * bits[2] + 7) / 8;
    out->halo_rows = g->mode == SE_MODE_FULL ? 2u * ((1u << g->levels) - 1u) : 0u;
    return SE_OK;
}

static int fused_checks(const se_geom* g, const uint8_t* key, const uint8_t* iv, se_layout& lay) {
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv) return SE_EINVAL;
    if (lay.n_blocks > kMaxBlocks) return SE_EINVAL;          // 2^32 blocks (256 GiB) per call
    if ((g->block_offset * lay.a_bits) % 128) return SE_EINVAL;
    // FULL mode transforms the whole matrix: a stripe would need its
    // neighbours' halo rows, which this entry point does not take.
    if (g->mode == SE_MODE_FULL && g->block_offset) return SE_ENOTSUP;
    return SE_OK;
}

static DwtParams dwt_params(const se_geom* g, const se_layout& lay) {
    DwtParams p;
    memset(&p, 0, sizeof p);
    p.n_bytes = g->n_bytes; p.n_blocks = lay.n_blocks;
    p.width = g->width; p.bpr = g->width / 8; p.rows = (uint32_t)lay.rows; p.one = 1;
    p.row0 = 0; p.rows_out = lay.rows; p.src_row0 = 0; p.src_rows = lay.rows;   // whole matrix
    return p;
}


}  // extern "C"

namespace se {

// FULL mode: the R x W int16 Mallat coefficients between the transform and
// the footprint kernels live in the caller's workspace.
static uint64_t full_ws_bytes(uint64_t rows, uint32_t width) { return rows * width * sizeof(int16_t); }

// Kernel choice for single-file BLOCK8 calls on device buffers: the
// persistent tile kernels (k_tile.cu) or the per-CTA kernels (k_block8.cu).
// SE_KERNEL=tile|cta or se_kernel_choice() force one (measurement knob).
static std::atomic<int> g_kernel_choice{-1};   // -1: not yet read from SE_KERNEL

static int kernel_choice() {          // 0 auto, 1 tile, 2 cta
    int v = g_kernel_choice.load(std::memory_order_relaxed);
    if (v < 0) {
        const char* e = getenv("SE_KERNEL");
        v = !e ? 0 : strcmp(e, "tile") == 0 ? 1 : strcmp(e, "cta") == 0 ? 2 : 0;
        g_kernel_choice.store(v, std::memory_order_relaxed);
    }
    return v;
}

static bool use_tile(bool mask) {
    const int k = kernel_choice();
    if (k) return k == 1;
    // measured on C2 / C3 / C4: masked (ALU-bound on SHA-2)
    // the per-CTA kernels are ahead at every size (finer work units; the
    // keystream kernels overlap); PUBLIC_PLAIN the tile kernels at every size
    return !mask;
}

extern "C" int se_kernel_choice(int choice) {
    const int prev = kernel_choice();
    if (choice >= 0 && choice <= 2) g_kernel_choice.store(choice, std::memory_order_relaxed);
    return prev;
}

static bool ks_out_enabled() {
    static const int v = [] {
        const char* e = getenv("SE_KS_OUT");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// Masked per-CTA protect: the keystream kernel first (1), or AES inside the
// fused kernel (0).  SE_PROT_KS in the environment overrides (measurement knob).
static bool prot_ks_enabled(uint64_t n_blocks) {
    static const int v = [] {
        const char* e = getenv("SE_PROT_KS");
        return e ? atoi(e) : -1;
    }();
    if (v >= 0) return v != 0;
    (void)n_blocks;
    return true;
}

static int launch_keystream_into(const FusedParams& p, uint8_t* out, uint64_t n, void* stream,
                                 se_report* init_report = nullptr, uint32_t cta_ablocks = 0) {
    CipherParams cp;
    memset(&cp, 0, sizeof cp);
    cp.report = init_report;
    cp.cta_ablocks = cta_ablocks;
    cp.bpr = p.bpr;
    cp.width = p.width;
    cp.out = out;
    cp.n = n;
    static const int lut = [] {
        const char* e = getenv("SE_KS_LUT");
        return e ? atoi(e) : 1;
    }();
    // 1: the 64 KB lane-replicated table (measured: C4 masked protect 4.855 ->
    // 4.721 ms against the 5 KB tables, C2 / C3 slightly faster)
    cp.lane_lut = lut;
    // SE_KS_LANE_NARROW=1: one 128-thread lane-table CTA per SM beside the
    // fused kernel instead of 1024-thread CTAs on few SMs.  Measured slower
    // (C2 89.6 vs 92.5 GB/s, C4 112.8 vs 114.9: the narrow keystream
    // finishes late and the fused CTAs wait for it at copy-out), so off.
    static const int narrow = [] {
        const char* e = getenv("SE_KS_LANE_NARROW");
        return e ? atoi(e) : 0;
    }();
    cp.narrow = narrow;
    memcpy(cp.ctr, p.ctr, sizeof cp.ctr);
    memcpy(cp.rk, p.rk, sizeof cp.rk);
    return launch_cipher_ctr(cp, stream);
}

// {-1, 0} by one small kernel (one stream operation instead of two memsets;
// the fused kernel after it is a programmatic launch and waits for it)
static int report_init(se_report* r, cudaStream_t s) {
    return launch_report_init(r, 1, s) ? SE_ECUDA : SE_OK;
}

// Protect (rows a1-a9).  BLOCK8 on device buffers: PUBLIC_PLAIN on the
// persistent tile kernel (k_tile.cu, AES warps inside), masked on the per-CTA
// kernel (k_block8.cu) behind the keystream kernel.  BLOCK8 with o.mapped
// (fragments in page-locked host memory, se_host.cu): the per-CTA kernel with
// in-kernel AES, whose plain stores suit PCIe writes.  FULL: whole-matrix
// transform into o.ws, then the footprint kernel (in-kernel AES).
int protect_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in, void* d_a,
                 void* d_b, void* d_c, const ImplOpts& o, void* stream) {
    se_layout lay;
    int rc = fused_checks(g, key, iv, lay);
    if (rc) return rc;
    if (g->n_bytes == 0) return SE_OK;
    if (!d_in || !d_a || !d_c || (lay.b_bytes && !d_b)) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_a) || !aligned16(d_c) || (d_b && !aligned16(d_b))) return SE_EALIGN;
    FusedParams p;
    fill_fused(p, g, lay, key, iv);
    p.in = (const uint8_t*)d_in;
    p.a = (uint8_t*)d_a; p.b = (uint8_t*)d_b; p.c = (uint8_t*)d_c;
    const bool mask = !(g->flags & SE_FLAG_PUBLIC_PLAIN);
    if (g->mode == SE_MODE_BLOCK8) {
        if (!o.mapped && use_tile(mask))
            return launch_tile_block8(p, g->levels, mask, false, stream) ? SE_ECUDA : SE_OK;
        // per-CTA kernel; masked: the keystream kernel writes A' first and the
        // fused kernel XORs it in at its copy-out (programmatic launch overlap);
        // unmasked (and host-mapped A'): AES inside the fused kernel
        if (mask && !o.mapped && prot_ks_enabled(lay.n_blocks)) {
            p.ks_in_a = 1;
            if (launch_keystream_into(p, p.a, lay.a_bytes, stream)) return SE_ECUDA;
        }
        return launch_protect_block8(p, g->levels, mask, stream) ? SE_ECUDA : SE_OK;
    }
    if (!o.ws || o.ws_bytes < full_ws_bytes(lay.rows, g->width)) return SE_EINVAL;
    if (!aligned16(o.ws)) return SE_EALIGN;
    int16_t* ws = (int16_t*)o.ws;
    DwtParams dp = dwt_params(g, lay);
    dp.in = p.in; dp.coef = ws;
    p.ws = ws; p.rows = lay.rows;
    // the footprint kernel encrypts A itself (a keystream kernel between the
    // transform and it measured slower: C4-FULL protect 198.9 -> 190.5 GB/s)
    int e = launch_dwt_full_fwd(dp, g->levels, stream);
    if (!e) e = launch_protect_full(p, g->levels, mask, stream);
    return e ? SE_ECUDA : SE_OK;
}

// Recover (row a10), the mirror of protect_impl.  The report is set to
// {-1, 0} here unless o.report_ready.
int recover_impl(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a, const void* d_b,
                 const void* d_c, void* d_out, se_report* d_report, const ImplOpts& o, void* stream) {
    se_layout lay;
    int rc = fused_checks(g, key, iv, lay);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->n_bytes != 0) {
        if (!d_out || !d_a || !d_c || (lay.b_bytes && !d_b)) return SE_EINVAL;
        if (!aligned16(d_out) || !aligned16(d_a) || !aligned16(d_c) || (d_b && !aligned16(d_b))) return SE_EALIGN;
        if (g->mode == SE_MODE_FULL) {
            if (!o.ws || o.ws_bytes < full_ws_bytes(lay.rows, g->width)) return SE_EINVAL;
            if (!aligned16(o.ws)) return SE_EALIGN;
        }
    }
    const bool mask = !(g->flags & SE_FLAG_PUBLIC_PLAIN);
    const bool tile = g->mode == SE_MODE_BLOCK8 && !o.mapped && use_tile(mask);
    // masked per-CTA recovery on whole 1024-byte-multiple rows (C2, C3, C4): the
    // keystream kernel writes each CTA's A-slice keystream into the start of
    // that CTA's own output region and initialises the report
    const bool ks_out = g->mode == SE_MODE_BLOCK8 && !o.mapped && !tile && mask && g->levels >= 2 &&
                        g->width % 1024 == 0 && g->n_bytes == lay.rows * g->width && g->n_bytes && ks_out_enabled();
    if (d_report && !o.report_ready && !ks_out && report_init(d_report, s)) return SE_ECUDA;
    if (g->n_bytes == 0) return SE_OK;
    FusedParams p;
    fill_fused(p, g, lay, key, iv);
    p.out = (uint8_t*)d_out;
    p.a = (uint8_t*)d_a; p.b = (uint8_t*)d_b; p.c = (uint8_t*)d_c;
    p.report = d_report;
    if (g->mode == SE_MODE_BLOCK8) {
        if (tile) return launch_tile_block8(p, g->levels, mask, true, stream) ? SE_ECUDA : SE_OK;
        if (ks_out) {
            p.ks_in_out = 1;
            if (launch_keystream_into(p, p.out, lay.a_bytes, stream, o.report_ready ? nullptr : d_report,
                                      kBlocksPerCta * lay.a_bits / 128))
                return SE_ECUDA;
        }
        return launch_recover_block8(p, g->levels, mask, stream) ? SE_ECUDA : SE_OK;
    }
    int16_t* ws = (int16_t*)o.ws;
    p.ws = ws; p.rows = lay.rows;
    DwtParams dp = dwt_params(g, lay);
    dp.out = p.out; dp.coef = ws;
    int e = 0;
    if (mask && !o.mapped && lay.a_bytes <= g->n_bytes) {     // keystream parked in out (written last)
        p.ks_in_out = 2;
        e = launch_keystream_into(p, p.out, lay.a_bytes, stream);
    }
    if (!e) e = launch_recover_full(p, g->levels, mask, stream);               // unmask + scatter
    if (!e) e = launch_dwt_full_inv(dp, g->levels, d_report, stream);          // inverse + report
    return e ? SE_ECUDA : SE_OK;
}

}  // namespace se

extern "C" {

int fragment_workspace_size(const se_geom* g, const se_stripe* st, uint64_t* bytes) {
    if (!bytes) return SE_EINVAL;
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    *bytes = 0;
    if (g->mode != SE_MODE_FULL) return SE_OK;
    if (!st) {
        *bytes = full_ws_bytes(lay.rows, g->width);
        return SE_OK;
    }
    // stripes: the larger of the protect window (the stripe's rows) and the
    // recover window (its fragment block rows, halos included)
    const uint64_t rows = std::max(st->row_end > st->row_begin ? st->row_end - st->row_begin : 0, st->src_rows);
    *bytes = full_ws_bytes(rows, g->width);
    return SE_OK;
}

int fragment_protect_ws(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in, void* d_a,
                        void* d_b, void* d_c, void* d_ws, uint64_t ws_bytes, void* stream) {
    SE_RANGE("fragment_protect_ws");
    ImplOpts o;
    o.ws = d_ws;
    o.ws_bytes = ws_bytes;
    return protect_impl(g, key, iv, d_in, d_a, d_b, d_c, o, stream);
}

int fragment_recover_ws(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a,
                        const void* d_b, const void* d_c, void* d_out, se_report* d_report, void* d_ws,
                        uint64_t ws_bytes, void* stream) {
    SE_RANGE("fragment_recover_ws");
    ImplOpts o;
    o.ws = d_ws;
    o.ws_bytes = ws_bytes;
    return recover_impl(g, key, iv, d_a, d_b, d_c, d_out, d_report, o, stream);
}

int fragment_protect(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in,
                     void* d_a, void* d_b, void* d_c, void* stream) {
    SE_RANGE("fragment_protect");
    return protect_impl(g, key, iv, d_in, d_a, d_b, d_c, ImplOpts(), stream);
}

int fragment_recover(const se_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a,
                     const void* d_b, const void* d_c, void* d_out, se_report* d_report, void* stream) {
    SE_RANGE("fragment_recover");
    return recover_impl(g, key, iv, d_a, d_b, d_c, d_out, d_report, ImplOpts(), stream);
}

// ---------------------------------------------------------------- FULL-mode stripes (row e for a11)

static bool stripe_aligned(const se_layout& lay, uint64_t blocks_before) {
    const uint64_t bits[3] = {lay.a_bits, lay.b_bits, lay.c_bits};
    for (uint64_t b : bits)
        if ((blocks_before * b) % 8) return false;
    return (blocks_before * lay.a_bits) % 128 == 0;                         // CTR start whole AES blocks
}

static int stripe_checks(const se_geom* g, const se_stripe* st, const uint8_t* key, const uint8_t* iv,
                         se_layout& lay, bool recover) {
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (!st || !key || !iv || g->mode != SE_MODE_FULL || g->n_bytes == 0) return SE_EINVAL;
    if ((g->block_offset * lay.a_bits) % 128) return SE_EINVAL;
    const uint64_t R = lay.rows, bpr = g->width / 8;
    if (st->row_begin % 8 || st->row_end % 8 || st->row_begin >= st->row_end || st->row_end > R) return SE_EINVAL;
    const uint64_t s0 = st->src_row0, s1 = st->src_row0 + st->src_rows;
    if (s1 > R || s0 >= s1) return SE_EINVAL;
    // (protect windows may end before need1 only where the file has no bytes)
    // halo: input rows (protect) or whole halo block rows of fragments (recover)
    const uint64_t halo = recover ? (lay.halo_rows + 7) / 8 * 8 : lay.halo_rows;
    const uint64_t need0 = st->row_begin >= halo ? st->row_begin - halo : 0;
    // protect: rows past the file's last byte read as zero (C18) and need not be present
    const uint64_t data_rows = recover ? R : (g->n_bytes + g->width - 1) / g->width;
    const uint64_t need1 = std::min<uint64_t>(std::min<uint64_t>(R, data_rows), st->row_end + halo);
    if (s0 > need0 || s1 < need1) return SE_EINVAL;
    if (!stripe_aligned(lay, st->row_begin / 8 * bpr)) return SE_EINVAL;
    if (recover && (s0 % 8 || s1 % 8 || !stripe_aligned(lay, s0 / 8 * bpr))) return SE_EINVAL;
    return SE_OK;
}

// FusedParams for the blocks of rows [r0, r1) of a FULL file (local Mallat of those rows)
static void stripe_fused(FusedParams& p, const se_geom* g, const se_layout& lay, const uint8_t key[16],
                         const uint8_t iv[16], uint64_t r0, uint64_t r1) {
    fill_fused(p, g, lay, key, iv);
    const uint64_t bpr = g->width / 8, nb = (r1 - r0) / 8 * bpr;
    p.n_blocks = nb;
    p.block_offset = g->block_offset + r0 / 8 * bpr;
    p.a_bytes = (nb * lay.a_bits + 7) / 8;
    p.b_bytes = (nb * lay.b_bits + 7) / 8;
    p.c_bytes = (nb * lay.c_bits + 7) / 8;
    p.rows = r1 - r0;
    ctr_base(iv, p.block_offset * lay.a_bits / 128, p.ctr);
}

}  // extern "C"

extern "C" {

int fragment_protect_stripe(const se_geom* g, const se_stripe* st, const uint8_t key[16], const uint8_t iv[16],
                            const void* d_in, void* d_a, void* d_b, void* d_c, void* d_ws, uint64_t ws_bytes,
                            void* stream) {
    SE_RANGE("fragment_protect_stripe");
    se_layout lay;
    int rc = stripe_checks(g, st, key, iv, lay, false);
    if (rc) return rc;
    if (!d_in || !d_a || !d_c || (lay.b_bits && !d_b)) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_a) || !aligned16(d_c) || (d_b && !aligned16(d_b))) return SE_EALIGN;
    if (!d_ws || ws_bytes < full_ws_bytes(st->row_end - st->row_begin, g->width)) return SE_EINVAL;
    if (!aligned16(d_ws)) return SE_EALIGN;
    FusedParams p;
    stripe_fused(p, g, lay, key, iv, st->row_begin, st->row_end);
    p.a = (uint8_t*)d_a; p.b = (uint8_t*)d_b; p.c = (uint8_t*)d_c;
    DwtParams dp = dwt_params(g, lay);
    dp.in = (const uint8_t*)d_in; dp.coef = (int16_t*)d_ws;
    dp.row0 = st->row_begin; dp.rows_out = st->row_end - st->row_begin;
    dp.src_row0 = st->src_row0; dp.src_rows = st->src_rows;
    p.ws = (int16_t*)d_ws;
    const bool mask = !(g->flags & SE_FLAG_PUBLIC_PLAIN);
    int e = launch_dwt_full_fwd(dp, g->levels, stream);
    if (!e) e = launch_protect_full(p, g->levels, mask, stream);
    return e ? SE_ECUDA : SE_OK;
}

int fragment_recover_stripe(const se_geom* g, const se_stripe* st, const uint8_t key[16], const uint8_t iv[16],
                            const void* d_a, const void* d_b, const void* d_c, void* d_out, se_report* d_report,
                            void* d_ws, uint64_t ws_bytes, void* stream) {
    SE_RANGE("fragment_recover_stripe");
    se_layout lay;
    int rc = stripe_checks(g, st, key, iv, lay, true);
    if (rc) return rc;
    if (!d_a || !d_c || !d_out || (lay.b_bits && !d_b)) return SE_EINVAL;
    if (!aligned16(d_a) || !aligned16(d_c) || (d_b && !aligned16(d_b))) return SE_EALIGN;
    const uint64_t e0 = st->src_row0, e1 = st->src_row0 + st->src_rows;
    if (!d_ws || ws_bytes < full_ws_bytes(e1 - e0, g->width)) return SE_EINVAL;
    if (!aligned16(d_ws)) return SE_EALIGN;
    cudaStream_t s = (cudaStream_t)stream;
    if (d_report && report_init(d_report, s)) return SE_ECUDA;
    FusedParams p;
    stripe_fused(p, g, lay, key, iv, e0, e1);                              // the halo-extended block rows
    p.a = (uint8_t*)d_a; p.b = (uint8_t*)d_b; p.c = (uint8_t*)d_c;
    p.ws = (int16_t*)d_ws;
    const bool mask = !(g->flags & SE_FLAG_PUBLIC_PLAIN);
    DwtParams dp = dwt_params(g, lay);
    dp.out = (uint8_t*)d_out; dp.coef = (int16_t*)d_ws;
    dp.row0 = st->row_begin; dp.rows_out = st->row_end - st->row_begin;
    dp.src_row0 = e0; dp.src_rows = e1 - e0;
    const uint64_t out_bytes = std::min<uint64_t>(g->n_bytes, st->row_end * (uint64_t)g->width) -
                               st->row_begin * (uint64_t)g->width;
    int e = 0;
    if (mask && p.a_bytes <= out_bytes) {          // keystream parked in the stripe's output (written last)
        p.ks_in_out = 2;
        p.out = (uint8_t*)d_out;
        e = launch_keystream_into(p, p.out, p.a_bytes, stream);
    }
    if (!e) e = launch_recover_full(p, g->levels, mask, stream);          // unmask + scatter (halo too)
    if (!e) e = launch_dwt_full_inv(dp, g->levels, d_report, stream);     // the stripe's rows
    return e ? SE_ECUDA : SE_OK;
}

int dwt_fwd(const se_geom* g, const void* d_in, int16_t* d_coef, void* stream) {
    SE_RANGE("dwt_fwd");
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (g->n_bytes == 0) return SE_OK;
    if (!d_in || !d_coef) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_coef)) return SE_EALIGN;
    DwtParams p = dwt_params(g, lay);
    p.in = (const uint8_t*)d_in; p.coef = d_coef;
    const int e = g->mode == SE_MODE_BLOCK8 ? launch_dwt_fwd_block8(p, g->levels, stream)
                                            : launch_dwt_full_fwd(p, g->levels, stream);
    return e ? SE_ECUDA : SE_OK;
}

int dwt_inv(const se_geom* g, const int16_t* d_coef, void* d_out, void* stream) {
    SE_RANGE("dwt_inv");
    se_layout lay;
    int rc = fragment_layout(g, &lay);
    if (rc) return rc;
    if (g->n_bytes == 0) return SE_OK;
    if (!d_out || !d_coef) return SE_EINVAL;
    if (!aligned16(d_out) || !aligned16(d_coef)) return SE_EALIGN;
    DwtParams p = dwt_params(g, lay);
    p.out = (uint8_t*)d_out; p.coef = (int16_t*)d_coef;
    const int e = g->mode == SE_MODE_BLOCK8 ? launch_dwt_inv_block8(p, g->levels, stream)
                                            : launch_dwt_full_inv(p, g->levels, nullptr, stream);
    return e ? SE_ECUDA : SE_OK;
}

int cipher_encrypt(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block_offset, const void* d_in,
                   void* d_out, uint64_t n, void* stream) {
    SE_RANGE("cipher_encrypt");
    if (!key || !iv) return SE_EINVAL;
    if (n == 0) return SE_OK;
    if (!d_in || !d_out) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_out)) return SE_EALIGN;
    CipherParams p;
    memset(&p, 0, sizeof p);
    p.in = (const uint8_t*)d_in; p.out = (uint8_t*)d_out; p.n = n;
    ctr_base(iv, ctr_block_offset, p.ctr);
    key_expansion(key, p.rk);
    return launch_cipher_ctr(p, stream) ? SE_ECUDA : SE_OK;
}

int cipher_decrypt(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block_offset, const void* d_in,
                   void* d_out, uint64_t n, void* stream) {
    SE_RANGE("cipher_decrypt");
    return cipher_encrypt(key, iv, ctr_block_offset, d_in, d_out, n, stream);
}

int se_stats_accumulate(const void* d_x, const void* d_y, uint64_t n, uint32_t width, se_stats* d_stats,
                        uint32_t* d_joint, void* stream) {
    SE_RANGE("se_stats_accumulate");
    if (width == 0 || !d_stats) return SE_EINVAL;
    if (n == 0) return SE_OK;
    if (!d_y) return SE_EINVAL;
    return launch_stats(d_x, d_y, n, width, d_stats, d_x ? d_joint : nullptr, stream) ? SE_ECUDA : SE_OK;
}

int64_t fragment_batch_plan(se_job* jobs, uint32_t n_jobs, uint32_t levels, const uint8_t key[16]) {
    SE_RANGE("fragment_batch_plan");
    if (!jobs || !key || levels < 1 || levels > 3) return SE_EINVAL;
    uint64_t cta = 0;
    for (uint32_t j = 0; j < n_jobs; ++j) {
        se_job& job = jobs[j];
        se_geom g = {job.n_bytes, job.width, levels, SE_MODE_BLOCK8, 0, job.block_offset};
        se_layout lay;
        if (fragment_layout(&g, &lay) != SE_OK) return SE_EINVAL;
        if ((job.block_offset * lay.a_bits) % 128) return SE_EINVAL;
        if (job.n_bytes && (!job.a || !job.c || (lay.b_bytes && !job.b))) return SE_EINVAL;
        if (job.n_bytes && (!aligned16(job.a) || !aligned16(job.c) || (job.b && !aligned16(job.b)) ||
                            !aligned16(job.in ? (const void*)job.in : (const void*)job.out)))
            return SE_EALIGN;
        job.cta_begin = cta;
        cta += (lay.n_blocks + kBlocksPerCta - 1) / kBlocksPerCta;
        // per-file constants: counter base and SHA midstates over K || IV (C13, C15)
        FusedParams p;
        fill_fused(p, &g, lay, key, job.iv);
        JobDerived d;
        memcpy(d.ctr, p.ctr, sizeof d.ctr);
        memcpy(d.kiv, p.kiv, sizeof d.kiv);
        memcpy(d.mid256, p.mid256, sizeof d.mid256);
        memcpy(d.mid512, p.mid512, sizeof d.mid512);
        d.s512 = p.s512;
        memset(job.derived, 0, sizeof job.derived);
        memcpy(job.derived, &d, sizeof d);
    }
    if (cta > 0x7fffffffull) return SE_EINVAL;       // one launch: grid.x < 2^31
    return (int64_t)cta;
}

static int batch_common(uint32_t n_jobs, const se_job* d_jobs, uint64_t total_ctas, uint32_t levels,
                        uint32_t flags, const uint8_t key[16], se_report* d_reports, bool recover, void* stream) {
    if (!key || levels < 1 || levels > 3 || (flags & ~(uint32_t)SE_FLAG_PUBLIC_PLAIN)) return SE_EINVAL;
    if (n_jobs == 0) return SE_OK;
    if (!d_jobs) return SE_EINVAL;
    if (!aligned16(d_jobs)) return SE_EALIGN;
    BatchParams bp;
    memset(&bp, 0, sizeof bp);
    bp.jobs = d_jobs;
    bp.reports = d_reports;
    bp.n_jobs = n_jobs;
    se_geom g = {0, 8, levels, SE_MODE_BLOCK8, flags, 0};
    se_layout lay;
    fragment_layout(&g, &lay);
    const uint8_t zero_iv[16] = {0};
    fill_fused(bp.base, &g, lay, key, zero_iv);       // shared fields: round keys, H(0), one
    bp.total_ctas = total_ctas;
    const bool mask = !(flags & SE_FLAG_PUBLIC_PLAIN);
    // masked protect: a keystream kernel writes every file's keystream into its
    // A' and the batch kernel XORs it in; otherwise the AES-CTR of each A slice
    // runs inside the batch kernel.  No scratch either way.
    // Masked recover: the same kernel parks each qualifying CTA's keystream in
    // that CTA's own output region (batch_ks_out_cta: whole 1024-byte rows -
    // the big files), the others run their AES in the batch kernel.
    if (mask && total_ctas) {
        if (recover) bp.base.ks_in_out = 1;
        else bp.base.ks_in_a = 1;
        if (recover && d_reports) {      // reports first: the batch kernel then skips its start-of-kernel wait
            if (launch_report_init(d_reports, n_jobs, stream)) return SE_ECUDA;
            bp.reports_ready = 1;
        }
        if (launch_batch_keystream(bp, lay.a_bits, stream)) return SE_ECUDA;
    }
    return launch_batch_block8(bp, total_ctas, levels, mask, recover, stream) ? SE_ECUDA : SE_OK;
}

int fragment_protect_batch(uint32_t n_jobs, const se_job* d_jobs, uint64_t total_ctas, uint32_t levels,
                           uint32_t flags, const uint8_t key[16], void* stream) {
    SE_RANGE("fragment_protect_batch");
    return batch_common(n_jobs, d_jobs, total_ctas, levels, flags, key, nullptr, false, stream);
}

int fragment_recover_batch(uint32_t n_jobs, const se_job* d_jobs, uint64_t total_ctas, uint32_t levels,
                           uint32_t flags, const uint8_t key[16], se_report* d_reports, void* stream) {
    SE_RANGE("fragment_recover_batch");
    return batch_common(n_jobs, d_jobs, total_ctas, levels, flags, key, d_reports, true, stream);
}


}  // extern "C"
