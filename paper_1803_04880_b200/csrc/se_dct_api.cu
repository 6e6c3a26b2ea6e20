// se_dct_api.cu — host side of the Chapter 4 DCT SE calls (include/se_dct.h,
// row f3): geometry checks, the AES-CTR keystream launch and the fused DCT
// kernel launch (k_dct.cu) on the caller's stream.
#include <cuda_runtime.h>
#include <string.h>

#include "se_internal.h"

using namespace se;

// Level-2 protect's keystream kernel on the 64 KB lane-replicated table (1)
// or the 5 KB tables (0).  Round 2 (tools/gpu_r2_call50.sh, two passes):
// 4800x4800 protect 95.5 -> 93.3 us, the smaller Table 4.1 images unchanged.
// (Level 1 with a separate lane-table keystream instead of the in-kernel AES:
// 4800x4800 28.8 -> 27.5 us but 1024x768 10.6 -> 14.0 us, so level 1 keeps it.)
#ifndef SE_DCT_LANE_KS
#define SE_DCT_LANE_KS 1
#endif

static int check_dct(const se_dct_geom* g, bool need_level) {
    if (!g) return SE_EINVAL;
    if (g->width == 0 || g->height == 0 || g->width % 8 || g->height % 8) return SE_EINVAL;   // D11
    if (g->channels != 1 && g->channels != 3 && g->channels != 4) return SE_EINVAL;
    if (need_level && g->level != 1 && g->level != 2) return SE_EINVAL;
    if (g->flags & ~(uint32_t)SE_DCT_KEYED) return SE_EINVAL;
    if ((g->block_offset * 66) % 128) return SE_EINVAL;                                     // D8
    return SE_OK;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static DctParams dct_params(const se_dct_geom* g, const se_dct_layout& lay) {
    DctParams p;
    memset(&p, 0, sizeof p);
    p.n_pos = lay.records / g->channels;
    p.a_bytes = lay.a_bytes;
    p.block_offset = g->block_offset;
    p.width = g->width;
    p.bpr = g->width / 8;
    p.one = 1;
    return p;
}

static int launch_ks(const uint8_t key[16], const uint8_t iv[16], const se_dct_geom* g, uint8_t* out, uint64_t n,
                     void* stream) {
    CipherParams cp;
    memset(&cp, 0, sizeof cp);
    cipher_setup(key, iv, g->block_offset * 66 / 128, cp);
    cp.in = nullptr;
    cp.out = out;
    cp.n = n;
    cp.lane_lut = SE_DCT_LANE_KS;
    return launch_cipher_ctr(cp, stream);
}

static void aes_params(DctParams& p, const uint8_t key[16], const uint8_t iv[16], const se_dct_geom* g) {
    CipherParams cp;
    memset(&cp, 0, sizeof cp);
    cipher_setup(key, iv, g->block_offset * 66 / 128, cp);
    memcpy(p.ctr, cp.ctr, sizeof p.ctr);
    memcpy(p.rk, cp.rk, sizeof p.rk);
}

extern "C" {

int dct_layout(const se_dct_geom* g, se_dct_layout* out) {
    int rc = check_dct(g, true);
    if (rc) return rc;
    if (!out) return SE_EINVAL;
    const uint64_t pos = (uint64_t)(g->width / 8) * (g->height / 8);
    out->records = pos * g->channels;
    out->a_bits = 66;
    out->a_bytes = (out->records * 66 + 7) / 8;
    out->p_bytes = (uint64_t)g->width * g->height * g->channels;
    out->reserved = 0;
    return SE_OK;
}

int dct_protect(const se_dct_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in, void* d_a,
                void* d_p, void* stream) {
    SE_RANGE("dct_protect");
    se_dct_layout lay;
    int rc = dct_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv || !d_in || !d_a || !d_p) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_a) || !aligned16(d_p)) return SE_EALIGN;
    DctParams p = dct_params(g, lay);
    p.in = (const uint8_t*)d_in;
    p.out = (uint8_t*)d_p;
    p.a = (uint8_t*)d_a;
    if (g->level == 2) {
        sha512_kiv(key, iv, p.kiv, p.mid512, p.h512);
        dct_sched_consts(p, (g->flags & SE_DCT_KEYED) != 0);
    }
    aes_params(p, key, iv, g);
    if (!dct_fused_aes(0, g->level, p.n_pos) && launch_ks(key, iv, g, p.a, lay.a_bytes, stream)) return SE_ECUDA;
    return launch_dct(p, g->channels, g->level, (g->flags & SE_DCT_KEYED) != 0, 0, stream) ? SE_ECUDA : SE_OK;
}

int dct_recover(const se_dct_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a,
                const void* d_p, void* d_out, void* stream) {
    SE_RANGE("dct_recover");
    se_dct_layout lay;
    int rc = dct_layout(g, &lay);
    if (rc) return rc;
    if (!key || !iv || !d_a || !d_p || !d_out) return SE_EINVAL;
    if (!aligned16(d_a) || !aligned16(d_p) || !aligned16(d_out)) return SE_EALIGN;
    DctParams p = dct_params(g, lay);
    p.in = (const uint8_t*)d_p;
    p.out = (uint8_t*)d_out;
    p.a = (uint8_t*)d_a;
    if (g->level == 2) {
        sha512_kiv(key, iv, p.kiv, p.mid512, p.h512);
        dct_sched_consts(p, (g->flags & SE_DCT_KEYED) != 0);
    }
    aes_params(p, key, iv, g);
    // recovery always decrypts Fragment 1 inside the kernel: no keystream scratch
    return launch_dct(p, g->channels, g->level, (g->flags & SE_DCT_KEYED) != 0, 1, stream) ? SE_ECUDA : SE_OK;
}

int dct_select(const se_dct_geom* g, const void* d_in, float* d_coef, void* stream) {
    SE_RANGE("dct_select");
    int rc = check_dct(g, false);
    if (rc) return rc;
    if (!d_in || !d_coef) return SE_EINVAL;
    if (!aligned16(d_in) || ((uintptr_t)d_coef & 3u)) return SE_EALIGN;
    se_dct_layout lay;
    se_dct_geom g2 = *g;
    g2.level = 1;
    dct_layout(&g2, &lay);
    DctParams p = dct_params(g, lay);
    p.in = (const uint8_t*)d_in;
    p.coef = d_coef;
    return launch_dct(p, g->channels, 1, false, 2, stream) ? SE_ECUDA : SE_OK;
}

static int dct8_common(const se_dct_geom* g, se_dct_layout& lay) {
    int rc = check_dct(g, false);
    if (rc) return rc;
    se_dct_geom g2 = *g;
    g2.level = 1;
    g2.flags = 0;
    g2.block_offset = 0;
    return dct_layout(&g2, &lay);
}

int dct8_forward(const se_dct_geom* g, const void* d_in, float* d_coef, void* stream) {
    SE_RANGE("dct8_forward");
    se_dct_layout lay;
    int rc = dct8_common(g, lay);
    if (rc) return rc;
    if (!d_in || !d_coef) return SE_EINVAL;
    if (!aligned16(d_in) || !aligned16(d_coef)) return SE_EALIGN;
    DctParams p = dct_params(g, lay);
    p.in = (const uint8_t*)d_in;
    p.coef = d_coef;
    return launch_dct(p, g->channels, 1, false, 3, stream) ? SE_ECUDA : SE_OK;
}

int dct8_inverse(const se_dct_geom* g, const float* d_coef, void* d_out, void* stream) {
    SE_RANGE("dct8_inverse");
    se_dct_layout lay;
    int rc = dct8_common(g, lay);
    if (rc) return rc;
    if (!d_coef || !d_out) return SE_EINVAL;
    if (!aligned16(d_out) || !aligned16(d_coef)) return SE_EALIGN;
    DctParams p = dct_params(g, lay);
    p.coef = const_cast<float*>(d_coef);
    p.out = (uint8_t*)d_out;
    return launch_dct(p, g->channels, 1, false, 4, stream) ? SE_ECUDA : SE_OK;
}

}  // extern "C"
