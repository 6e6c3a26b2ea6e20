// se_container.cpp — fragment containers and dispersion layouts (row f4,
// include/se_container.h).  Host-only: serialisation, validation, content
// digests (FIPS 180-4 SHA-256 on the host) and the placement / storage
// accounting of the paper's two layouts.
#include <string.h>

#include "../../include/se.h"
#include "../../include/se_container.h"
#include "../../include/se_dct.h"
#include "tables.h"

namespace {

const uint32_t kK[64] = SE_SHA256_K_INIT;
const uint32_t kH0[8] = SE_SHA256_H0_INIT;

inline uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void sha256_block(uint32_t h[8], const uint8_t* p) {
    uint32_t w[64];
    for (int t = 0; t < 16; ++t)
        w[t] = (uint32_t)p[4 * t] << 24 | (uint32_t)p[4 * t + 1] << 16 | (uint32_t)p[4 * t + 2] << 8 | p[4 * t + 3];
    for (int t = 16; t < 64; ++t) {
        const uint32_t s0 = ror(w[t - 15], 7) ^ ror(w[t - 15], 18) ^ (w[t - 15] >> 3);
        const uint32_t s1 = ror(w[t - 2], 17) ^ ror(w[t - 2], 19) ^ (w[t - 2] >> 10);
        w[t] = w[t - 16] + s0 + w[t - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int t = 0; t < 64; ++t) {
        const uint32_t t1 = hh + (ror(e, 6) ^ ror(e, 11) ^ ror(e, 25)) + ((e & f) ^ (~e & g)) + kK[t] + w[t];
        const uint32_t t2 = (ror(a, 2) ^ ror(a, 13) ^ ror(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

void put16(uint8_t* p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
void put32(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i)); }
void put64(uint8_t* p, uint64_t v) { for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i)); }
uint32_t get16(const uint8_t* p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8; }
uint32_t get32(const uint8_t* p) {
    return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
uint64_t get64(const uint8_t* p) { return (uint64_t)get32(p) | (uint64_t)get32(p + 4) << 32; }

constexpr uint32_t kHeader = 72, kEntry = 56, kVersion = 1;
inline uint64_t align8(uint64_t v) { return (v + 7) & ~7ull; }

uint32_t scheme_mask(uint32_t scheme) {
    if (scheme == SE_SCHEME_DCT) return 1u << SE_STREAM_A | 1u << SE_STREAM_P;
    return 1u << SE_STREAM_A | 1u << SE_STREAM_B | 1u << SE_STREAM_C;
}

}  // namespace

extern "C" {

void se_sha256(const void* data, uint64_t len, uint8_t out[32]) {
    uint32_t h[8];
    memcpy(h, kH0, sizeof h);
    const uint8_t* p = (const uint8_t*)data;
    uint64_t n = len;
    for (; n >= 64; n -= 64, p += 64) sha256_block(h, p);
    uint8_t tail[128] = {0};
    memcpy(tail, p, n);
    tail[n] = 0x80;                                                     // FIPS 180-4 §5.1.1
    const uint64_t nb = (n + 9 <= 64) ? 64 : 128;
    const uint64_t bits = len * 8;
    for (int i = 0; i < 8; ++i) tail[nb - 1 - i] = (uint8_t)(bits >> (8 * i));
    sha256_block(h, tail);
    if (nb == 128) sha256_block(h, tail + 64);
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 4; ++k) out[4 * i + k] = (uint8_t)(h[i] >> (24 - 8 * k));
}

int se_container_streams(const se_container_info* info, uint64_t lens[4]) {
    if (!info || !lens) return SE_EINVAL;
    for (int i = 0; i < 4; ++i) lens[i] = 0;
    if (info->scheme == SE_SCHEME_DCT) {
        se_dct_geom g;
        memset(&g, 0, sizeof g);
        g.width = info->width; g.height = info->height; g.channels = info->channels;
        g.level = info->levels; g.flags = info->flags; g.block_offset = info->block_offset;
        se_dct_layout lay;
        int rc = dct_layout(&g, &lay);
        if (rc) return rc;
        if (info->n_bytes != lay.p_bytes) return SE_EINVAL;               // n_bytes = the image size
        lens[SE_STREAM_A] = lay.a_bytes;
        lens[SE_STREAM_P] = lay.p_bytes;
        return SE_OK;
    }
    if (info->scheme != SE_SCHEME_DWT_BLOCK8 && info->scheme != SE_SCHEME_DWT_FULL) return SE_EINVAL;
    if (info->height != 0 || info->channels != 1) return SE_EINVAL;
    se_geom g;
    memset(&g, 0, sizeof g);
    g.n_bytes = info->n_bytes; g.width = info->width; g.levels = info->levels;
    g.mode = info->scheme == SE_SCHEME_DWT_FULL ? SE_MODE_FULL : SE_MODE_BLOCK8;
    g.flags = info->flags; g.block_offset = info->block_offset;
    se_layout lay;
    int rc = fragment_layout(&g, &lay);
    if (rc) return rc;
    lens[SE_STREAM_A] = lay.a_bytes;
    lens[SE_STREAM_B] = lay.b_bytes;
    lens[SE_STREAM_C] = lay.c_bytes;
    return SE_OK;
}

int se_container_size(const se_container_info* info, uint32_t stream_mask, uint64_t* out_bytes) {
    uint64_t lens[4];
    int rc = se_container_streams(info, lens);
    if (rc) return rc;
    if (!out_bytes || !stream_mask || (stream_mask & ~scheme_mask(info->scheme))) return SE_EINVAL;
    uint64_t n = 0;
    for (int id = 0; id < 4; ++id) n += (stream_mask >> id) & 1u;
    uint64_t off = kHeader + kEntry * n;
    for (int id = 0; id < 4; ++id)
        if ((stream_mask >> id) & 1u) off = align8(off) + lens[id];
    *out_bytes = off;
    return SE_OK;
}

int se_container_pack(const se_container_info* info, uint32_t stream_mask, const void* const streams[4],
                      uint8_t* out, uint64_t cap, uint64_t* written) {
    uint64_t total = 0, lens[4];
    int rc = se_container_size(info, stream_mask, &total);
    if (rc) return rc;
    se_container_streams(info, lens);
    if (!out || !streams || cap < total) return SE_EINVAL;
    for (int id = 0; id < 4; ++id)
        if (((stream_mask >> id) & 1u) && lens[id] && !streams[id]) return SE_EINVAL;
    memset(out, 0, total);
    memcpy(out, "SEFR", 4);
    put16(out + 4, kVersion);
    put16(out + 6, kHeader);
    put32(out + 8, info->scheme); put32(out + 12, info->flags); put32(out + 16, info->levels);
    put32(out + 20, info->width); put32(out + 24, info->height); put32(out + 28, info->channels);
    put64(out + 32, info->n_bytes); put64(out + 40, info->block_offset);
    memcpy(out + 48, info->iv, 16);
    uint32_t e = 0;
    for (int id = 0; id < 4; ++id) e += (stream_mask >> id) & 1u;
    put32(out + 64, e);
    uint64_t off = kHeader + kEntry * (uint64_t)e;
    uint32_t k = 0;
    for (int id = 0; id < 4; ++id) {
        if (!((stream_mask >> id) & 1u)) continue;
        off = align8(off);
        uint8_t* ent = out + kHeader + kEntry * k++;
        put32(ent, (uint32_t)id);
        put64(ent + 8, off);
        put64(ent + 16, lens[id]);
        if (lens[id]) memcpy(out + off, streams[id], lens[id]);
        se_sha256(out + off, lens[id], ent + 24);
        off += lens[id];
    }
    if (written) *written = total;
    return SE_OK;
}

int se_container_open(const uint8_t* buf, uint64_t len, int verify, se_container_info* info,
                      uint32_t* stream_mask, const uint8_t* streams[4], uint32_t* bad_mask) {
    if (!buf || !info || !stream_mask || !streams) return SE_EINVAL;
    if (bad_mask) *bad_mask = 0;
    if (len < kHeader || memcmp(buf, "SEFR", 4) != 0) return SE_EFORMAT;
    if (get16(buf + 4) != kVersion || get16(buf + 6) != kHeader || get32(buf + 68) != 0) return SE_EFORMAT;
    se_container_info h;
    h.scheme = get32(buf + 8); h.flags = get32(buf + 12); h.levels = get32(buf + 16);
    h.width = get32(buf + 20); h.height = get32(buf + 24); h.channels = get32(buf + 28);
    h.n_bytes = get64(buf + 32); h.block_offset = get64(buf + 40);
    memcpy(h.iv, buf + 48, 16);
    uint64_t lens[4];
    if (se_container_streams(&h, lens)) return SE_EFORMAT;                 // geometry must be valid
    const uint32_t e = get32(buf + 64);
    if (e == 0 || e > 4 || kHeader + (uint64_t)kEntry * e > len) return SE_EFORMAT;
    uint32_t mask = 0;
    const uint8_t* ptr[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t prev_end = kHeader + (uint64_t)kEntry * e;
    uint32_t bad = 0;
    for (uint32_t k = 0; k < e; ++k) {
        const uint8_t* ent = buf + kHeader + kEntry * k;
        const uint32_t id = get32(ent);
        const uint64_t off = get64(ent + 8), n = get64(ent + 16);
        if (id > 3 || get32(ent + 4) != 0 || ((mask >> id) & 1u)) return SE_EFORMAT;
        if (!((scheme_mask(h.scheme) >> id) & 1u) || n != lens[id]) return SE_EFORMAT;
        if (off % 8 || off < prev_end || off > len || n > len - off) return SE_EFORMAT;
        prev_end = off + n;
        mask |= 1u << id;
        ptr[id] = buf + off;
        if (verify) {
            uint8_t d[32];
            se_sha256(buf + off, n, d);
            if (memcmp(d, ent + 24, 32) != 0) bad |= 1u << id;
        }
    }
    *info = h;
    *stream_mask = mask;
    for (int id = 0; id < 4; ++id) streams[id] = ptr[id];
    if (bad_mask) *bad_mask = bad;
    return bad ? (int)SE_EINTEGRITY : (int)SE_OK;
}

int se_disperse_plan(uint32_t layout, uint32_t scheme, uint32_t* local_mask, uint32_t remote_masks[2]) {
    if (!local_mask || !remote_masks) return SE_EINVAL;
    if (scheme != SE_SCHEME_DWT_BLOCK8 && scheme != SE_SCHEME_DWT_FULL && scheme != SE_SCHEME_DCT)
        return SE_EINVAL;
    const uint32_t A = 1u << SE_STREAM_A, B = 1u << SE_STREAM_B, C = 1u << SE_STREAM_C, P = 1u << SE_STREAM_P;
    if (scheme == SE_SCHEME_DCT) {                       // Fragment 1 local, Fragment 2 remote
        if (layout != SE_LAYOUT_A_LOCAL) return SE_EINVAL;
        *local_mask = A; remote_masks[0] = P; remote_masks[1] = 0;
        return SE_OK;
    }
    if (layout == SE_LAYOUT_A_LOCAL) {                   // P:2285 reliable channel; P:2748 two clouds
        *local_mask = A; remote_masks[0] = B; remote_masks[1] = C;
    } else if (layout == SE_LAYOUT_AB_LOCAL) {           // P:2283 unreliable channel: 164 b local
        *local_mask = A | B; remote_masks[0] = C; remote_masks[1] = 0;
    } else {
        return SE_EINVAL;
    }
    return SE_OK;
}

int se_storage_footprint(const se_container_info* info, uint32_t layout, double* local_frac, double* total_frac) {
    if (!info || !local_frac || !total_frac) return SE_EINVAL;
    uint32_t lm, rm[2];
    int rc = se_disperse_plan(layout, info->scheme, &lm, rm);
    if (rc) return rc;
    const uint64_t n = info->n_bytes;
    if (n == 0) return SE_EINVAL;
    uint64_t local = 0, total = 0;
    rc = se_container_size(info, lm, &local);
    if (rc) return rc;
    total = local;
    for (int k = 0; k < 2; ++k) {
        if (!rm[k]) continue;
        uint64_t s = 0;
        rc = se_container_size(info, rm[k], &s);
        if (rc) return rc;
        total += s;
    }
    *local_frac = (double)local / (double)n;
    *total_frac = (double)total / (double)n;
    return SE_OK;
}

}  // extern "C"
