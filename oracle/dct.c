/*
 * dct.c — oracle: the Chapter 4 DCT 8x8 selective encryption of bitmaps
 * (NEXT row f3; TEST INFRASTRUCTURE, see oracle.h).
 *
 * Follows, in the paper's order (PAPER.md "Design of SE for bitmaps based on
 * DCT", and "DCT transformation ..."):
 *   1. each colour layer is processed as a grey-scale image
 *   2. subtract 128 from each pixel
 *   3. DCT 8x8 of every block, Eq. 4.1 (alpha: Eq. 4.3);
 *      C(0,0) = alpha(0)^2 * sum f, Eq. 4.4
 *   4. Fragment 1 = coefficients [0,0],[0,1],[1,0],[2,0],[1,1],[0,2]
 *
 *      stored with the 11-bit store method: 1 sign bit + 10 bits of
 *      magnitude, 66 bits per block
 *   5. Fragment 2 = iDCT (Eq. 4.2) of the coefficients with DC padded with
 *      1024 and the 5 selected AC padded with 0, rounded to 8-bit unsigned
 *      integers in [0, 255]
 *   6. Fragment 1 is encrypted with AES-128
 *   7. level 2: Fragment 2 ^= SHA-512(the 6 selected coefficients), the 64
 *      digest bytes over the 64 pixels of the block
 *   recover: DCT of Fragment 2, the 6 stored coefficients put back, iDCT,
 *   + 128, rounded to [0, 255] ("rebuilt image").
 *
 * Readings (D1-D12):
 *   D1  f(x, y): x = row, y = column of the 8x8 block; coefficient [u,v]
 *       has vertical frequency u (Eq. 4.1 with x <-> u, y <-> v).
 *   D2  the printed matrix of Eq. 4.6 is C[x][u] = alpha(u) cos(pi(2x+1)u/16)
 *       (its FIRST COLUMN is constant), so the forward transform of Eq. 4.1
 *       is C^T X C; Eq. 4.5 "C x Input x C^T" is read as Eq. 4.1 (Eq. 4.1
 *       is the authority).
 *   D3  every rounding is IEEE-754 round-to-nearest, ties-to-even (rint).
 *   D4  the DC coefficient is quantised from Eq. 4.4 exactly (sum/8 is exact
 *       in binary floating point).
 *   D5  11-bit store: sign bit (1 = negative) then |q| in 10 bits, |q|
 *       saturated at 1023 (the all-zero block has DC = -1024, one past the
 *       10-bit range the paper states).
 *   D6  record = the 6 fields in the order of P:1423, MSB-first; records of
 *       a file concatenated densely in record order (as C11).
 *   D7  record order: block-major, row-major over blocks, then colour layer:
 *       r = ((br * W/8) + bc) * channels + ch; pixels stored interleaved,
 *       byte (row, col, ch) at ((row * W) + col) * channels + ch.
 *   D8  AES-128-CTR on the dense Fragment-1 stream, counter = IV +
 *       (block_offset * 66 / 128) + j (C12, C13).
 *   D9  level-2 message = the 66-bit record zero-padded to 9 bytes; with
 *       flag KEYED the message is K || IV || be64(block_offset + r) || rec9
 *       (the Chapter 5 framing C15).
 *   D10 digest byte 8x + y masks pixel (x, y) of the block.
 *   D11 width and height are multiples of 8 (the paper's images are).
 *   D12 recovery computes the DCT of Fragment 2 as stored (uncentered): only
 *       the DC differs from the centered DCT, and it is replaced.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

static const int kSel[6][2] = {{0, 0}, {0, 1}, {1, 0}, {2, 0}, {1, 1}, {0, 2}};

/* Eq. 4.3 */
static double alpha(int u) { return u == 0 ? sqrt(1.0 / 8.0) : 0.5; }

/* the cosine factor cos[pi (2x+1) u / 16] of Eq. 4.1 / 4.2 */
static const double kPi = 3.14159265358979323846;
static double cosf16(int x, int u) { return cos(kPi * (2 * x + 1) * u / 16.0); }

void oracle_dct_basis(double m[64]) {
    for (int x = 0; x < 8; ++x)
        for (int u = 0; u < 8; ++u) m[x * 8 + u] = alpha(u) * cosf16(x, u);    /* Eq. 4.6 layout (D2) */
}

/* Eq. 4.1 written out: C(u,v) = a(u) a(v) sum_x sum_y f(x,y) cos cos */
void oracle_dct8_fwd(const double f[64], double c[64]) {
    for (int u = 0; u < 8; ++u)
        for (int v = 0; v < 8; ++v) {
            double s = 0.0;
            for (int x = 0; x < 8; ++x)
                for (int y = 0; y < 8; ++y) s += f[x * 8 + y] * cosf16(x, u) * cosf16(y, v);
            c[u * 8 + v] = alpha(u) * alpha(v) * s;
        }
}

/* Eq. 4.2 written out: f(x,y) = sum_u sum_v a(u) a(v) C(u,v) cos cos */
void oracle_dct8_inv(const double c[64], double f[64]) {
    for (int x = 0; x < 8; ++x)
        for (int y = 0; y < 8; ++y) {
            double s = 0.0;
            for (int u = 0; u < 8; ++u)
                for (int v = 0; v < 8; ++v) s += alpha(u) * alpha(v) * c[u * 8 + v] * cosf16(x, u) * cosf16(y, v);
            f[x * 8 + y] = s;
        }
}

int oracle_dct_layout(uint32_t width, uint32_t height, uint32_t channels, uint64_t out[4]) {
    if (width == 0 || height == 0 || width % 8 || height % 8) return -1;        /* D11 */
    if (channels != 1 && channels != 3 && channels != 4) return -1;
    uint64_t nrec = (uint64_t)(width / 8) * (height / 8) * channels;
    out[0] = nrec;                                            /* records */
    out[1] = 66;                                              /* bits per record */
    out[2] = (nrec * 66 + 7) / 8;                             /* Fragment 1 bytes */
    out[3] = (uint64_t)width * height * channels;             /* Fragment 2 bytes = image */
    return 0;
}

/* ---- bit stream helpers (MSB-first, D6) ---------------------------------- */
static void put_bits(uint8_t* s, uint64_t pos, uint32_t v, int n) {
    for (int k = n - 1; k >= 0; --k, ++pos)
        if ((v >> k) & 1u) s[pos / 8] |= (uint8_t)(0x80u >> (pos % 8));
}

static uint32_t get_bits(const uint8_t* s, uint64_t pos, int n) {
    uint32_t v = 0;
    for (int k = 0; k < n; ++k, ++pos) v = (v << 1) | ((s[pos / 8] >> (7 - pos % 8)) & 1u);
    return v;
}

/* 11-bit store method (D5) */
static uint32_t store11(double q) {
    long m = lrint(fabs(q));
    if (m > 1023) m = 1023;
    return (q < 0 && m != 0 ? 1u << 10 : 0u) | (uint32_t)m;
}

static double load11(uint32_t w) { return (w >> 10) ? -(double)(w & 1023u) : (double)(w & 1023u); }

static void block_get(const uint8_t* img, uint32_t W, uint32_t ch, uint32_t nch, uint64_t br, uint64_t bc,
                      double f[64]) {
    for (int x = 0; x < 8; ++x)
        for (int y = 0; y < 8; ++y) f[x * 8 + y] = img[((8 * br + x) * W + 8 * bc + y) * nch + ch];
}

static void block_put(uint8_t* img, uint32_t W, uint32_t ch, uint32_t nch, uint64_t br, uint64_t bc,
                      const uint8_t p[64]) {
    for (int x = 0; x < 8; ++x)
        for (int y = 0; y < 8; ++y) img[((8 * br + x) * W + 8 * bc + y) * nch + ch] = p[x * 8 + y];
}

/* "round all iDCT coefficients to 8-bit unsigned integers" in [0, 255] (D3) */
static uint8_t to_u8(double v) {
    double r = rint(v);
    if (r < 0) r = 0;
    if (r > 255) r = 255;
    return (uint8_t)r;
}

/* Level-2 mask of one record (D9, D10). */
static void level2_digest(uint32_t flags, const uint8_t key[16], const uint8_t iv[16], uint64_t gr,
                          const uint8_t rec9[9], uint8_t dig[64]) {
    uint8_t m[49];
    size_t n = 0;
    if (flags & ORACLE_DCT_KEYED) {
        memcpy(m, key, 16);
        memcpy(m + 16, iv, 16);
        for (int k = 0; k < 8; ++k) m[32 + k] = (uint8_t)(gr >> (56 - 8 * k));
        n = 40;
    }
    memcpy(m + n, rec9, 9);
    oracle_sha512(m, n + 9, dig);
}

/* the 6 selected coefficients of one centered block, Eq. 4.1 / Eq. 4.4 */
static void select6(const double f[64], double c[64], double sel[6]) {
    double g[64];
    for (int k = 0; k < 64; ++k) g[k] = f[k] - 128.0;
    oracle_dct8_fwd(g, c);                                                         /* Eq. 4.1 */
    double s = 0.0;
    for (int k = 0; k < 64; ++k) s += g[k];
    c[0] = s / 8.0;                                  /* Eq. 4.4 (alpha(0)^2 = 1/8), exact (D4) */
    for (int k = 0; k < 6; ++k) sel[k] = c[kSel[k][0] * 8 + kSel[k][1]];
}

/* The full DCT 8x8 of an image (Table 4.1's operation): every block of
 * every layer, minus 128, by Eq. 4.1; coefficient (u, v) of block
 * (br, bc) of layer ch at ((8br + u) * W + 8bc + v) * channels + ch. */
int oracle_dct_image_fwd(uint32_t width, uint32_t height, uint32_t channels, const uint8_t* in, double* coef) {
    uint64_t lay[4];
    if (oracle_dct_layout(width, height, channels, lay)) return -1;
    for (uint64_t br = 0; br < height / 8; ++br)
        for (uint64_t bc = 0; bc < width / 8; ++bc)
            for (uint32_t ch = 0; ch < channels; ++ch) {
                double f[64], c[64];
                block_get(in, width, ch, channels, br, bc, f);
                for (int k = 0; k < 64; ++k) f[k] -= 128.0;
                oracle_dct8_fwd(f, c);
                for (int u = 0; u < 8; ++u)
                    for (int v = 0; v < 8; ++v) coef[((8 * br + u) * width + 8 * bc + v) * channels + ch] = c[u * 8 + v];
            }
    return 0;
}

/* Its inverse by Eq. 4.2, + 128, rounded to bytes in [0, 255] (D3). */
int oracle_dct_image_inv(uint32_t width, uint32_t height, uint32_t channels, const double* coef, uint8_t* out) {
    uint64_t lay[4];
    if (oracle_dct_layout(width, height, channels, lay)) return -1;
    for (uint64_t br = 0; br < height / 8; ++br)
        for (uint64_t bc = 0; bc < width / 8; ++bc)
            for (uint32_t ch = 0; ch < channels; ++ch) {
                double c[64], f[64];
                uint8_t b[64];
                for (int u = 0; u < 8; ++u)
                    for (int v = 0; v < 8; ++v) c[u * 8 + v] = coef[((8 * br + u) * width + 8 * bc + v) * channels + ch];
                oracle_dct8_inv(c, f);
                for (int k = 0; k < 64; ++k) b[k] = to_u8(f[k] + 128.0);
                block_put(out, width, ch, channels, br, bc, b);
            }
    return 0;
}

int oracle_dct_select(uint32_t width, uint32_t height, uint32_t channels, const uint8_t* in, double* coef6) {
    uint64_t lay[4];
    if (oracle_dct_layout(width, height, channels, lay)) return -1;
    const uint64_t bpr = width / 8, nb = height / 8;
    for (uint64_t br = 0; br < nb; ++br)
        for (uint64_t bc = 0; bc < bpr; ++bc)
            for (uint32_t ch = 0; ch < channels; ++ch) {
                double f[64], c[64];
                block_get(in, width, ch, channels, br, bc, f);
                select6(f, c, coef6 + ((br * bpr + bc) * channels + ch) * 6);
            }
    return 0;
}

int oracle_dct_protect(uint32_t width, uint32_t height, uint32_t channels, uint32_t level, uint32_t flags,
                       uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16], const uint8_t* in,
                       uint8_t* a, uint8_t* p, double* p_real) {
    uint64_t lay[4];
    if (oracle_dct_layout(width, height, channels, lay) || (level != 1 && level != 2)) return -1;
    if ((block_offset * 66) % 128) return -1;                                     /* D8 */
    memset(a, 0, lay[2]);
    const uint64_t bpr = width / 8, nb = height / 8;
    for (uint64_t br = 0; br < nb; ++br)
        for (uint64_t bc = 0; bc < bpr; ++bc)
            for (uint32_t ch = 0; ch < channels; ++ch) {
                const uint64_t r = (br * bpr + bc) * channels + ch;                /* D7 */
                double f[64], c[64], sel[6], g[64];
                block_get(in, width, ch, channels, br, bc, f);
                select6(f, c, sel);
                uint8_t rec9[9] = {0};
                for (int k = 0; k < 6; ++k) {                                     /* Fragment 1 */
                    uint32_t w = store11(sel[k]);
                    put_bits(a, r * 66 + 11 * k, w, 11);
                    put_bits(rec9, 11 * k, w, 11);
                }
                for (int k = 1; k < 6; ++k) c[kSel[k][0] * 8 + kSel[k][1]] = 0.0; /* P:1487 padding */
                c[0] = 1024.0;
                oracle_dct8_inv(c, g);                                             /* Eq. 4.2 */
                uint8_t pb[64];
                for (int k = 0; k < 64; ++k) {
                    pb[k] = to_u8(g[k]);
                    if (p_real) p_real[r * 64 + k] = g[k];
                }
                if (level == 2) {
                    uint8_t dig[64];
                    level2_digest(flags, key, iv, block_offset + r, rec9, dig);
                    for (int k = 0; k < 64; ++k) pb[k] ^= dig[k];                  /* D10 */
                }
                block_put(p, width, ch, channels, br, bc, pb);
            }
    oracle_aes128_ctr(key, iv, block_offset * 66 / 128, a, a, lay[2]);          /* P:1410, D8 */
    return 0;
}

int oracle_dct_recover(uint32_t width, uint32_t height, uint32_t channels, uint32_t level, uint32_t flags,
                       uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16], const uint8_t* a_enc,
                       const uint8_t* p, uint8_t* out, double* out_real) {
    uint64_t lay[4];
    if (oracle_dct_layout(width, height, channels, lay) || (level != 1 && level != 2)) return -1;
    if ((block_offset * 66) % 128) return -1;
    uint8_t* a = (uint8_t*)malloc(lay[2] ? lay[2] : 1);
    if (!a) return -1;
    oracle_aes128_ctr(key, iv, block_offset * 66 / 128, a_enc, a, lay[2]);
    const uint64_t bpr = width / 8, nb = height / 8;
    for (uint64_t br = 0; br < nb; ++br)
        for (uint64_t bc = 0; bc < bpr; ++bc)
            for (uint32_t ch = 0; ch < channels; ++ch) {
                const uint64_t r = (br * bpr + bc) * channels + ch;
                uint8_t rec9[9] = {0};
                double q[6];
                for (int k = 0; k < 6; ++k) {
                    uint32_t w = get_bits(a, r * 66 + 11 * k, 11);
                    put_bits(rec9, 11 * k, w, 11);
                    q[k] = load11(w);
                }
                double f[64], c[64], g[64];
                block_get(p, width, ch, channels, br, bc, f);
                if (level == 2) {
                    uint8_t dig[64];
                    level2_digest(flags, key, iv, block_offset + r, rec9, dig);
                    for (int k = 0; k < 64; ++k) f[k] = (double)((uint8_t)f[k] ^ dig[k]);
                }
                oracle_dct8_fwd(f, c);                                             /* Eq. 4.1, D12 */
                for (int k = 0; k < 6; ++k) c[kSel[k][0] * 8 + kSel[k][1]] = q[k];
                oracle_dct8_inv(c, g);                                             /* Eq. 4.2 */
                uint8_t ob[64];
                for (int k = 0; k < 64; ++k) {
                    g[k] += 128.0;                                                 /* undo P:1483 */
                    ob[k] = to_u8(g[k]);
                    if (out_real) out_real[r * 64 + k] = g[k];
                }
                block_put(out, width, ch, channels, br, bc, ob);
            }
    free(a);
    return 0;
}
