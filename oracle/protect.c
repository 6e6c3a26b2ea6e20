/*
 * protect.c — oracle: fragmentation, storage layout and protection of the
 * Chapter 5 agnostic SE scheme (TEST INFRASTRUCTURE).
 *
 * Follows, in the paper's order (PAPER.md "Design of DWT based SE"):
 *   1. bytes -> chunk matrix -> 8x8 blocks
 *   2. 2-level 5/3 DWT per block                          (dwt53.c)
 *   3. private fragment A = 2nd-level LL ("4 out of 64")
 *      1st public fragment B = rest of the 2nd level
 *      2nd public fragment C = 1st-level details          (C25)
 *   4. storage: 10-bit fields, 11-bit for 2nd HH -> 40/124/480 bits
 *
 *   5. A protected with AES-128                           (CTR, C12)
 *      B ^= SHA-256(key, A)                               (framing C15)
 *      C ^= SHA-512(B', key)                              (C19)
 *   recover = the exact inverse
 * Readings C9–C26:
 *   C9  field value v stored offset-binary u = v + 2^(w-1) in w bits.
 *   C10 record order: A = LL_L row-major; B = HL_l, LH_l, HH_l for
 *       l = L..2 (each row-major); C = HL1, LH1, HH1 (each row-major).
 *   C11 records concatenated densely, MSB-first, in block order.
 *   C13 CTR counter = IV + (global A-stream byte / 16).
 *   C15 M_B = K || IV || be64(b) || bytes(A_b);  M_C = K || IV || be64(b) ||
 *       bytes(B'_b)  (bytes() = record bits MSB-first, zero-padded to bytes).
 *   C16 b = global block index (block_offset + local index).
 *   C17 the first |B| (|C|) digest bits, MSB-first, are XORed on the record.
 *   C21 L = 1: A = LL1 (160 b), B empty, M_C hashes bytes(A_b) (plain);
 *       L = 3: A = LL3, B = level-3 then level-2 details (155 b).
 *   C22/C23 widths: BLOCK8 HH_l (l >= 2) 11 bits, all else 10;
 *       FULL: every B field 11 bits, A and C fields 10 bits.
 *   C26 flags bit0 PUBLIC_PLAIN: B and C left unmasked.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

enum { LL = 0, HL = 1, LH = 2, HH = 3 };

/* ---- record field lists (C10, C21–C23) ----------------------------------- */
typedef struct { int level, band, row, col, width; } field;

static int band_fields(field* f, int n, int level, int band, int width) {
    int s = 8 >> level;                       /* band side inside one 8x8 footprint */
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) {
            f[n].level = level; f[n].band = band; f[n].row = i; f[n].col = j;
            f[n].width = width; ++n;
        }
    return n;
}

static int record_fields(int L, int mode, int stream, field* f) {
    int n = 0;
    if (stream == 0) {
        n = band_fields(f, n, L, LL, 10);
    } else if (stream == 1) {
        for (int l = L; l >= 2; --l) {
            int wd = (mode == 1) ? 11 : 10;
            n = band_fields(f, n, l, HL, wd);
            n = band_fields(f, n, l, LH, wd);
            n = band_fields(f, n, l, HH, 11);
        }
    } else {
        n = band_fields(f, n, 1, HL, 10);
        n = band_fields(f, n, 1, LH, 10);
        n = band_fields(f, n, 1, HH, 10);
    }
    return n;
}

int oracle_record_fields(uint32_t levels, uint32_t mode, int stream, int32_t* level,
                         int32_t* band, int32_t* row, int32_t* col, int32_t* width) {
    field f[64];
    int n = record_fields((int)levels, (int)mode, stream, f);
    for (int k = 0; k < n; ++k) {
        level[k] = f[k].level; band[k] = f[k].band; row[k] = f[k].row;
        col[k] = f[k].col; width[k] = f[k].width;
    }
    return n;
}

static int record_bits(int L, int mode, int stream) {
    field f[64];
    int n = record_fields(L, mode, stream, f), bits = 0;
    for (int k = 0; k < n; ++k) bits += f[k].width;
    return bits;
}

static uint64_t rows_of(uint64_t n, uint32_t w) {
    uint64_t r = (n + w - 1) / w;
    return (r + 7) / 8 * 8;
}

int oracle_layout(uint64_t n, uint32_t w, uint32_t L, uint32_t mode, uint64_t out[8]) {
    if (w == 0 || w % 8 || L < 1 || L > 3 || mode > 1) return -1;
    uint64_t R = rows_of(n, w);
    uint64_t nb = (R / 8) * (w / 8);
    out[0] = R; out[1] = nb;
    for (int s = 0; s < 3; ++s) {
        uint64_t bits = (uint64_t)record_bits((int)L, (int)mode, s);
        out[2 + s] = bits;
        out[5 + s] = (nb * bits + 7) / 8;
    }
    return 0;
}

/* ---- bit I/O, MSB-first (C11) ------------------------------------------- */
static void put_bit(uint8_t* s, uint64_t pos, int bit) {
    uint8_t m = (uint8_t)(0x80u >> (pos % 8));
    if (bit) s[pos / 8] |= m; else s[pos / 8] &= (uint8_t)~m;
}
static int get_bit(const uint8_t* s, uint64_t pos) { return (s[pos / 8] >> (7 - pos % 8)) & 1; }
static void put_bits(uint8_t* s, uint64_t pos, uint32_t v, int w) {
    for (int i = 0; i < w; ++i) put_bit(s, pos + (uint64_t)i, (int)((v >> (w - 1 - i)) & 1u));
}
static uint32_t get_bits(const uint8_t* s, uint64_t pos, int w) {
    uint32_t v = 0;
    for (int i = 0; i < w; ++i) v = (v << 1) | (uint32_t)get_bit(s, pos + (uint64_t)i);
    return v;
}

/* ---- coefficient addressing -------------------------------------------- */
/* BLOCK8: inside the 8x8 dyadic block.  FULL: inside the R x W Mallat matrix,
 * at footprint (br, bc). */
static int64_t coef_index(int mode, uint64_t R, uint32_t W, uint64_t br, uint64_t bc,
                          const field* f) {
    if (mode == 0) {
        int s = 8 >> f->level;
        int ro = (f->band == LH || f->band == HH) ? s : 0;
        int co = (f->band == HL || f->band == HH) ? s : 0;
        return (int64_t)((ro + f->row) * 8 + co + f->col);
    }
    uint64_t rs = R >> f->level, cs = W >> f->level;
    uint64_t ro = (f->band == LH || f->band == HH) ? rs : 0;
    uint64_t co = (f->band == HL || f->band == HH) ? cs : 0;
    uint64_t r = ro + ((8 * br) >> f->level) + (uint64_t)f->row;
    uint64_t c = co + ((8 * bc) >> f->level) + (uint64_t)f->col;
    return (int64_t)(r * W + c);
}

static int32_t centered(const uint8_t* in, uint64_t n, uint32_t w, uint64_t r, uint64_t c) {
    uint64_t idx = r * w + c;
    return (int32_t)((idx < n) ? in[idx] : 0) - 128;
}

/* record -> whole bytes, MSB-first, zero pad (C15) */
static int record_bytes(const uint8_t* rec, int bits, uint8_t* out) {
    int nbytes = (bits + 7) / 8;
    memset(out, 0, (size_t)nbytes);
    for (int i = 0; i < bits; ++i) put_bit(out, (uint64_t)i, get_bit(rec, (uint64_t)i));
    return nbytes;
}

/* D = SHA-256/512(K || IV || be64(b) || bytes(rec)); rec ^= first bits of D */
static void mask_record(int use512, const uint8_t key[16], const uint8_t iv[16],
                        uint64_t gb, const uint8_t* src_rec, int src_bits,
                        uint8_t* dst_rec, int dst_bits) {
    uint8_t msg[128], dig[64];
    memcpy(msg, key, 16);
    memcpy(msg + 16, iv, 16);
    for (int i = 0; i < 8; ++i) msg[32 + i] = (uint8_t)(gb >> (56 - 8 * i));
    int len = 40 + record_bytes(src_rec, src_bits, msg + 40);
    if (use512) oracle_sha512(msg, (uint64_t)len, dig);
    else oracle_sha256(msg, (uint64_t)len, dig);
    for (int i = 0; i < dst_bits; ++i)
        put_bit(dst_rec, (uint64_t)i, get_bit(dst_rec, (uint64_t)i) ^ get_bit(dig, (uint64_t)i));
}

/* A stream CTR over local bytes [p0, p1) (C12, C13) */
static void ctr_range(const uint8_t key[16], const uint8_t iv[16], uint64_t base_byte,
                      uint8_t* a, uint64_t p0, uint64_t p1) {
    if (p1 <= p0) return;
    /* keystream for global A bytes [base+p0, base+p1): KS block j = AES_K(IV + j) */
    uint64_t first = base_byte + p0, skip = first % 16, len = p1 - p0;
    uint8_t* ks = (uint8_t*)calloc((size_t)(skip + len), 1);
    oracle_aes128_ctr(key, iv, first / 16, ks, ks, skip + len);   /* 0 ^ KS = KS */
    for (uint64_t p = p0; p < p1; ++p) a[p] ^= ks[skip + (p - p0)];
    free(ks);
}

static int check_range_args(uint64_t nb, uint64_t b0, uint64_t b1) { return b0 <= b1 && b1 <= nb; }

static uint64_t stream_end(uint64_t b, uint64_t nb, uint64_t bits) {
    return (b == nb) ? (nb * bits + 7) / 8 : (b * bits) / 8;
}

int oracle_protect_range(uint64_t n, uint32_t w, uint32_t L, uint32_t mode, uint32_t flags,
                         uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16],
                         const uint8_t* in, uint8_t* a, uint8_t* b, uint8_t* c,
                         uint64_t b0, uint64_t b1) {
    uint64_t lay[8];
    if (oracle_layout(n, w, L, mode, lay)) return -1;
    uint64_t R = lay[0], nb = lay[1];
    int abits = (int)lay[2], bbits = (int)lay[3], cbits = (int)lay[4];
    if (!check_range_args(nb, b0, b1)) return -1;
    if ((block_offset * (uint64_t)abits) % 8) return -1;
    field fa[64], fb[64], fc[64];
    int na = record_fields((int)L, (int)mode, 0, fa);
    int nbf = record_fields((int)L, (int)mode, 1, fb);
    int nc = record_fields((int)L, (int)mode, 2, fc);

    int32_t* full = NULL;
    if (mode == 1) {                        /* a11: whole-matrix Mallat DWT */
        full = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R * w));
        for (uint64_t r = 0; r < R; ++r)
            for (uint64_t col = 0; col < w; ++col) full[r * w + col] = centered(in, n, w, r, col);
        oracle_dwt2_fwd_region(full, w, (int)R, (int)w, (int)L);
    }
    uint64_t bpr = w / 8;
    for (uint64_t blk = b0; blk < b1; ++blk) {
        uint64_t br = blk / bpr, bc = blk % bpr;
        int32_t x[64];
        const int32_t* src;
        if (mode == 0) {
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) x[i * 8 + j] = centered(in, n, w, 8 * br + i, 8 * bc + j);
            oracle_dwt2_fwd_region(x, 8, 8, 8, (int)L);
            src = x;
        } else {
            src = full;
        }
        uint8_t ra[64] = {0}, rb[64] = {0}, rc[64] = {0};
        const field* fl[3] = {fa, fb, fc};
        int cnt[3] = {na, nbf, nc};
        uint8_t* rec[3] = {ra, rb, rc};
        for (int s = 0; s < 3; ++s) {
            int pos = 0;
            for (int k = 0; k < cnt[s]; ++k) {
                int32_t v = src[coef_index((int)mode, R, w, br, bc, &fl[s][k])];
                int wd = fl[s][k].width;
                int32_t u = v + (1 << (wd - 1));                  /* C9 */
                if (u < 0 || u >= (1 << wd)) { free(full); return -2; }
                put_bits(rec[s], (uint64_t)pos, (uint32_t)u, wd);
                pos += wd;
            }
        }
        if (!(flags & 1u)) {
            uint64_t gb = block_offset + blk;
            if (bbits) mask_record(0, key, iv, gb, ra, abits, rb, bbits);       /* B' */
            if (bbits) mask_record(1, key, iv, gb, rb, bbits, rc, cbits);       /* C' */
            else mask_record(1, key, iv, gb, ra, abits, rc, cbits);             /* C21 */
        }
        for (int i = 0; i < abits; ++i) put_bit(a, blk * (uint64_t)abits + (uint64_t)i, get_bit(ra, (uint64_t)i));
        for (int i = 0; i < bbits; ++i) put_bit(b, blk * (uint64_t)bbits + (uint64_t)i, get_bit(rb, (uint64_t)i));
        for (int i = 0; i < cbits; ++i) put_bit(c, blk * (uint64_t)cbits + (uint64_t)i, get_bit(rc, (uint64_t)i));
    }
    free(full);
    /* zero the pad bits of each stream's final byte (C11) */
    if (b1 == nb && nb) {
        uint64_t ends[3] = {nb * (uint64_t)abits, nb * (uint64_t)bbits, nb * (uint64_t)cbits};
        uint8_t* st[3] = {a, b, c};
        for (int s = 0; s < 3; ++s)
            for (uint64_t p = ends[s]; p % 8; ++p) put_bit(st[s], p, 0);
    }
    /* AES-128-CTR over the A bytes of this range (C12, C13) */
    ctr_range(key, iv, block_offset * (uint64_t)abits / 8, a,
              stream_end(b0, nb, (uint64_t)abits), stream_end(b1, nb, (uint64_t)abits));
    return 0;
}

int oracle_protect(uint64_t n, uint32_t w, uint32_t L, uint32_t mode, uint32_t flags,
                   uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16],
                   const uint8_t* in, uint8_t* a, uint8_t* b, uint8_t* c) {
    uint64_t lay[8];
    if (oracle_layout(n, w, L, mode, lay)) return -1;
    return oracle_protect_range(n, w, L, mode, flags, block_offset, key, iv, in, a, b, c, 0, lay[1]);
}

int oracle_recover_range(uint64_t n, uint32_t w, uint32_t L, uint32_t mode, uint32_t flags,
                         uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16],
                         const uint8_t* a, const uint8_t* b, const uint8_t* c, uint8_t* out,
                         int64_t report[2], uint64_t b0, uint64_t b1) {
    uint64_t lay[8];
    if (oracle_layout(n, w, L, mode, lay)) return -1;
    uint64_t R = lay[0], nb = lay[1];
    int abits = (int)lay[2], bbits = (int)lay[3], cbits = (int)lay[4];
    if (!check_range_args(nb, b0, b1)) return -1;
    if ((block_offset * (uint64_t)abits) % 8) return -1;
    report[0] = -1; report[1] = 0;
    field fa[64], fb[64], fc[64];
    int na = record_fields((int)L, (int)mode, 0, fa);
    int nbf = record_fields((int)L, (int)mode, 1, fb);
    int nc = record_fields((int)L, (int)mode, 2, fc);
    const field* fl[3] = {fa, fb, fc};
    int cnt[3] = {na, nbf, nc};

    /* FULL mode needs every footprint's coefficients for the inverse. */
    uint64_t u0 = (mode == 1) ? 0 : b0, u1 = (mode == 1) ? nb : b1;
    uint8_t* aplain = (uint8_t*)malloc((size_t)lay[5] + 1);
    memcpy(aplain, a, (size_t)lay[5]);
    ctr_range(key, iv, block_offset * (uint64_t)abits / 8, aplain,
              stream_end(u0, nb, (uint64_t)abits), stream_end(u1, nb, (uint64_t)abits));
    int32_t* full = NULL;
    if (mode == 1) full = (int32_t*)calloc((size_t)(R * w), sizeof(int32_t));
    uint64_t bpr = w / 8;
    for (uint64_t blk = u0; blk < u1; ++blk) {
        uint64_t br = blk / bpr, bc = blk % bpr;
        uint8_t ra[64] = {0}, rb[64] = {0}, rc[64] = {0};
        for (int i = 0; i < abits; ++i) put_bit(ra, (uint64_t)i, get_bit(aplain, blk * (uint64_t)abits + (uint64_t)i));
        for (int i = 0; i < bbits; ++i) put_bit(rb, (uint64_t)i, get_bit(b, blk * (uint64_t)bbits + (uint64_t)i));
        for (int i = 0; i < cbits; ++i) put_bit(rc, (uint64_t)i, get_bit(c, blk * (uint64_t)cbits + (uint64_t)i));
        if (!(flags & 1u)) {
            uint64_t gb = block_offset + blk;
            if (bbits) mask_record(1, key, iv, gb, rb, bbits, rc, cbits);   /* C from B' */
            else mask_record(1, key, iv, gb, ra, abits, rc, cbits);
            if (bbits) mask_record(0, key, iv, gb, ra, abits, rb, bbits);   /* B from A */
        }
        int32_t x[64];
        memset(x, 0, sizeof x);
        int32_t* dst = (mode == 0) ? x : full;
        uint8_t* rec[3] = {ra, rb, rc};
        for (int s = 0; s < 3; ++s) {
            int pos = 0;
            for (int k = 0; k < cnt[s]; ++k) {
                int wd = fl[s][k].width;
                int32_t v = (int32_t)get_bits(rec[s], (uint64_t)pos, wd) - (1 << (wd - 1));
                dst[coef_index((int)mode, R, w, br, bc, &fl[s][k])] = v;
                pos += wd;
            }
        }
        if (mode == 0) {
            oracle_dwt2_inv_region(x, 8, 8, 8, (int)L);
            int badblk = 0;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    int32_t v = x[i * 8 + j] + 128;
                    if (v < 0 || v > 255) badblk = 1;
                    uint64_t idx = (8 * br + (uint64_t)i) * w + 8 * bc + (uint64_t)j;
                    if (idx < n) out[idx] = (uint8_t)(v & 0xFF);
                }
            if (badblk) {
                if (report[0] < 0) report[0] = (int64_t)blk;
                report[1]++;
            }
        }
    }
    if (mode == 1) {
        oracle_dwt2_inv_region(full, w, (int)R, (int)w, (int)L);
        for (uint64_t blk = b0; blk < b1; ++blk) {
            uint64_t br = blk / bpr, bc = blk % bpr;
            int badblk = 0;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    uint64_t idx = (8 * br + (uint64_t)i) * w + 8 * bc + (uint64_t)j;
                    int32_t v = full[idx] + 128;
                    if (v < 0 || v > 255) badblk = 1;
                    if (idx < n) out[idx] = (uint8_t)(v & 0xFF);
                }
            if (badblk) {
                if (report[0] < 0) report[0] = (int64_t)blk;
                report[1]++;
            }
        }
    }
    free(full);
    free(aplain);
    return 0;
}

int oracle_recover(uint64_t n, uint32_t w, uint32_t L, uint32_t mode, uint32_t flags,
                   uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16],
                   const uint8_t* a, const uint8_t* b, const uint8_t* c, uint8_t* out,
                   int64_t report[2]) {
    uint64_t lay[8];
    if (oracle_layout(n, w, L, mode, lay)) return -1;
    return oracle_recover_range(n, w, L, mode, flags, block_offset, key, iv, a, b, c, out,
                                report, 0, lay[1]);
}
