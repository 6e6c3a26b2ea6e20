/*
 * aes128.c — oracle: FIPS-197 AES-128 forward cipher + SP 800-38A CTR
 * (TEST INFRASTRUCTURE).
 *
 * The paper protects the private fragment with "AES-128"
 * without fixing a mode; reading C12 takes CTR over the whole A stream
 * ("AES has a counter mode ... in parallel"; length preserving, so
 * the 7.8% of P:2736 holds).  Reading C13: the caller's 16-byte IV is the
 * initial counter block; block j uses IV + j as a 128-bit big-endian integer
 * (SP 800-38A §B.1 standard incrementing function over the whole block).
 *
 * Byte-oriented and table-free: the S-box is computed from its definition
 * (FIPS-197 §5.1.1: multiplicative inverse in GF(2^8) mod x^8+x^4+x^3+x+1,
 * then the affine transform with c = 0x63); MixColumns uses xtime (§4.2.1).
 */
#include "oracle.h"
#include <string.h>

/* FIPS-197 §4.2: multiplication in GF(2^8) by repeated xtime. */
static uint8_t xtime(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0x00)); }
static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    for (int i = 0; i < 8; ++i) {
        if (b & 1) p ^= a;
        a = xtime(a);
        b >>= 1;
    }
    return p;
}
/* multiplicative inverse: a^254 (a^255 = 1 for a != 0); 0 maps to 0 */
static uint8_t ginv(uint8_t a) {
    if (a == 0) return 0;
    uint8_t r = 1;
    for (int i = 0; i < 254; ++i) r = gmul(r, a);
    return r;
}
static uint8_t rotl8(uint8_t x, int s) { return (uint8_t)((x << s) | (x >> (8 - s))); }

/* FIPS-197 §5.1.1 eq. (5.1): b' = b ^ b<<<1 ^ b<<<2 ^ b<<<3 ^ b<<<4 ^ 0x63 */
static uint8_t sbox_def(uint8_t x) {
    uint8_t b = ginv(x);
    return (uint8_t)(b ^ rotl8(b, 1) ^ rotl8(b, 2) ^ rotl8(b, 3) ^ rotl8(b, 4) ^ 0x63);
}

void oracle_aes128_sbox(uint8_t sbox[256]) {
    for (int i = 0; i < 256; ++i) sbox[i] = sbox_def((uint8_t)i);
}

/* FIPS-197 §5.2 KeyExpansion, Nk = 4, Nr = 10: 44 words as 176 bytes. */
static void key_expansion(const uint8_t key[16], const uint8_t sbox[256], uint8_t w[176]) {
    memcpy(w, key, 16);
    uint8_t rcon = 0x01;
    for (int i = 4; i < 44; ++i) {
        uint8_t t[4];
        memcpy(t, w + 4 * (i - 1), 4);
        if (i % 4 == 0) {
            uint8_t t0 = t[0];                       /* RotWord */
            t[0] = t[1]; t[1] = t[2]; t[2] = t[3]; t[3] = t0;
            for (int k = 0; k < 4; ++k) t[k] = sbox[t[k]];   /* SubWord */
            t[0] ^= rcon;                            /* Rcon[i/Nk] = x^(i/Nk - 1) */
            rcon = xtime(rcon);
        }
        for (int k = 0; k < 4; ++k) w[4 * i + k] = (uint8_t)(w[4 * (i - 4) + k] ^ t[k]);
    }
}

/* state s[r][c] = in[r + 4c] (FIPS-197 §3.4) */
static void add_round_key(uint8_t s[4][4], const uint8_t* rk) {
    for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) s[r][c] ^= rk[4 * c + r];
}
static void sub_bytes(uint8_t s[4][4], const uint8_t sbox[256]) {
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) s[r][c] = sbox[s[r][c]];
}
static void shift_rows(uint8_t s[4][4]) {               /* §5.1.2: row r left by r */
    uint8_t t[4];
    for (int r = 1; r < 4; ++r) {
        for (int c = 0; c < 4; ++c) t[c] = s[r][(c + r) % 4];
        for (int c = 0; c < 4; ++c) s[r][c] = t[c];
    }
}
static void mix_columns(uint8_t s[4][4]) {              /* §5.1.3 */
    for (int c = 0; c < 4; ++c) {
        uint8_t a0 = s[0][c], a1 = s[1][c], a2 = s[2][c], a3 = s[3][c];
        s[0][c] = (uint8_t)(gmul(a0, 2) ^ gmul(a1, 3) ^ a2 ^ a3);
        s[1][c] = (uint8_t)(a0 ^ gmul(a1, 2) ^ gmul(a2, 3) ^ a3);
        s[2][c] = (uint8_t)(a0 ^ a1 ^ gmul(a2, 2) ^ gmul(a3, 3));
        s[3][c] = (uint8_t)(gmul(a0, 3) ^ a1 ^ a2 ^ gmul(a3, 2));
    }
}

static void cipher(const uint8_t w[176], const uint8_t sbox[256], const uint8_t in[16], uint8_t out[16]) {
    uint8_t s[4][4];
    for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) s[r][c] = in[r + 4 * c];
    add_round_key(s, w);
    for (int round = 1; round < 10; ++round) {
        sub_bytes(s, sbox);
        shift_rows(s);
        mix_columns(s);
        add_round_key(s, w + 16 * round);
    }
    sub_bytes(s, sbox);
    shift_rows(s);
    add_round_key(s, w + 160);
    for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) out[r + 4 * c] = s[r][c];
}

void oracle_aes128_encrypt_block(const uint8_t key[16], const uint8_t in[16], uint8_t out[16]) {
    uint8_t sbox[256], w[176];
    oracle_aes128_sbox(sbox);
    key_expansion(key, sbox, w);
    cipher(w, sbox, in, out);
}

/* 128-bit big-endian add of a 64-bit value (SP 800-38A, wraps mod 2^128) */
static void counter_add(const uint8_t iv[16], uint64_t j, uint8_t out[16]) {
    unsigned carry = 0;
    for (int i = 15; i >= 0; --i) {
        unsigned add = (i >= 8) ? (unsigned)((j >> (8 * (15 - i))) & 0xFF) : 0u;
        unsigned v = (unsigned)iv[i] + add + carry;
        out[i] = (uint8_t)(v & 0xFF);
        carry = v >> 8;
    }
}

void oracle_aes128_ctr(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_offset,
                       const uint8_t* in, uint8_t* out, uint64_t n) {
    uint8_t sbox[256], w[176], base[16], ctr[16], ks[16];
    oracle_aes128_sbox(sbox);
    key_expansion(key, sbox, w);
    /* counter of block j = IV + ctr_offset + j, all mod 2^128 (two 128-bit adds,
     * so ctr_offset + j may exceed 2^64) */
    counter_add(iv, ctr_offset, base);
    for (uint64_t i = 0; i < n; i += 16) {
        counter_add(base, i / 16, ctr);
        cipher(w, sbox, ctr, ks);
        for (uint64_t k = 0; k < 16 && i + k < n; ++k) out[i + k] = in[i + k] ^ ks[k];
    }
}
