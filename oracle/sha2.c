/*
 * sha2.c — oracle: FIPS 180-4 SHA-256 and SHA-512 (TEST INFRASTRUCTURE).
 *
 * The paper masks the first public fragment with "a 256-bit sequence by
 * using SHA-256" and the second with "a bit sequence generated from
 * SHA-512" (citing the FIPS hash standard).  This file follows FIPS
 * 180-4 §4.1.2/§4.1.3 (functions), §5.1 (padding), §6.2/§6.4 (computation).
 *
 * Constants are not typed in: they are computed from their definitions
 * (§4.2.2/§4.2.3: K = first 32/64 bits of the fractional parts of the cube
 * roots of the first 64/80 primes; §5.3.3/§5.3.5: H(0) = first 32/64 bits of
 * the fractional parts of the square roots of the first 8 primes) with exact
 * integer roots over a small 256-bit fixed-point.
 */
#include "oracle.h"
#include <string.h>

typedef unsigned __int128 u128;

/* ---- 256-bit unsigned helpers (4 little-endian 64-bit limbs) ------------ */
static void mul256(const uint64_t a[4], const uint64_t b[4], uint64_t r[4]) {
    uint64_t t[8] = {0};
    for (int i = 0; i < 4; ++i) {
        uint64_t carry = 0;
        for (int j = 0; j < 4; ++j) {
            u128 cur = (u128)a[i] * b[j] + t[i + j] + carry;
            t[i + j] = (uint64_t)cur;
            carry = (uint64_t)(cur >> 64);
        }
        t[i + 4] += carry;
    }
    for (int i = 0; i < 4; ++i) r[i] = t[i];   /* callers stay below 2^256 */
}
static int cmp256(const uint64_t a[4], const uint64_t b[4]) {
    for (int i = 3; i >= 0; --i) {
        if (a[i] < b[i]) return -1;
        if (a[i] > b[i]) return 1;
    }
    return 0;
}
/* largest y < 2^nbits with y^k <= N, k in {2,3}; returns y as 2 limbs */
static void iroot(const uint64_t N[4], int k, int nbits, uint64_t y[2]) {
    y[0] = y[1] = 0;
    for (int bit = nbits - 1; bit >= 0; --bit) {
        uint64_t t[4] = {y[0], y[1], 0, 0};
        t[bit / 64] |= (uint64_t)1 << (bit % 64);
        uint64_t p[4];
        mul256(t, t, p);
        if (k == 3) mul256(p, t, p);
        if (cmp256(p, N) <= 0) { y[0] = t[0]; y[1] = t[1]; }
    }
}
static int is_prime(int p) {
    if (p < 2) return 0;
    for (int d = 2; d * d <= p; ++d)
        if (p % d == 0) return 0;
    return 1;
}
static void first_primes(int count, int* out) {
    int n = 0;
    for (int p = 2; n < count; ++p)
        if (is_prime(p)) out[n++] = p;
}
/* first 64 fractional bits of p^(1/k):  floor(root(p * 2^(64k))) mod 2^64 */
static uint64_t frac_root64(int p, int k) {
    uint64_t N[4] = {0, 0, 0, 0};
    N[k] = (uint64_t)p;                         /* p * 2^(64k), k in {2,3} */
    uint64_t y[2];
    iroot(N, k, 72, y);                         /* root < 2^(64+9) */
    return y[0];
}

static uint64_t K512[80], H512[8];
static uint32_t K256[64], H256[8];
static int consts_ready = 0;

/* computed once at load (constructor) so concurrent callers never race */
__attribute__((constructor)) static void init_consts(void) {
    if (consts_ready) return;
    int primes[80];
    first_primes(80, primes);
    for (int t = 0; t < 80; ++t) K512[t] = frac_root64(primes[t], 3);
    for (int i = 0; i < 8; ++i) H512[i] = frac_root64(primes[i], 2);
    for (int t = 0; t < 64; ++t) K256[t] = (uint32_t)(K512[t] >> 32);   /* first 32 bits */
    for (int i = 0; i < 8; ++i) H256[i] = (uint32_t)(H512[i] >> 32);
    consts_ready = 1;
}

/* ---- SHA-256 (§4.1.2, §6.2) --------------------------------------------- */
static uint32_t rotr32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
static uint32_t ch32(uint32_t x, uint32_t y, uint32_t z) { return (x & y) ^ (~x & z); }
static uint32_t maj32(uint32_t x, uint32_t y, uint32_t z) { return (x & y) ^ (x & z) ^ (y & z); }
static uint32_t S0_256(uint32_t x) { return rotr32(x, 2) ^ rotr32(x, 13) ^ rotr32(x, 22); }
static uint32_t S1_256(uint32_t x) { return rotr32(x, 6) ^ rotr32(x, 11) ^ rotr32(x, 25); }
static uint32_t s0_256(uint32_t x) { return rotr32(x, 7) ^ rotr32(x, 18) ^ (x >> 3); }
static uint32_t s1_256(uint32_t x) { return rotr32(x, 17) ^ rotr32(x, 19) ^ (x >> 10); }

static void sha256_block(uint32_t H[8], const uint8_t* blk) {
    uint32_t W[64];
    for (int t = 0; t < 16; ++t)
        W[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
               ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
    for (int t = 16; t < 64; ++t)
        W[t] = s1_256(W[t - 2]) + W[t - 7] + s0_256(W[t - 15]) + W[t - 16];
    uint32_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
    for (int t = 0; t < 64; ++t) {
        uint32_t T1 = h + S1_256(e) + ch32(e, f, g) + K256[t] + W[t];
        uint32_t T2 = S0_256(a) + maj32(a, b, c);
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

void oracle_sha256(const uint8_t* msg, uint64_t len, uint8_t out[32]) {
    init_consts();
    uint32_t H[8];
    memcpy(H, H256, sizeof H);
    /* §5.1.1: append 1 bit, k zero bits, 64-bit big-endian bit length */
    uint64_t total = ((len + 8) / 64 + 1) * 64;
    uint8_t blk[64];
    for (uint64_t off = 0; off < total; off += 64) {
        for (int i = 0; i < 64; ++i) {
            uint64_t p = off + (uint64_t)i;
            uint8_t v;
            if (p < len) v = msg[p];
            else if (p == len) v = 0x80;
            else if (p >= total - 8) v = (uint8_t)(((len * 8) >> (8 * (total - 1 - p))) & 0xFF);
            else v = 0;
            blk[i] = v;
        }
        sha256_block(H, blk);
    }
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 4; ++k) out[4 * i + k] = (uint8_t)(H[i] >> (24 - 8 * k));
}

/* ---- SHA-512 (§4.1.3, §6.4) --------------------------------------------- */
static uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }
static uint64_t ch64(uint64_t x, uint64_t y, uint64_t z) { return (x & y) ^ (~x & z); }
static uint64_t maj64(uint64_t x, uint64_t y, uint64_t z) { return (x & y) ^ (x & z) ^ (y & z); }
static uint64_t S0_512(uint64_t x) { return rotr64(x, 28) ^ rotr64(x, 34) ^ rotr64(x, 39); }
static uint64_t S1_512(uint64_t x) { return rotr64(x, 14) ^ rotr64(x, 18) ^ rotr64(x, 41); }
static uint64_t s0_512(uint64_t x) { return rotr64(x, 1) ^ rotr64(x, 8) ^ (x >> 7); }
static uint64_t s1_512(uint64_t x) { return rotr64(x, 19) ^ rotr64(x, 61) ^ (x >> 6); }

static void sha512_block(uint64_t H[8], const uint8_t* blk) {
    uint64_t W[80];
    for (int t = 0; t < 16; ++t) {
        uint64_t v = 0;
        for (int k = 0; k < 8; ++k) v = (v << 8) | blk[8 * t + k];
        W[t] = v;
    }
    for (int t = 16; t < 80; ++t)
        W[t] = s1_512(W[t - 2]) + W[t - 7] + s0_512(W[t - 15]) + W[t - 16];
    uint64_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
    for (int t = 0; t < 80; ++t) {
        uint64_t T1 = h + S1_512(e) + ch64(e, f, g) + K512[t] + W[t];
        uint64_t T2 = S0_512(a) + maj64(a, b, c);
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

void oracle_sha512(const uint8_t* msg, uint64_t len, uint8_t out[64]) {
    init_consts();
    uint64_t H[8];
    memcpy(H, H512, sizeof H);
    /* §5.1.2: 1 bit, zeros, 128-bit big-endian length (high 64 bits zero here) */
    uint64_t total = ((len + 16) / 128 + 1) * 128;
    uint8_t blk[128];
    for (uint64_t off = 0; off < total; off += 128) {
        for (int i = 0; i < 128; ++i) {
            uint64_t p = off + (uint64_t)i;
            uint8_t v;
            if (p < len) v = msg[p];
            else if (p == len) v = 0x80;
            else if (p >= total - 8) v = (uint8_t)(((len * 8) >> (8 * (total - 1 - p))) & 0xFF);
            else v = 0;
            blk[i] = v;
        }
        sha512_block(H, blk);
    }
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 8; ++k) out[8 * i + k] = (uint8_t)(H[i] >> (56 - 8 * k));
}
