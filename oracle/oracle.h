/*
 * oracle.h — CPU ORACLE for the Chapter 5 agnostic selective-encryption path
 * of arxiv/paper_1803_04880 (PAPER.md, "Design of DWT based SE").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product (libse.so, paper_1803_04880_b200/) never links, includes or
 * calls anything in this directory, and this directory never includes the
 * product's headers: the two share no code, tables or constant generators.
 *
 * The oracle is deliberately plain and slow: scalar lifting with explicit
 * extension, floor division written out, bit-by-bit packing, byte-oriented
 * FIPS-197 AES whose S-box is computed from its GF(2^8) definition, FIPS
 * 180-4 SHA-2 whose constants are computed from the fractional parts of
 * prime roots.  Every function cites the passage it follows.  Where the
 * paper is silent, the reading is the one frozen in SURVEY.md §8.4.1
 * (C1–C26) and listed in DESIGN.md §3.
 *
 * Conventions (all integers little-endian in memory; byte streams MSB-first):
 *   geometry  n bytes -> W x R matrix, W % 8 == 0, R = ceil(n/W) rounded up
 *             to a multiple of 8, zero fill (C18).
 *   blocks    8x8, row-major block order b = br*(W/8) + bc (C11).
 *   mode 0    BLOCK8: per-block 2-D DWT (C1).  mode 1: FULL-matrix DWT (a11).
 *
 * Parity unpinned: the byte-level conventions C9–C21
 * (field encoding, record order, hash framing, digest truncation) are
 * frozen readings the paper cannot confirm; they are cross-checked only by
 * round trip and by re-deriving the masks with hashlib in the tests.
 */
#ifndef SE_ORACLE_H
#define SE_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- layout (C21–C23) ---------------------------
 * out[0]=rows R, out[1]=n_blocks, out[2]=a_bits, out[3]=b_bits,
 * out[4]=c_bits, out[5]=a_bytes, out[6]=b_bytes, out[7]=c_bytes.
 * Returns 0, or -1 on invalid geometry. */
int oracle_layout(uint64_t n_bytes, uint32_t width, uint32_t levels,
                  uint32_t mode, uint64_t out[8]);

/* ---- 1-D lifting, Eq. 5.1–5.2 with C2/C3/C4/C6 ------------ */
void oracle_lift_fwd_1d(const int32_t* x, int32_t* y, int n);
void oracle_lift_inv_1d(const int32_t* y, int32_t* x, int n);

/* ---- 2-D DWT of the whole input, coefficient matrix R x W (int32) -------
 * mode 0: per 8x8 block, dyadic layout inside each block.
 * mode 1: Mallat layout over the whole matrix (a11).  Input centered by
 * subtracting 128 (C8).  dwt_inv writes exactly n_bytes bytes and returns
 * the number of reconstructed samples outside [0,255]. */
int oracle_dwt_fwd(const uint8_t* in, uint64_t n_bytes, uint32_t width,
                   uint32_t levels, uint32_t mode, int32_t* coef);
int64_t oracle_dwt_inv(const int32_t* coef, uint64_t n_bytes, uint32_t width,
                       uint32_t levels, uint32_t mode, uint8_t* out);

/* ---- FIPS-197 AES-128 and SP 800-38A CTR (C12, C13) -------------------- */
void oracle_aes128_sbox(uint8_t sbox[256]);
void oracle_aes128_encrypt_block(const uint8_t key[16], const uint8_t in[16],
                                 uint8_t out[16]);
/* out[i] = in[i] ^ KS, KS block j = AES_K(IV + ctr_offset + j) (128-bit BE) */
void oracle_aes128_ctr(const uint8_t key[16], const uint8_t iv[16],
                       uint64_t ctr_offset, const uint8_t* in, uint8_t* out,
                       uint64_t n);

/* ---- FIPS 180-4 SHA-256 / SHA-512 -------------------------------------- */
void oracle_sha256(const uint8_t* msg, uint64_t len, uint8_t out[32]);
void oracle_sha512(const uint8_t* msg, uint64_t len, uint8_t out[64]);

/* ---- protect / recover (C9–C26) --------------------
 * Streams a, b, c must be sized from oracle_layout (a_bytes, b_bytes,
 * c_bytes).  block_offset = global index of this input's first block
 * (hash nonce, C16) — the A-stream counter starts at
 * block_offset*a_bits/128, which must be integral.
 * The *_range variants process local blocks [b0, b1) only; b0*bits and
 * b1*bits must be multiples of 8 for every stream unless b1 == n_blocks.
 * flags bit0 = PUBLIC_PLAIN (C26: skip the SHA masks). */
int oracle_protect_range(uint64_t n_bytes, uint32_t width, uint32_t levels,
                         uint32_t mode, uint32_t flags, uint64_t block_offset,
                         const uint8_t key[16], const uint8_t iv[16],
                         const uint8_t* in, uint8_t* a, uint8_t* b, uint8_t* c,
                         uint64_t b0, uint64_t b1);
int oracle_protect(uint64_t n_bytes, uint32_t width, uint32_t levels,
                   uint32_t mode, uint32_t flags, uint64_t block_offset,
                   const uint8_t key[16], const uint8_t iv[16],
                   const uint8_t* in, uint8_t* a, uint8_t* b, uint8_t* c);
/* report[0] = first bad local block or -1, report[1] = number of bad blocks
 * (a block is bad if any reconstructed sample falls outside [0,255]). */
int oracle_recover_range(uint64_t n_bytes, uint32_t width, uint32_t levels,
                         uint32_t mode, uint32_t flags, uint64_t block_offset,
                         const uint8_t key[16], const uint8_t iv[16],
                         const uint8_t* a, const uint8_t* b, const uint8_t* c,
                         uint8_t* out, int64_t report[2],
                         uint64_t b0, uint64_t b1);
int oracle_recover(uint64_t n_bytes, uint32_t width, uint32_t levels,
                   uint32_t mode, uint32_t flags, uint64_t block_offset,
                   const uint8_t key[16], const uint8_t iv[16],
                   const uint8_t* a, const uint8_t* b, const uint8_t* c,
                   uint8_t* out, int64_t report[2]);

/* ---- security battery sums (NEXT row f2) -------------------- */
#define ORACLE_STATS_WORDS (1 + 256 + 256 + 6 + 18)
void oracle_stats(const uint8_t* x, const uint8_t* y, uint64_t n, uint32_t width, uint64_t* out,
                  uint64_t* joint);

/* ---- Chapter 4 DCT 8x8 selective encryption (NEXT row f3, dct.c) --------
 * Readings D1-D12 in dct.c and DESIGN.md §3.  Image W x H (multiples of 8)
 * with `channels` interleaved layers; records of 66 bits. */
#define ORACLE_DCT_KEYED 1u
void oracle_dct_basis(double m[64]);                       /* Eq. 4.6, m[x*8+u] */
void oracle_dct8_fwd(const double f[64], double c[64]);    /* Eq. 4.1 */
void oracle_dct8_inv(const double c[64], double f[64]);    /* Eq. 4.2 */
/* out[0]=records, out[1]=66, out[2]=Fragment-1 bytes, out[3]=Fragment-2 bytes */
int oracle_dct_layout(uint32_t width, uint32_t height, uint32_t channels, uint64_t out[4]);
/* full DCT 8x8 of an image minus 128 (Eq. 4.1), coefficients in pixel layout;
 * and its inverse (Eq. 4.2) + 128 rounded to bytes (Table 4.1's operation) */
int oracle_dct_image_fwd(uint32_t width, uint32_t height, uint32_t channels, const uint8_t* in, double* coef);
int oracle_dct_image_inv(uint32_t width, uint32_t height, uint32_t channels, const double* coef, uint8_t* out);
/* the 6 selected real coefficients per record (DC from Eq. 4.4) */
int oracle_dct_select(uint32_t width, uint32_t height, uint32_t channels, const uint8_t* in, double* coef6);
/* p_real / out_real (optional, 64 doubles per record, block row-major):
 * the real values before rounding to bytes (used by the tests to find ties). */
int oracle_dct_protect(uint32_t width, uint32_t height, uint32_t channels, uint32_t level, uint32_t flags,
                       uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16], const uint8_t* in,
                       uint8_t* a, uint8_t* p, double* p_real);
int oracle_dct_recover(uint32_t width, uint32_t height, uint32_t channels, uint32_t level, uint32_t flags,
                       uint64_t block_offset, const uint8_t key[16], const uint8_t iv[16], const uint8_t* a,
                       const uint8_t* p, uint8_t* out, double* out_real);

/* ---- exposed internals used by the pins --------------------------------- */
/* Multi-level dyadic 2-D lifting in place on the top-left rows x cols region
 * of an int32 array with row stride `stride` (any magnitude; used by the
 * tests to read off the exact linear weights with 2^20 impulses). */
void oracle_dwt2_fwd_region(int32_t* a, size_t stride, int rows, int cols, int levels);
void oracle_dwt2_inv_region(int32_t* a, size_t stride, int rows, int cols, int levels);
/* The coefficient list of one record: for stream s (0=A,1=B,2=C), entry k
 * gives level, band (0=LL,1=HL,2=LH,3=HH), row, col inside the band, and
 * field width.  Returns the number of entries. */
int oracle_record_fields(uint32_t levels, uint32_t mode, int stream,
                         int32_t* level, int32_t* band, int32_t* row,
                         int32_t* col, int32_t* width);

#ifdef __cplusplus
}
#endif
#endif
