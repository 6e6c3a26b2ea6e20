/*
 * se_dct.h — C ABI of libse.so, part 2: the Chapter 4 DCT 8x8 selective
 * encryption of bitmaps (NEXT row f3 of SURVEY.md §8; PAPER.md "Design of SE
 * for bitmaps based on DCT").
 *
 * The operation.  A grey-scale image (each colour layer of a colour image is
 * handled as one) is cut into 8x8 blocks; each block, minus 128
 * (P:1483), goes through the DCT 8x8 of Eq. 4.1.  Per block:
 *   Fragment 1 (private): the coefficients [0,0],[0,1],[1,0],[2,0],[1,1],
 *     [0,2], rounded, each stored in 11 bits (sign + 10-bit
 *     magnitude): 66 bits per block; encrypted with
 *     AES-128.
 *   Fragment 2 (public): the iDCT (Eq. 4.2) of the block's coefficients with
 *     the DC padded with 1024 and the 5 selected AC padded with 0, rounded to
 *     bytes in [0, 255] — an image of the input's size.
 *   Level 1 leaves Fragment 2 plain; level 2 XORs its
 *     64 bytes with SHA-512 of the block's 6 selected coefficients.
 * Recovery puts the 6 stored values back into the DCT of
 * Fragment 2 and inverts; it is lossy by design (two roundings):
 * the paper reports PSNR ~ 62.8 dB (Table 4.2).
 *
 * Readings where the paper is silent (D1-D12): f(x,y) has x =
 * row; every rounding is round-half-to-even; the DC is rounded from Eq. 4.4
 * exactly; |q| saturates at 1023; records are MSB-first, concatenated in the
 * order r = ((br * W/8) + bc) * channels + ch; AES-128-CTR with counter
 * IV + block_offset*66/128 (C12/C13); the level-2 message is the 66-bit
 * record zero-padded to 9 bytes (flag SE_DCT_KEYED: K || IV || be64(block_offset
 * + r) || record, the Chapter 5 framing); digest byte 8x+y masks pixel (x,y).
 *
 * Arithmetic: fp32 (the paper's precision).  Only the 6 selected
 * coefficients are formed: Fragment 2 = x - (their iDCT) is the same real
 * number as the paper's pad-and-invert (f3), so results agree
 * with the fp64 oracle except where an fp32 value lies within ~1e-3 of a
 * rounding boundary (the tests compare everywhere else and check the rest is
 * off by one).  The DC, and hence its quantisation, is exact.
 *
 * Conventions as in se.h: device pointers caller-owned and 16-byte aligned
 * (SE_EALIGN), key/IV 16-byte host buffers read during the call, stream =
 * cudaStream_t as void*, asynchronous, status codes se_status.  Images are
 * raw pixel arrays (no BMP header), row-major, channels interleaved.
 */
#ifndef SE_DCT_H
#define SE_DCT_H
#include <stdint.h>

#include "se.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { SE_DCT_KEYED = 1u << 0 };   /* level 2: key, IV and record index in the hash (D9) */

/* width, height: pixels, multiples of 8 (D11) ; channels 1, 3 or 4 ;
 * level 1 or 2 ; block_offset: global record index of this image's first
 * record (CTR start and hash nonce), block_offset*66 a multiple of 128. */
typedef struct {
    uint32_t width, height, channels, level;
    uint32_t flags, reserved;
    uint64_t block_offset;
} se_dct_geom;

typedef struct {
    uint64_t records;      /* (W/8) * (H/8) * channels                        */
    uint64_t a_bytes;      /* Fragment 1: ceil(66 * records / 8)              */
    uint64_t p_bytes;      /* Fragment 2: W * H * channels (= input size)     */
    uint32_t a_bits;       /* 66 per record                          */
    uint32_t reserved;
} se_dct_layout;

/* Sizes of the fragments.  SE_EINVAL on bad geometry. */
int dct_layout(const se_dct_geom* g, se_dct_layout* out);

/* Protect one image: d_in (p_bytes) -> d_a (a_bytes, encrypted Fragment 1)
 * and d_p (p_bytes, Fragment 2, masked at level 2).  Level 1: one kernel
 * (DCT, records and their AES-CTR); level 2: the AES-CTR keystream into d_a,
 * then the DCT + SHA-512 kernel.  d_in must not alias d_a or d_p. */
int dct_protect(const se_dct_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_in,
                void* d_a, void* d_p, void* stream);

/* Rebuild the image from both fragments into d_out (p_bytes).  Lossy by
 * design (see above); a wrong key yields a wrong image, not an error.  One
 * kernel (AES-CTR of Fragment 1 inside). */
int dct_recover(const se_dct_geom* g, const uint8_t key[16], const uint8_t iv[16], const void* d_a,
                const void* d_p, void* d_out, void* stream);

/* Inspection: the 6 selected coefficients of every record as fp32 (records x
 * 6, order [0,0],[0,1],[1,0],[2,0],[1,1],[0,2]; [0,0] from Eq. 4.4 exactly),
 * before rounding.  g->level and key material are not used. */
int dct_select(const se_dct_geom* g, const void* d_in, float* d_coef, void* stream);

/* The DCT 8x8 itself (Eq. 4.1 / 4.2; the operation of Table 4.1),
 * fp32, for every 8x8 block of every layer.  dct8_forward: coefficients of
 * (pixel - 128) into d_coef (W*H*channels floats, pixel layout:
 * coefficient (u, v) of block (br, bc), layer ch at ((8br+u)*W + 8bc+v)*ch_n
 * + ch).  dct8_inverse: Eq. 4.2 + 128, rounded half-to-even and clamped to
 * [0, 255] (D3) into d_out.  g->level / flags / block_offset unused.
 * d_coef 16-byte aligned. */
int dct8_forward(const se_dct_geom* g, const void* d_in, float* d_coef, void* stream);
int dct8_inverse(const se_dct_geom* g, const float* d_coef, void* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
