/*
 * se_container.h — C ABI of libse.so, part 3: fragment containers and
 * dispersion layouts (NEXT row f4 of SURVEY.md §8; host-only, no GPU).
 *
 * The paper stores the fragments of a chunk in different places: the private
 * fragment locally or on a direct channel, the public and protected ones on
 * (different) cloud servers (Figs. 5.16-5.17).  Two
 * placements are named:
 *   SE_LAYOUT_A_LOCAL   A local (40 b / block, 7.8 %), B and C remote — for a
 *                       reliable channel; local storage is minimal;
 *   SE_LAYOUT_AB_LOCAL  A and B local (164 b / block, 32.0 %), C remote —
 *                       for an unreliable channel: a bit error in C' then
 *                       stays a 1-bit error in C after unmasking.
 * Total storage is 644 b per 512 b block, "about 26 % more".  For
 * the Chapter 4 DCT scheme the private Fragment 1 is local and Fragment 2
 * remote ("dispersion step ... separate the storage of the two parts").
 *
 * The paper defines no on-disk format; this one (SEFR v1) is this library's
 * (f4).  A container holds a public header and one or more
 * fragment streams with SHA-256 content digests, so corruption at rest or in
 * transit is detected before any decryption — and can be bypassed (verify =
 * 0) to exercise the paper's error-confinement property.  No key material is
 * ever written; the IV is public (it is the CTR nonce).
 *
 * Wire format, all integers little-endian, every stream 8-byte aligned:
 *   0   4  magic "SEFR"
 *   4   2  version = 1             6   2  header bytes = 72
 *   8   4  scheme (SE_SCHEME_*)    12  4  flags (SE_FLAG_* / SE_DCT_KEYED)
 *   16  4  levels (DWT) or protection level (DCT)
 *   20  4  width                   24  4  height (DCT; 0 for DWT)
 *   28  4  channels (DCT; 1 for DWT)
 *   32  8  n_bytes (original length)   40  8  block_offset
 *   48 16  IV                      64  4  entry count E   68  4  reserved 0
 *   72 + 56 e: entry e: u32 stream id (SE_STREAM_*), u32 reserved 0,
 *              u64 offset (from the container start), u64 length,
 *              u8[32] SHA-256 of the stream bytes
 *   streams at their offsets, in entry order, zero padding between.
 * Stream lengths must equal the layout's (fragment_layout / dct_layout of the
 * header's geometry): a container is self-describing and checkable.
 */
#ifndef SE_CONTAINER_H
#define SE_CONTAINER_H
#include <stdint.h>

#include "se.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { SE_SCHEME_DWT_BLOCK8 = 1, SE_SCHEME_DWT_FULL = 2, SE_SCHEME_DCT = 3 };
/* stream ids; bit (1 << id) in a stream mask */
enum { SE_STREAM_A = 0, SE_STREAM_B = 1, SE_STREAM_C = 2, SE_STREAM_P = 3 };
enum { SE_LAYOUT_A_LOCAL = 0, SE_LAYOUT_AB_LOCAL = 1 };
enum { SE_EFORMAT = -5,      /* bad magic, version, header or stream table   */
       SE_EINTEGRITY = -6 }; /* a stream's SHA-256 does not match its entry  */

typedef struct {
    uint32_t scheme, flags, levels, width, height, channels;
    uint64_t n_bytes, block_offset;
    uint8_t iv[16];
} se_container_info;

/* Byte lengths of the 4 streams (A, B, C, P) for this geometry (0 where the
 * scheme has none).  SE_EINVAL on bad geometry. */
int se_container_streams(const se_container_info* info, uint64_t lens[4]);

/* Size of a container holding the streams of `stream_mask`. */
int se_container_size(const se_container_info* info, uint32_t stream_mask, uint64_t* out_bytes);

/* Serialise: host stream buffers streams[id] (lengths from the layout; only
 * the ids in stream_mask are read) into out[0 .. cap).  *written = bytes.
 * SE_EINVAL: bad geometry, empty or foreign mask, NULL stream, cap too small. */
int se_container_pack(const se_container_info* info, uint32_t stream_mask, const void* const streams[4],
                      uint8_t* out, uint64_t cap, uint64_t* written);

/* Parse and check a container in buf[0 .. len): magic, version, header and
 * stream table (bounds, alignment, lengths == layout) -> SE_EFORMAT; with
 * verify != 0 every stream's SHA-256 -> SE_EINTEGRITY, *bad_mask = the
 * failing ids.  On success (or SE_EINTEGRITY) fills *info, *stream_mask and
 * streams[id] = pointers INTO buf (NULL for absent ids). */
int se_container_open(const uint8_t* buf, uint64_t len, int verify, se_container_info* info,
                      uint32_t* stream_mask, const uint8_t* streams[4], uint32_t* bad_mask);

/* Placement of a scheme's streams for a layout: local (trusted) mask and up to
 * two remote (public) masks, one container each. */
int se_disperse_plan(uint32_t layout, uint32_t scheme, uint32_t* local_mask, uint32_t remote_masks[2]);

/* Storage accounting of a layout for this geometry, headers included:
 * local bytes / n_bytes and all containers' bytes / n_bytes. */
int se_storage_footprint(const se_container_info* info, uint32_t layout, double* local_frac, double* total_frac);

/* SHA-256 (FIPS 180-4) of a host buffer: the content digest of the table. */
void se_sha256(const void* data, uint64_t len, uint8_t out[32]);

#ifdef __cplusplus
}
#endif
#endif
