/*
 * se.h — C ABI of libse.so: B200-native (sm_100a) agnostic selective
 * encryption, the Chapter 5 hot path of arxiv/paper_1803_04880.
 *
 * The operation (PAPER.md "Design of DWT based SE"): any byte
 * stream is read as a 2-D matrix of 8-bit "pixels", tiled into 8x8
 * blocks; each block is transformed by a lossless integer Le Gall 5/3 lifting
 * DWT (Eq. 5.1-5.2), two levels; the coefficients are
 * split into three fragments per block (D_iA, D_iB, D_iC):
 *   A  private fragment  = 2nd-level LL, 4 x 10 bits = 40 bits
 *   B  1st public frag.  = 2nd-level HL/LH/HH, 124 bits
 *   C  2nd public frag.  = 1st-level HL/LH/HH, 480 bits
 * A is encrypted with AES-128; B is XORed with SHA-256 of (key, A)
 * (P:2130); C is XORed with SHA-512 of (B', key).  Recovery is the
 * exact inverse.  Where the paper is silent the readings are
 * those of DESIGN.md §3; the byte-exact definition is the
 * oracle in oracle/ (which this library does not use).
 *
 * Conventions shared by every call:
 *   Geometry   n_bytes bytes form a W x R matrix, W = width (a positive
 *              multiple of 8), R = ceil(n_bytes / W) rounded up to a multiple
 *              of 8; bytes past n_bytes read as 0 (C18).  Blocks are numbered
 *              row-major: b = br * (W/8) + bc (C11).
 *   Levels     1, 2 (the paper) or 3 (C21).  L = 1: A = LL1 (160 b), B empty;
 *              L = 3: A = LL3 (10 b), B = level-3 + level-2 details (155 b).
 *   Streams    A', B', C' are dense bit streams, records in block order,
 *              MSB-first, fields offset-binary (C9-C11), the final byte zero-
 *              padded; sizes from fragment_layout().
 *   Key, IV    16-byte HOST buffers, read during the call only.  The IV is
 *              the initial AES-CTR counter block (C13) and enters the hash
 *              framing (C15): M_B = K||IV||be64(b)||A_b, M_C = K||IV||be64(b)||B'_b.
 *   Device ptrs  caller-owned device memory (e.g. torch tensors), 16-byte
 *              aligned (else SE_EALIGN), valid until the stream reaches the
 *              work.  No device-resident call allocates device memory or
 *              synchronises; FULL mode takes a caller workspace (below).
 *   stream     a cudaStream_t passed as void* (NULL = legacy default stream).
 *              Calls are asynchronous on it; all run on the current device.
 *   Errors     return se_status; nothing is printed.  Launch failures are
 *              SE_ECUDA (cudaGetLastError).  Data-dependent corruption (wrong
 *              key, damaged fragments) is NOT an error: recover reports it in
 *              a device-resident se_report.
 *   Threading  stateless and reentrant; concurrent calls on different streams
 *              or devices are safe.
 */
#ifndef SE_H
#define SE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SE_OK = 0,
    SE_EINVAL = -1,   /* null pointer, bad width/levels/mode, bad offsets    */
    SE_EALIGN = -2,   /* device pointer not 16-byte aligned                  */
    SE_ECUDA = -3,    /* CUDA launch / runtime failure                       */
    SE_ENOTSUP = -4   /* combination not implemented                         */
} se_status;

enum { SE_MODE_BLOCK8 = 0,   /* per-8x8-block DWT: the paper   */
       SE_MODE_FULL = 1 };   /* whole-matrix Mallat DWT: extension row a11       */

enum { SE_FLAG_PUBLIC_PLAIN = 1u << 0,   /* skip the SHA masks on B and C:
                                             measurement mode (C26) */
       SE_FLAG_HOST_MAPPED = 1u << 1 };  /* *_host calls only (BLOCK8): the
                                             host buffers are page-locked and the
                                             kernels read / write them directly
                                             over PCIe (zero-copy), no staging */

/* block_offset: global index of this input's first 8x8 block inside the
 * logical file (0 for a whole file).  It is the hash nonce base (C16) and
 * sets the CTR start counter IV + block_offset*a_bits/128, so it must make
 * block_offset*a_bits a multiple of 128 (any multiple of 128 blocks does). */
typedef struct {
    uint64_t n_bytes;
    uint32_t width, levels, mode, flags;
    uint64_t block_offset;
} se_geom;

typedef struct {
    uint64_t rows, n_blocks, a_bytes, b_bytes, c_bytes;
    uint32_t a_bits, b_bits, c_bits;   /* bits per block record            */
    uint32_t halo_rows;                /* input rows a stripe needs beyond
                                          its own (0 in BLOCK8; FULL: 2(2^L-1)) */
} se_layout;

/* Device-resident corruption report written by fragment_recover.
 * first_bad_block = -1 when clean, else the smallest local block index
 * with a reconstructed sample outside [0, 255]; bad_blocks = their count. */
typedef struct {
    int64_t first_bad_block;
    uint64_t bad_blocks;
} se_report;

/* ---- layout (host, pure) ------------------------------------------------
 * Sizes of the matrix and of the three fragment streams (P:2243, P:2285,
 * 40/124/480 bits per block = 7.8/24.2/93.8 % at L = 2). */
int fragment_layout(const se_geom* g, se_layout* out);

/* ---- protect: rows a1-a9 in one kernel -----------------------------------
 * d_in: n_bytes input bytes (device).  d_a, d_b, d_c: device buffers of
 * a_bytes, b_bytes, c_bytes (d_b may be NULL when b_bytes == 0).  Writes the
 * protected streams A', B', C'.  n_bytes == 0 is a no-op.  One kernel launch
 * (BLOCK8); AES-128-CTR of A runs inside it (no scratch).  At most 2^32
 * 8x8 blocks (256 GiB) per call, else SE_EINVAL.  FULL mode needs a
 * workspace: use fragment_protect_ws (fragment_protect returns SE_EINVAL). */
int fragment_protect(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                     const void* d_in, void* d_a, void* d_b, void* d_c, void* stream);

/* ---- recover: row a10 -----------------------------------------------------
 * Inverse of fragment_protect; writes exactly n_bytes bytes to d_out.
 * d_report (nullable, device) receives the corruption report (set to
 * {-1, 0} by the call, then updated by the kernel).  FULL mode: use
 * fragment_recover_ws. */
int fragment_recover(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                     const void* d_a, const void* d_b, const void* d_c, void* d_out,
                     se_report* d_report, void* stream);

/* ---- caller-owned workspace (FULL mode, row a11) ---------------------------
 * No call allocates device memory.  FULL mode keeps the R x W int16 Mallat
 * coefficients of the matrix (stripe calls: of the stripe's row window)
 * between its transform and footprint kernels in a workspace the caller
 * provides: fragment_workspace_size returns its size in *bytes (0 in BLOCK8
 * mode; st = NULL for the whole-file calls, else the stripe the
 * fragment_*_stripe call will get).  The _ws calls are fragment_protect /
 * fragment_recover plus that workspace (16-byte aligned device memory, at
 * least the queried size, else SE_EINVAL / SE_EALIGN; it may be reused as
 * soon as the stream has passed the call). */
typedef struct {
    uint64_t row_begin, row_end, src_row0, src_rows;
} se_stripe;
int fragment_workspace_size(const se_geom* g, const se_stripe* st, uint64_t* bytes);
int fragment_protect_ws(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                        const void* d_in, void* d_a, void* d_b, void* d_c,
                        void* d_ws, uint64_t ws_bytes, void* stream);
int fragment_recover_ws(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                        const void* d_a, const void* d_b, const void* d_c, void* d_out,
                        se_report* d_report, void* d_ws, uint64_t ws_bytes, void* stream);

/* ---- batched protect / recover (many independent files, one launch) -----
 * "batch of 10,000 mixed-size files ... sharded by file" (BASELINE.json C5;
 * the paper's chunks D_i are independent).  The caller fills one
 * se_job per file in HOST memory (pointers are device pointers; IV per file),
 * calls fragment_batch_plan (host, pure: validates every job, assigns each its
 * first CTA and derives the per-file counter base, SHA midstates and SHA-512
 * schedule constants over K || IV into `derived`), copies the array (16-byte
 * aligned) to device memory, then launches.  All jobs of a batch share the
 * key, levels and flags.  Mode is BLOCK8. */
typedef struct {
    const uint8_t* in;        /* protect: input bytes (device)                */
    uint8_t* out;             /* recover: output bytes (device)               */
    uint8_t *a, *b, *c;       /* fragment streams (device), sized per layout  */
    uint64_t n_bytes;
    uint64_t block_offset;    /* as se_geom.block_offset                      */
    uint32_t width;           /* matrix width W of this file                  */
    uint32_t reserved0;
    uint8_t iv[16];
    uint64_t cta_begin;       /* set by fragment_batch_plan                   */
    uint32_t derived[132];    /* set by fragment_batch_plan (library-private) */
} se_job;

/* Returns the total number of CTAs of the launch (>= 0), or a negative
 * se_status (SE_EINVAL: bad geometry / alignment / pointers in a job). */
int64_t fragment_batch_plan(se_job* h_jobs, uint32_t n_jobs, uint32_t levels, const uint8_t key[16]);
int fragment_protect_batch(uint32_t n_jobs, const se_job* d_jobs, uint64_t total_ctas,
                           uint32_t levels, uint32_t flags, const uint8_t key[16],
                           void* stream);
/* d_reports: nullable device array of n_jobs reports (one per file). */
int fragment_recover_batch(uint32_t n_jobs, const se_job* d_jobs, uint64_t total_ctas,
                           uint32_t levels, uint32_t flags, const uint8_t key[16],
                           se_report* d_reports, void* stream);

/* ---- host-resident streaming protect / recover (NEXT row f1) -------------
 * h_* are HOST buffers (pinned or pageable).  The library stages chunks of
 * whole 8-row block-rows through its own pinned + device buffers on
 * n_streams CUDA streams, overlapping H2D copy, kernel and D2H copy
 * (the paper's transfer/compute overlap).  Blocking: returns
 * after the last D2H completes.  chunk_bytes = input bytes per chunk
 * (rounded to whole 128-block groups; 0 = n/4 within [4 MiB, 16 MiB]). */
int fragment_protect_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                          const void* h_in, void* h_a, void* h_b, void* h_c,
                          uint64_t chunk_bytes, uint32_t n_streams);
int fragment_recover_host(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                          const void* h_a, const void* h_b, const void* h_c, void* h_out,
                          se_report* h_report, uint64_t chunk_bytes, uint32_t n_streams);

/* Asynchronous forms: the same work enqueued on the library's per-device
 * streams; the call returns once everything is enqueued and hands back a
 * ticket.  A recover may name a protect ticket (`after`) whose fragments it
 * reads: each of its chunks then waits only for the protect chunks it
 * overlaps, so the recover's host-to-device copies run under the protect's
 * device-to-host traffic (one pipeline fill and drain for the round trip,
 * P:2682-2695).  se_host_wait blocks until a ticket's work is done, fills
 * *h_report (nullable; recover tickets), frees the ticket and returns the
 * call's status.  Host buffers must stay valid until then.  One ticket per
 * direction and device is in flight at a time: a new call of the same
 * direction first waits for the previous one's work (its report is kept). */
typedef struct se_host_ticket se_host_ticket;
int fragment_protect_host_async(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                                const void* h_in, void* h_a, void* h_b, void* h_c,
                                uint64_t chunk_bytes, uint32_t n_streams, se_host_ticket** ticket);
int fragment_recover_host_async(const se_geom* g, const uint8_t key[16], const uint8_t iv[16],
                                const void* h_a, const void* h_b, const void* h_c, void* h_out,
                                uint64_t chunk_bytes, uint32_t n_streams, const se_host_ticket* after,
                                se_host_ticket** ticket);
int se_host_wait(se_host_ticket* ticket, se_report* h_report);

/* ---- FULL-mode row stripes with halo rows (row e for a11) ---------------
 * A FULL-mode file (whole-matrix DWT) split into stripes of block rows for
 * several GPUs.  Lifting reaches 2(2^L - 1) input rows beyond a stripe
 * (layout.halo_rows: 6 at L = 2), so each stripe is protected from its rows
 * plus that many halo rows per side, and recovered from the fragments of its
 * block rows plus ceil(halo_rows / 8) halo block rows per side.  Concatenated
 * in row order, the stripes' streams and bytes equal the whole-file ones.
 *   g          the WHOLE file (mode SE_MODE_FULL; block_offset of its block 0)
 *   row_begin, row_end   the stripe's rows, multiples of 8 (row_end may be R);
 *              row_begin * W/8 * bits must be a multiple of 8 for every
 *              stream and of 128 for A (any multiple of 128 blocks is)
 *   src_row0, src_rows   the rows present at the source pointer:
 *              protect: input bytes of rows [src_row0, src_row0 + src_rows),
 *              covering [row_begin - halo, row_end + halo] clipped to [0, R);
 *              recover: fragments of block rows [src_row0/8, (src_row0 +
 *              src_rows)/8) (multiples of 8, src_row0 aligned like row_begin),
 *              covering the halo block rows.
 * Outputs: protect writes the stripe's blocks' records (stream slices at
 * byte offset first_block * bits / 8 of the whole-file streams); recover
 * writes the stripe's bytes (row_begin * W onwards, clipped at n_bytes) and
 * reports bad blocks with stripe-local indices.  SE_EINVAL on a bad window.
 * d_ws / ws_bytes: the workspace of fragment_workspace_size(g, s, ...). */
int fragment_protect_stripe(const se_geom* g, const se_stripe* s, const uint8_t key[16], const uint8_t iv[16],
                            const void* d_in, void* d_a, void* d_b, void* d_c, void* d_ws, uint64_t ws_bytes,
                            void* stream);
int fragment_recover_stripe(const se_geom* g, const se_stripe* s, const uint8_t key[16], const uint8_t iv[16],
                            const void* d_a, const void* d_b, const void* d_c, void* d_out,
                            se_report* d_report, void* d_ws, uint64_t ws_bytes, void* stream);

/* ---- transform only: rows a1-a4 / a11 ------------------------------------
 * d_coef: R x W int16 (R = layout.rows).  BLOCK8: block (br, bc) coefficient
 * (i, j) at [(8br+i)*W + 8bc+j], dyadic quadrants inside each block (LL top-
 * left, HL top-right, LH bottom-left, HH bottom-right; C7).  FULL: Mallat
 * layout over the whole matrix.  dwt_inv writes n_bytes bytes; samples
 * outside [0,255] are stored modulo 256. */
int dwt_fwd(const se_geom* g, const void* d_in, int16_t* d_coef, void* stream);
int dwt_inv(const se_geom* g, const int16_t* d_coef, void* d_out, void* stream);

/* ---- cipher only: AES-128-CTR (row a6; the paper's full-AES comparator,
 * P:219) ----------------------------------------------------
 * out[i] = in[i] ^ KS[i], KS block j = AES_K(IV + ctr_block_offset + j),
 * 128-bit big-endian counter (SP 800-38A).  In place allowed (d_in == d_out).
 * cipher_decrypt is the same operation (CTR). */
int cipher_encrypt(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block_offset,
                   const void* d_in, void* d_out, uint64_t n, void* stream);
int cipher_decrypt(const uint8_t key[16], const uint8_t iv[16], uint64_t ctr_block_offset,
                   const void* d_in, void* d_out, uint64_t n, void* stream);

/* ---- security battery (NEXT row f2) --------------------------------------
 * The paper validates the public fragments statistically (PAPER.md "Security
 * analysis"): PDF / uniformity, entropy Eq. 5.6
 * (P:2454-2463), correlation r_xy Eq. 5.8 between original and fragment
 * and between adjacent elements h / v / d, bit
 * difference Dif, NMI, key sensitivity KS = bit difference
 * of the fragments under two keys one bit apart.
 * se_stats_accumulate makes ONE pass over two equal-length byte sequences
 * x and y (y also read as a W-wide matrix for the adjacency sums) and ADDS
 * exact integer sums into a caller-zeroed, device-resident se_stats (and,
 * if d_joint != NULL, into a 65536-bin joint histogram indexed x*256 + y,
 * for NMI).  The metrics are plain arithmetic on these sums (binding:
 * paper_1803_04880_b200.stats_metrics).  d_x may be NULL (y-only sums). */
typedef struct {
    uint64_t n;                      /* byte pairs accumulated                 */
    uint64_t hist_x[256], hist_y[256];
    uint64_t sx, sy, sxx, syy, sxy;  /* moments of x, y over the n pairs       */
    uint64_t diff_bits;              /* popcount(x ^ y)                        */
    uint64_t adj[3][6];              /* y pairs (a, b) horizontal, vertical,
                                        diagonal: count, sa, sb, saa, sbb, sab */
} se_stats;

int se_stats_accumulate(const void* d_x, const void* d_y, uint64_t n, uint32_t width, se_stats* d_stats,
                        uint32_t* d_joint, void* stream);

/* ---- misc ----------------------------------------------------------------- */
const char* se_strerror(int status);
/* Number of kernel launches issued by this thread since the last reset
 * (bench/test evidence of native launches). */
uint64_t se_launch_count(int reset);
/* Which kernels serve single-file BLOCK8 calls on device buffers: 0 = auto
 * (persistent tile kernels from 8 tiles per SM up, else the per-CTA kernels),
 * 1 = tile, 2 = per-CTA; -1 only queries.  Returns the previous choice.
 * Process-wide; a test / measurement knob (env SE_KERNEL=tile|cta). */
int se_kernel_choice(int choice);
/* Rows per segment of the streaming FULL-mode transform: 32, 64, 128, 256, or
 * 0 = chosen by matrix size (default).  Returns the previous value (SE_EINVAL
 * for another value).  Process-wide test knob: each length runs different
 * halo / window code, so the tests compare every length with the oracle. */
int se_full_segment_rows(int rows);

#ifdef __cplusplus
}
#endif
#endif
