/*
 * dwt53.c — oracle: integer Le Gall 5/3 lifting DWT (TEST INFRASTRUCTURE).
 *
 * PAPER.md "DWT" subsection, Eq. (5.1)-(5.2):
 *   y(2n+1) = x_ext(2n+1) - floor((x_ext(2n) + x_ext(2n+2)) / 2)
 *   y(2n)   = x_ext(2n)   + floor((y(2n-1) + y(2n+1) + 2) / 4)
 * Readings (SURVEY C2–C8):
 *   C3  the update term is ADDED: the paper's matrix A and the
 *       "1.5 times" low-band range fix the sign; the "-" printed in
 *       Eq. 5.2 contradicts both.
 *   C2  x_ext is whole-sample symmetric extension: x_ext(-i) = x(i),
 *       x_ext(N-1+i) = x(N-1-i)  (matrix A columns 3 and 7).
 *   C4  floor is the mathematical floor ("largest integer not exceeding a").
 *   C6  one 1-D pass stores [y(0), y(2), ... | y(1), y(3), ...]: "the first 4
 *       are low frequency and last 4 are high frequency".
 *   C5  2-D: rows ("horizontal direction") first, then columns.
 *   A6  multi-level: level l+1 transforms only the LL quadrant of level l
 *       (dyadic decomposition).
 *   C8  bytes are centered to [-128, 127] before level 1.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

/* floor(a / b) for b > 0, written out (no shifts) — C4. */
static int32_t floor_div(int32_t a, int32_t b) {
    int32_t q = a / b;
    if ((a % b) != 0 && a < 0) q -= 1;
    return q;
}

/* whole-sample symmetric extension index (C2) */
static int reflect(int i, int n) {
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}

/* Eq. 5.1 evaluated at odd position 2k+1 (k may be -1: y(-1) is needed by
 * Eq. 5.2 at n = 0 and is computed from x_ext, not assumed). */
static int32_t predict_at(const int32_t* x, int n, int k) {
    int32_t xo = x[reflect(2 * k + 1, n)];
    int32_t xl = x[reflect(2 * k, n)];
    int32_t xr = x[reflect(2 * k + 2, n)];
    return xo - floor_div(xl + xr, 2);
}

void oracle_lift_fwd_1d(const int32_t* x, int32_t* y, int n) {
    int h = n / 2;
    int32_t* s = (int32_t*)malloc(sizeof(int32_t) * (size_t)h);
    int32_t* d = (int32_t*)malloc(sizeof(int32_t) * (size_t)h);
    for (int k = 0; k < h; ++k) d[k] = predict_at(x, n, k);          /* Eq. 5.1 */
    for (int k = 0; k < h; ++k) {                                      /* Eq. 5.2 */
        int32_t dm1 = (k == 0) ? predict_at(x, n, -1) : d[k - 1];
        s[k] = x[2 * k] + floor_div(dm1 + d[k] + 2, 4);
    }
    for (int k = 0; k < h; ++k) { y[k] = s[k]; y[h + k] = d[k]; }      /* C6 */
    free(s); free(d);
}

/* Exact inverse: undo the update (Eq. 5.2) then undo the predict (Eq. 5.1).
 * d(-1) = d(0) holds for every forward output under symmetric extension
 * (x_ext(-1) = x(1), x_ext(-2) = x(2)), so it is used here. */
void oracle_lift_inv_1d(const int32_t* y, int32_t* x, int n) {
    int h = n / 2;
    const int32_t* s = y;
    const int32_t* d = y + h;
    for (int k = 0; k < h; ++k) {
        int32_t dm1 = (k == 0) ? d[0] : d[k - 1];
        x[2 * k] = s[k] - floor_div(dm1 + d[k] + 2, 4);
    }
    for (int k = 0; k < h; ++k) {
        int32_t xr = (2 * k + 2 < n) ? x[2 * k + 2] : x[reflect(2 * k + 2, n)];
        x[2 * k + 1] = d[k] + floor_div(x[2 * k] + xr, 2);
    }
}

/* One 2-D level on the top-left rows x cols region of a (stride) array:
 * rows first, then columns (C5). */
static void dwt2_level_fwd(int32_t* a, size_t stride, int rows, int cols) {
    int m = rows > cols ? rows : cols;
    int32_t* in = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int32_t* out = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j) in[j] = a[(size_t)i * stride + j];
        oracle_lift_fwd_1d(in, out, cols);
        for (int j = 0; j < cols; ++j) a[(size_t)i * stride + j] = out[j];
    }
    for (int j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) in[i] = a[(size_t)i * stride + j];
        oracle_lift_fwd_1d(in, out, rows);
        for (int i = 0; i < rows; ++i) a[(size_t)i * stride + j] = out[i];
    }
    free(in); free(out);
}

/* Inverse of one 2-D level: columns first, then rows. */
static void dwt2_level_inv(int32_t* a, size_t stride, int rows, int cols) {
    int m = rows > cols ? rows : cols;
    int32_t* in = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int32_t* out = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    for (int j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) in[i] = a[(size_t)i * stride + j];
        oracle_lift_inv_1d(in, out, rows);
        for (int i = 0; i < rows; ++i) a[(size_t)i * stride + j] = out[i];
    }
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j) in[j] = a[(size_t)i * stride + j];
        oracle_lift_inv_1d(in, out, cols);
        for (int j = 0; j < cols; ++j) a[(size_t)i * stride + j] = out[j];
    }
    free(in); free(out);
}

/* Multi-level dyadic transform of a rows x cols region (A6). */
void oracle_dwt2_fwd_region(int32_t* a, size_t stride, int rows, int cols, int levels) {
    for (int l = 0; l < levels; ++l) dwt2_level_fwd(a, stride, rows >> l, cols >> l);
}
void oracle_dwt2_inv_region(int32_t* a, size_t stride, int rows, int cols, int levels) {
    for (int l = levels - 1; l >= 0; --l) dwt2_level_inv(a, stride, rows >> l, cols >> l);
}

static uint64_t rows_of(uint64_t n, uint32_t w) {
    uint64_t r = (n + w - 1) / w;
    return (r + 7) / 8 * 8;
}

/* Centered sample of the zero-filled W x R matrix (C8, C18). */
static int32_t sample(const uint8_t* in, uint64_t n, uint32_t w, uint64_t r, uint64_t c) {
    uint64_t idx = r * w + c;
    int32_t byte = (idx < n) ? (int32_t)in[idx] : 0;
    return byte - 128;
}

int oracle_dwt_fwd(const uint8_t* in, uint64_t n, uint32_t w, uint32_t levels,
                   uint32_t mode, int32_t* coef) {
    if (w == 0 || w % 8 || levels < 1 || levels > 3 || mode > 1) return -1;
    uint64_t R = rows_of(n, w);
    if (mode == 0) {
        int32_t blk[64];
        for (uint64_t br = 0; br < R / 8; ++br)
            for (uint64_t bc = 0; bc < w / 8; ++bc) {
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        blk[i * 8 + j] = sample(in, n, w, 8 * br + i, 8 * bc + j);
                oracle_dwt2_fwd_region(blk, 8, 8, 8, (int)levels);
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        coef[(8 * br + i) * w + 8 * bc + j] = blk[i * 8 + j];
            }
    } else {
        for (uint64_t r = 0; r < R; ++r)
            for (uint64_t c = 0; c < w; ++c) coef[r * w + c] = sample(in, n, w, r, c);
        oracle_dwt2_fwd_region(coef, w, (int)R, (int)w, (int)levels);
    }
    return 0;
}

int64_t oracle_dwt_inv(const int32_t* coef, uint64_t n, uint32_t w, uint32_t levels,
                       uint32_t mode, uint8_t* out) {
    if (w == 0 || w % 8 || levels < 1 || levels > 3 || mode > 1) return -1;
    uint64_t R = rows_of(n, w);
    int64_t bad = 0;
    int32_t* x = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R * w + 1));
    memcpy(x, coef, sizeof(int32_t) * (size_t)(R * w));
    if (mode == 0) {
        int32_t blk[64];
        for (uint64_t br = 0; br < R / 8; ++br)
            for (uint64_t bc = 0; bc < w / 8; ++bc) {
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        blk[i * 8 + j] = x[(8 * br + i) * w + 8 * bc + j];
                oracle_dwt2_inv_region(blk, 8, 8, 8, (int)levels);
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        x[(8 * br + i) * w + 8 * bc + j] = blk[i * 8 + j];
            }
    } else {
        oracle_dwt2_inv_region(x, w, (int)R, (int)w, (int)levels);
    }
    for (uint64_t i = 0; i < R * w; ++i) {
        int32_t v = x[i] + 128;
        if (v < 0 || v > 255) bad++;
        if (i < n) out[i] = (uint8_t)(v & 0xFF);
    }
    free(x);
    return bad;
}
