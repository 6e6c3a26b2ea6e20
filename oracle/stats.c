/*
 * stats.c — oracle: the sums behind the paper's security battery (NEXT row
 * f2, PAPER.md "Security analysis" P:2296-2651), TEST INFRASTRUCTURE.
 *
 * Straight loops over the definitions: byte histograms (PDF, P:2392;
 * entropy Eq. 5.6), the moments of Eq. 5.8, the
 * bit difference (Dif P:2555, KS P:2578-2592), adjacent-element pairs of y
 * read as a W-wide matrix, horizontal / vertical / diagonal (all
 * pairs rather than 4096 random ones — reading in DESIGN.md §3), and the
 * joint histogram for NMI.  out[] layout (uint64): n, hist_x[256],
 * hist_y[256], sx, sy, sxx, syy, sxy, diff_bits, adj[3][6] (count, sa, sb,
 * saa, sbb, sab).  x may be NULL.
 */
#include "oracle.h"
#include <string.h>

static int popcount8(unsigned v) {
    int c = 0;
    for (int b = 0; b < 8; ++b) c += (v >> b) & 1u;
    return c;
}

void oracle_stats(const uint8_t* x, const uint8_t* y, uint64_t n, uint32_t width, uint64_t* out,
                  uint64_t* joint) {
    memset(out, 0, sizeof(uint64_t) * ORACLE_STATS_WORDS);
    if (joint) memset(joint, 0, sizeof(uint64_t) * 65536);
    uint64_t* hist_x = out + 1;
    uint64_t* hist_y = out + 1 + 256;
    uint64_t* mom = out + 513;
    uint64_t* adj = out + 519;
    out[0] = n;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t yv = y[i];
        hist_y[yv]++;
        mom[1] += yv;
        mom[3] += yv * yv;
        if (x) {
            const uint64_t xv = x[i];
            hist_x[xv]++;
            mom[0] += xv;
            mom[2] += xv * xv;
            mom[4] += xv * yv;
            mom[5] += (uint64_t)popcount8((unsigned)(xv ^ yv));
            if (joint) joint[xv * 256 + yv]++;
        }
        const uint64_t col = i % width;
        /* neighbours: right (i+1), down (i+W), down-right (i+W+1) */
        const int has[3] = {col + 1 < width && i + 1 < n, i + width < n, col + 1 < width && i + width + 1 < n};
        const uint64_t nb[3] = {i + 1, i + width, i + width + 1};
        for (int d = 0; d < 3; ++d) {
            if (!has[d]) continue;
            const uint64_t bv = y[nb[d]];
            adj[6 * d + 0] += 1;
            adj[6 * d + 1] += yv;
            adj[6 * d + 2] += bv;
            adj[6 * d + 3] += yv * yv;
            adj[6 * d + 4] += bv * bv;
            adj[6 * d + 5] += yv * bv;
        }
    }
}
