"""Host-side partitioning for multi-GPU runs (SURVEY.md §8.6, row e).

The path has no data-path exchange: every 8x8 block is independent
and its records land at stream offsets that are pure functions of its block
index.  So work is split, never communicated:

* one large file -> contiguous stripes of whole block-rows, one per rank.  A
  stripe is processed as its own input with `block_offset` = global index of
  its first block (hash nonce, C16; CTR start, C13).  Stripe boundaries are
  chosen so every stream slice starts on a byte boundary and the CTR counter
  of the stripe is integral; then the ranks' streams, concatenated in rank
  order, are byte-identical to the single-GPU streams.
* many files -> longest-processing-time-first assignment by size.

Pure Python on plain integers (no torch, no kernels): the CPU multi-process
tests (gloo) drive exactly this code.
"""
from __future__ import annotations

import heapq
import math

BITS = {1: (160, 0, 480), 2: (40, 124, 480), 3: (10, 155, 480)}   # BLOCK8 a/b/c bits per block
FULL_BITS = {1: (160, 0, 480), 2: (40, 132, 480), 3: (10, 165, 480)}   # FULL mode (C23)


def block_align(levels: int, full: bool = False) -> int:
    """Smallest block count g such that a stripe starting at a multiple of g
    has an integral AES-CTR start (block_offset*a_bits % 128 == 0) and byte-
    aligned B and C slices."""
    a, b, c = (FULL_BITS if full else BITS)[levels]
    g = 128 // math.gcd(128, a)
    for bits in (b, c):
        if bits:
            g = math.lcm(g, 8 // math.gcd(8, bits))
    return g


def plan_stripes(n_bytes: int, width: int, levels: int, world: int):
    """Split one file into `world` row stripes.  Returns a list of dicts with
    byte_begin/byte_end (input slice), block_offset, n_blocks and the slices
    of the three global streams each stripe produces."""
    if width <= 0 or width % 8:
        raise ValueError("width must be a positive multiple of 8")
    a_bits, b_bits, c_bits = BITS[levels]
    rows = -(-n_bytes // width)
    rows = -(-rows // 8) * 8
    block_rows = rows // 8
    bpr = width // 8
    g = block_align(levels)
    unit = g // math.gcd(g, bpr)               # block-rows per alignment unit
    n_units = -(-block_rows // unit)
    out = []
    for r in range(world):
        u0 = n_units * r // world
        u1 = n_units * (r + 1) // world
        br0, br1 = min(block_rows, u0 * unit), min(block_rows, u1 * unit)
        b0, b1 = br0 * bpr, br1 * bpr
        byte0 = min(n_bytes, br0 * 8 * width)
        byte1 = min(n_bytes, br1 * 8 * width)
        last = br1 == block_rows

        def sl(bits):
            lo = b0 * bits // 8
            hi = -(-b1 * bits // 8) if last else b1 * bits // 8
            return (lo, hi)
        out.append({"rank": r, "byte_begin": byte0, "byte_end": byte1, "block_offset": b0,
                    "n_blocks": b1 - b0, "a": sl(a_bits), "b": sl(b_bits), "c": sl(c_bits)})
    return out


def plan_files(sizes, world: int):
    """LPT: assign files (by size, largest first) to the least-loaded rank.
    Returns per-rank lists of file indices (each list in ascending order)."""
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    out = [[] for _ in range(world)]
    for i in sorted(range(len(sizes)), key=lambda k: -int(sizes[k])):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return [sorted(x) for x in out]


def plan_full_stripes(n_bytes: int, width: int, levels: int, world: int):
    """FULL mode (whole-matrix DWT, row a11) split into `world` stripes of
    block rows with halos (2(2^L - 1) input rows per side).
    Per stripe: rows [row_begin, row_end); the protect input window
    src = [row_begin - halo, row_end + halo) clipped to the matrix; the recover
    fragment window of whole halo block rows, widened to aligned block rows;
    and the byte slices of the whole-file streams each window produces or
    needs (se.h fragment_protect_stripe / fragment_recover_stripe)."""
    if width <= 0 or width % 8:
        raise ValueError("width must be a positive multiple of 8")
    bits = FULL_BITS[levels]
    rows = -(-n_bytes // width)
    rows = -(-rows // 8) * 8
    block_rows, bpr = rows // 8, width // 8
    g = block_align(levels, full=True)
    unit = g // math.gcd(g, bpr)               # block rows per alignment unit
    halo = 2 * ((1 << levels) - 1)
    hb = -(-halo // 8)                          # halo block rows for recovery
    n_units = -(-block_rows // unit)

    def slices(br0, br1):
        last = br1 == block_rows
        out = {}
        for name, b in zip("abc", bits):
            lo = br0 * bpr * b // 8
            hi = -(-br1 * bpr * b // 8) if last else br1 * bpr * b // 8
            out[name] = (lo, hi)
        return out

    plan = []
    for r in range(world):
        br0 = min(block_rows, n_units * r // world * unit)
        br1 = min(block_rows, n_units * (r + 1) // world * unit)
        if br0 == br1:
            plan.append(None)
            continue
        e0 = max(0, br0 - hb) // unit * unit                       # aligned down
        e1 = min(block_rows, -(-(br1 + hb) // unit) * unit)        # aligned up (or the end)
        row0, row1 = 8 * br0, 8 * br1
        src0, src1 = max(0, row0 - halo), min(rows, row1 + halo)
        plan.append({"rank": r, "row_begin": row0, "row_end": row1, "block_offset": br0 * bpr,
                     "n_blocks": (br1 - br0) * bpr,
                     "src_row0": src0, "src_rows": src1 - src0,
                     "byte_begin": min(n_bytes, row0 * width), "byte_end": min(n_bytes, row1 * width),
                     "src_byte_begin": min(n_bytes, src0 * width), "src_byte_end": min(n_bytes, src1 * width),
                     "out": slices(br0, br1),
                     "rec_row0": 8 * e0, "rec_rows": 8 * (e1 - e0), "rec_in": slices(e0, e1)})
    return plan
