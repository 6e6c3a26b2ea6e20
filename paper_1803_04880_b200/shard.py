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


def block_align(levels: int) -> int:
    """Smallest block count g such that a stripe starting at a multiple of g
    has an integral AES-CTR start (block_offset*a_bits % 128 == 0) and byte-
    aligned B and C slices."""
    a, b, c = BITS[levels]
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
