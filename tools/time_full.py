#!/usr/bin/env python3
"""Time the FULL-mode transform kernels alone (dwt_fwd / dwt_inv, MODE_FULL)
and FULL protect / recover on 64 MiB (W = 8192) and the C4 1 GiB file
(W = 32768), L = 2; L2 flushed before each timed call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 2):
        flush.fill_(1)
        flush.amax()                                  # write-back outside the timed region
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


for n, W in ((1 << 26, 8192), (1 << 30, 32768)):
    x = torch.from_numpy(synth.random_bytes(n, 4)).cuda()
    L = 2
    coef = se.dwt_fwd(x, W, L, mode=se.MODE_FULL)
    y = se.dwt_inv(coef, n, W, L, mode=se.MODE_FULL)
    assert torch.equal(x, y)
    tf = timed(lambda: se.dwt_fwd(x, W, L, mode=se.MODE_FULL, out=coef))
    ti = timed(lambda: se.dwt_inv(coef, n, W, L, mode=se.MODE_FULL, out=y))
    iv = synth.iv_for(4)
    a, b, c = se.fragment_protect(x, W, L, synth.KEY, iv, mode=se.MODE_FULL)
    tp = timed(lambda: se.fragment_protect(x, W, L, synth.KEY, iv, mode=se.MODE_FULL, out=(a, b, c)))
    tr = timed(lambda: se.fragment_recover(a, b, c, n, W, L, synth.KEY, iv, mode=se.MODE_FULL, out=y))
    print(f"n={n >> 20} MiB W={W}: dwt_fwd {tf:.1f} us ({3 * n / tf / 1e3:.0f} GB/s of 3n traffic), "
          f"dwt_inv {ti:.1f} us ({3 * n / ti / 1e3:.0f} GB/s); protect {tp:.1f} us ({n / tp / 1e3:.1f} GB/s), "
          f"recover {tr:.1f} us ({n / tr / 1e3:.1f} GB/s)")
    del x, coef, y, a, b, c
    torch.cuda.empty_cache()
