#!/usr/bin/env python3
"""FULL mode (row a11) protect + recover of a 64 MiB random file, W = 8192, L = 2 —
a short command for ncu launch lists / captures of the FULL kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

n, W, L = 1 << 26, 8192, 2
x = torch.from_numpy(synth.random_bytes(n, 4)).cuda()
for _ in range(3):
    a, b, c = se.fragment_protect(x, W, L, synth.KEY, synth.iv_for(4), mode=se.MODE_FULL)
    y, rep = se.fragment_recover(a, b, c, n, W, L, synth.KEY, synth.iv_for(4), mode=se.MODE_FULL)
torch.cuda.synchronize()
print("ok", bool(torch.equal(x, y)), rep.tolist())
