#!/usr/bin/env python3
"""Run dct_protect + dct_recover (row f3) on the 4800x4800 grey image a few
times — a short command for ncu captures of k_dct_protect / k_dct_recover.
Usage: prof_dct.py LEVEL [KEYED]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 1
flags = se.DCT_KEYED if len(sys.argv) > 2 and sys.argv[2] == "keyed" else 0
W = H = 4800
x = torch.from_numpy(synth.bitmap(H, W, 1, W + H).reshape(-1)).cuda()
for _ in range(4):
    a, p = se.dct_protect(x, W, H, 1, level, synth.KEY, synth.iv_for(6), flags=flags)
    y = se.dct_recover(a, p, W, H, 1, level, synth.KEY, synth.iv_for(6), flags=flags)
torch.cuda.synchronize()
print("ok", int((y.to(torch.int16) - x.to(torch.int16)).abs().max()))
