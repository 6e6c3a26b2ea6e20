#!/usr/bin/env python3
"""Two protect / recover / cipher calls (NVTX range check: under
`ncu --nvtx --nvtx-include "<call>/"` only that call's kernels are profiled)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

x = torch.from_numpy(synth.random_bytes(1 << 22, 1)).cuda()
for _ in range(2):
    a, b, c = se.fragment_protect(x, 1024, 2, synth.KEY, synth.iv_for(1))
    y, r = se.fragment_recover(a, b, c, x.numel(), 1024, 2, synth.KEY, synth.iv_for(1))
    e = se.cipher_encrypt(synth.KEY, synth.iv_for(1), x)
torch.cuda.synchronize()
assert torch.equal(x, y)
print("probe ok")
