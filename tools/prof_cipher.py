#!/usr/bin/env python3
"""Run cipher_encrypt (full-file AES-128-CTR, the paper's comparator) on the
C2 input a few times — a short command for ncu captures of k_cipher_ctr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

x = torch.from_numpy(synth.config_input(2)).cuda()
y = torch.empty_like(x)
for _ in range(5):
    se.cipher_encrypt(synth.KEY, synth.iv_for(2), x, out=y)
torch.cuda.synchronize()
print("ok", x.numel())
