#!/usr/bin/env python3
"""Small invocations of every libse entry point, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck, one tool per call):
ragged sizes, several CTAs, every level, both modes, batch, host streaming."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

key, iv = synth.KEY, synth.iv_for(9)
dev = torch.device("cuda:0")
ok = True
for (n, W) in [(1, 8), (1000, 24), (128 * 64 * 2 + 77, 1024), (256 * 136, 256)]:
    x = torch.from_numpy(synth.random_bytes(n, n)).to(dev)
    for L in (1, 2, 3):
        for mode in (se.MODE_BLOCK8, se.MODE_FULL):
            a, b, c = se.fragment_protect(x, W, L, key, iv, mode=mode)
            y, rep = se.fragment_recover(a, b, c, n, W, L, key, iv, mode=mode)
            coef = se.dwt_fwd(x, W, L, mode=mode)
            z = se.dwt_inv(coef, n, W, L, mode=mode)
            torch.cuda.synchronize()
            ok &= bool(torch.equal(x, y)) and bool(torch.equal(x, z)) and rep.cpu().tolist() == [-1, 0]
    e = se.cipher_encrypt(key, iv, x, ctr_block_offset=5)
    ok &= bool(torch.equal(se.cipher_decrypt(key, iv, e, ctr_block_offset=5), x))
files = [torch.from_numpy(synth.random_bytes(s, s)).to(dev) for s in (1, 5000, 70000)]
batch = se.Batch(files, [synth.width_rule(f.numel()) for f in files], [synth.iv_for(5, i) for i in range(3)], 2, key)
batch.protect()
outs, reps = batch.recover()
torch.cuda.synchronize()
ok &= all(torch.equal(o, f) for o, f in zip(outs, files))
hx = torch.from_numpy(synth.random_bytes(300000, 3)).pin_memory()
a, b, c = se.fragment_protect_host(hx, 512, 2, key, iv, chunk_bytes=64 * 1024)
back, rep = se.fragment_recover_host(a, b, c, hx.numel(), 512, 2, key, iv, chunk_bytes=64 * 1024)
ok &= bool(torch.equal(back, hx)) and rep == (-1, 0)
print("sanitize cases:", "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
