"""The README usage example, run as is (doc check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1803_04880_b200 as se
x = torch.randint(0, 256, (1 << 24,), dtype=torch.uint8, device="cuda")
key, iv = bytes(range(16)), bytes(16)
a, b, c = se.fragment_protect(x, 1024, 2, key, iv)          # private, public, public
y, report = se.fragment_recover(a, b, c, x.numel(), 1024, 2, key, iv)
assert torch.equal(x, y) and report.tolist() == [-1, 0]

img = torch.randint(0, 256, (4800 * 4800,), dtype=torch.uint8, device="cuda")
f1, f2 = se.dct_protect(img, 4800, 4800, 1, 2, key, iv)      # Chapter 4, level 2
back = se.dct_recover(f1, f2, 4800, 4800, 1, 2, key, iv)     # lossy by design (~60 dB)
print("readme example ok")
