"""Seeded random shapes through every single-file BLOCK8 kernel family: widths
(multiples of 8, with and without 16-byte rows), lengths (ragged tails, one
byte to a few MiB), levels 1-3, masked and PUBLIC_PLAIN, per-CTA and tile
kernels, block offsets (the CTR counter and the hash framing).  Every
fragment byte equals the oracle's and every file round-trips; a corrupted
fragment byte gives the oracle's report."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def cases(k=48, seed=20261019):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        W = 8 * int(rng.integers(1, 769))                     # 8 .. 6144
        rows = int(rng.integers(1, max(2, (3 << 20) // W)))
        n = max(1, rows * W - int(rng.integers(0, W)))
        L = int(rng.integers(1, 4))
        flags = int(rng.integers(0, 2))
        kernel = ("tile", "cta")[int(rng.integers(0, 2))]
        boff = int(rng.integers(0, 1 << 20)) * 128 if rng.random() < 0.3 else 0
        out.append((i, n, W, L, flags, kernel, boff))
    return out


@pytest.mark.parametrize("i,n,W,L,flags,kernel,boff", cases())
def test_fuzz_block8(dev, orc, i, n, W, L, flags, kernel, boff):
    prev = se.kernel_choice(se.KERNEL_TILE if kernel == "tile" else se.KERNEL_CTA)
    try:
        x = synth.random_bytes(n, 9000 + i) if i % 3 else synth.text_like(n, 9000 + i)
        iv = synth.iv_for(7, i)
        xt = torch.from_numpy(x).to(dev)
        a, b, c = se.fragment_protect(xt, W, L, KEY, iv, flags=flags, block_offset=boff)
        oa, ob, oc = orc.protect(x, W, L, KEY, iv, flags=flags, block_offset=boff)
        assert np.array_equal(a.cpu().numpy(), oa)
        assert np.array_equal(b.cpu().numpy(), ob)
        assert np.array_equal(c.cpu().numpy(), oc)
        back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, iv, flags=flags, block_offset=boff)
        assert torch.equal(back, xt) and rep.cpu().tolist() == [-1, 0]
        # one corrupted byte of a fragment: bytes and report equal the oracle's
        rng = np.random.default_rng(i)
        which = int(rng.integers(0, 3)) if ob.size else 2 * int(rng.integers(0, 2))
        frags = [oa.copy(), ob.copy(), oc.copy()]
        pos = int(rng.integers(0, frags[which].size))
        frags[which][pos] ^= 1 << int(rng.integers(0, 8))
        d = [torch.from_numpy(f).to(dev) for f in frags]
        gb, grep = se.fragment_recover(d[0], d[1], d[2], n, W, L, KEY, iv, flags=flags, block_offset=boff)
        ob2, orep = orc.recover(frags[0], frags[1], frags[2], n, W, L, KEY, iv, flags=flags, block_offset=boff)
        assert np.array_equal(gb.cpu().numpy(), ob2)
        assert tuple(grep.cpu().tolist()) == orep
    finally:
        se.kernel_choice(prev)
