"""Row f4 on the GPU: fault injection into protected fragments.

Single bit flips (and a burst) are injected into A', B', C' of a Chapter 5
file and into Fragment 1 / Fragment 2 of a Chapter 4 image; the GPU recovery
of the damaged fragments must equal the oracle's recovery of the same damaged
fragments (bit-exact for Chapter 5, decided bytes for Chapter 4) and the
damage must stay inside the 8x8 block(s) whose record holds the flipped bits.
The containers round-trip GPU-produced fragments (se_container.h).
"""
from __future__ import annotations

import numpy as np
import pytest

import synth
from dct_helpers import blocks, near_half

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = synth.iv_for(2, 7)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def to_dev(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def flip(s, bits):
    s = s.copy()
    for b in bits:
        s[b // 8] ^= 0x80 >> (b % 8)
    return s


def block_of(i, W):
    return (i // W) // 8 * (W // 8) + (i % W) // 8


@pytest.mark.parametrize("stream,rec_bits", [(0, 40), (1, 124), (2, 480)])
def test_bit_flips_dwt(dev, orc, stream, rec_bits):
    W, L, n = 1024, 2, 1 << 18
    x = synth.bitmap(n // 1536 + 1, 512, 3, 17).reshape(-1)[:n]
    st = list(orc.protect(x, W, L, KEY, IV))
    rng = np.random.default_rng(stream)
    nb = n // 64
    for trial in range(12):
        hit = sorted(set(int(b) for b in rng.integers(0, nb * rec_bits, size=1 + trial % 3)))
        dam = st.copy()
        dam[stream] = flip(st[stream], hit)
        back, rep = se.fragment_recover(*(to_dev(s, dev) for s in dam), n, W, L, KEY, IV)
        oback, orep = orc.recover(*dam, n, W, L, KEY, IV)
        got = back.cpu().numpy()
        assert np.array_equal(got, oback) and tuple(rep.cpu().tolist()) == orep
        blocks_hit = {b // rec_bits for b in hit}
        changed = {block_of(int(i), W) for i in np.nonzero(got != x)[0]}
        assert changed <= blocks_hit                  # confined
        if stream != 2:
            assert changed == blocks_hit              # A / B damage always shows (masks change)


def test_burst_error_dwt(dev, orc):
    """A 64-bit burst in C' (as a channel error would) touches at most the two
    records it straddles."""
    W, L, n = 256, 2, 256 * 64
    x = synth.random_bytes(n, 3)
    a, b, c = orc.protect(x, W, L, KEY, IV)
    start = 480 * 37 + 450                             # straddles records 37 and 38
    c2 = flip(c, range(start, start + 64))
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c2, dev), n, W, L, KEY, IV)
    oback, orep = orc.recover(a, b, c2, n, W, L, KEY, IV)
    got = back.cpu().numpy()
    assert np.array_equal(got, oback) and tuple(rep.cpu().tolist()) == orep
    assert {block_of(int(i), W) for i in np.nonzero(got != x)[0]} <= {37, 38}


@pytest.mark.parametrize("stream", ["A", "P"])
def test_bit_flips_dct(dev, orc, stream):
    W, H, level = 256, 64, 2
    x = synth.bitmap(H, W, 1, 23).reshape(-1)
    a, p = orc.dct_protect(x, W, H, 1, level, KEY, IV)
    clean = orc.dct_recover(a, p, W, H, 1, level, KEY, IV)
    rng = np.random.default_rng(7)
    nrec = (W // 8) * (H // 8)
    for _ in range(8):
        if stream == "A":
            bit = int(rng.integers(0, nrec * 66))
            a2, p2, rec = flip(a, [bit]), p, bit // 66
        else:
            i = int(rng.integers(0, W * H))
            a2, p2, rec = a, flip(p, [8 * i + int(rng.integers(0, 8))]), block_of(i, W)
        got = se.dct_recover(to_dev(a2, dev), to_dev(p2, dev), W, H, 1, level, KEY, IV).cpu().numpy()
        ref, real = orc.dct_recover(a2, p2, W, H, 1, level, KEY, IV, real=True)
        tie = near_half(real, 2.0 ** -8)
        g, r = blocks(got, W, H, 1).reshape(nrec, 64), blocks(ref, W, H, 1).reshape(nrec, 64)
        assert np.array_equal(g[~tie], r[~tie]) and np.abs(g.astype(int) - r).max() <= 1
        changed = {block_of(int(i), W) for i in np.nonzero(ref != clean)[0]}
        assert changed <= {rec}                                    # confined to its block


def test_containers_carry_gpu_fragments(dev, orc):
    """GPU protect -> host -> A+B-local / C-remote containers -> open -> GPU recover."""
    W, L, n = 1024, 2, 1 << 20
    x = synth.bitmap(n // 1536 + 1, 512, 3, 29).reshape(-1)[:n]
    a, b, c = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV)
    info = se.container_info(se.SCHEME_DWT_BLOCK8, n, W, L, IV)
    parts = se.disperse(info, {0: a, 1: b, 2: c}, se.LAYOUT_AB_LOCAL)
    merged = {}
    for part in [parts["local"]] + parts["remote"]:
        merged.update(se.container_open(part)[1])
    back, rep = se.fragment_recover(*(to_dev(merged[i], dev) for i in range(3)), n, W, L, KEY, IV)
    assert np.array_equal(back.cpu().numpy(), x) and rep.cpu().tolist() == [-1, 0]
