"""GPU parity of FULL-matrix mode (row a11) against the oracle, bit-exact:
whole-matrix Mallat coefficients (line-based lifting with row / column halos, borders reflected per
level), footprint fragments with the FULL widths (C23), recover and the
corruption report.  Sizes span several 64 x 128 tiles in both directions,
ragged tails and matrices smaller than one tile."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = bytes.fromhex("8899aabbccddeeff0011223344556677")
FULL = se.MODE_FULL

# (n, W): several tiles wide/tall, ragged tails, tiny matrices
CASES = [(64, 8), (8 * 24, 24), (1000, 40), (384 * 200 - 7, 384), (256 * 136, 256), (520 * 72 + 5, 520),
         (128 * 129, 128), (1024 * 96, 1024)]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def to_dev(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def data(n, seed):
    w = 64
    return synth.bitmap(-(-n // (3 * w)) + 1, w, 3, seed).reshape(-1)[:n] if seed % 2 else synth.random_bytes(n, seed)


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("n,W", CASES)
def test_dwt_full_parity(dev, orc, n, W, L):
    x = data(n, n + W + L)
    coef = se.dwt_fwd(to_dev(x, dev), W, L, mode=FULL)
    ref = orc.dwt_fwd(x, W, L, orc.MODE_FULL)
    got = coef.cpu().numpy().astype(np.int32)
    if not np.array_equal(got, ref):
        bad = np.argwhere(got != ref)
        pytest.fail(f"{len(bad)} coefficients differ, first at {bad[:5].tolist()}")
    back = se.dwt_inv(coef, n, W, L, mode=FULL)
    assert np.array_equal(back.cpu().numpy(), x)


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("n,W", CASES[:6])
def test_protect_recover_full_parity(dev, orc, n, W, L):
    x = data(n, 3 * n + L)
    for flags in (0, se.FLAG_PUBLIC_PLAIN):
        a, b, c = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV, mode=FULL, flags=flags)
        oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL, flags=flags)
        assert np.array_equal(a.cpu().numpy(), oa), "A'"
        assert np.array_equal(b.cpu().numpy(), ob), "B'"
        assert np.array_equal(c.cpu().numpy(), oc), "C'"
        back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, IV, mode=FULL, flags=flags)
        assert np.array_equal(back.cpu().numpy(), x)
        assert rep.cpu().tolist() == [-1, 0]


def test_full_corruption_report(dev, orc):
    n, W, L = 384 * 200, 384, 2
    x = data(n, 5)
    a, b, c = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
    c2 = c.copy()
    c2[480 * 300 // 8] ^= 0xF0           # damage footprint 300's level-1 details
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c2, dev), n, W, L, KEY, IV, mode=FULL)
    oback, orep = orc.recover(a, b, c2, n, W, L, KEY, IV, mode=orc.MODE_FULL)
    assert np.array_equal(back.cpu().numpy(), oback)
    assert tuple(rep.cpu().tolist()) == orep


def test_full_c4_shape_sampled(dev, orc):
    """C4-FULL geometry at reduced height (W = 32768 as in SURVEY §8.2.1): the
    whole-matrix transform round-trips and sampled footprints match the oracle."""
    W, R, L = 32768, 64, 2
    x = synth.random_bytes(W * R, 4)
    xt = to_dev(x, dev)
    a, b, c = se.fragment_protect(xt, W, L, KEY, IV, mode=FULL)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
    assert np.array_equal(a.cpu().numpy(), oa) and np.array_equal(b.cpu().numpy(), ob)
    assert np.array_equal(c.cpu().numpy(), oc)
    back, rep = se.fragment_recover(a, b, c, x.size, W, L, KEY, IV, mode=FULL)
    assert torch.equal(back, xt) and rep.cpu().tolist() == [-1, 0]


# FULL-mode row stripes with halo rows (row e for a11): (n, W) with several
# stripes per file, stripe edges inside 64-row tiles, ragged last stripe
STRIPE_CASES = [(256 * 200 + 77, 256), (128 * 520, 128), (1024 * 96, 1024), (64 * 1000 + 3, 64)]


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("n,W", STRIPE_CASES)
@pytest.mark.parametrize("world", [2, 3, 5])
def test_full_stripes_equal_whole_file(dev, orc, n, W, L, world):
    """Each stripe protected from its rows + halo rows only, and recovered from
    its fragments + halo block rows only: the concatenated streams equal the
    whole-file FULL streams (and the oracle's), the bytes equal the input."""
    from paper_1803_04880_b200 import shard
    x = data(n, n + W + L + world)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
    plan = [s for s in shard.plan_full_stripes(n, W, L, world) if s is not None]
    assert len(plan) >= 2
    got = {k: [] for k in "abc"}
    for st in plan:
        src = to_dev(x[st["src_byte_begin"]: st["src_byte_end"]], dev)
        a, b, c = se.fragment_protect_stripe(src, n, W, L, KEY, IV, st["row_begin"], st["row_end"], st["src_row0"])
        for k, t in zip("abc", (a, b, c)):
            got[k].append(t.cpu().numpy())
    for k, ref in zip("abc", (oa, ob, oc)):
        assert np.array_equal(np.concatenate(got[k]), ref), k
    back = []
    for st in plan:
        ins = [to_dev(s[slice(*st["rec_in"][k])], dev) for k, s in zip("abc", (oa, ob, oc))]
        out, rep = se.fragment_recover_stripe(*ins, n, W, L, KEY, IV, st["row_begin"], st["row_end"],
                                              st["rec_row0"], st["rec_rows"])
        assert rep.cpu().tolist() == [-1, 0]
        back.append(out.cpu().numpy())
    assert np.array_equal(np.concatenate(back), x)


def test_full_stripe_corruption_report(dev, orc):
    """A flipped C' bit in stripe 1: its bytes equal the oracle's whole-file
    recovery of the damaged streams; the report uses stripe-local indices."""
    from paper_1803_04880_b200 import shard
    n, W, L = 256 * 256, 256, 2
    x = data(n, 11)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
    plan = [s for s in shard.plan_full_stripes(n, W, L, 3) if s is not None]
    st = plan[1]
    blk = st["block_offset"] + 5
    oc2 = oc.copy()
    oc2[blk * 60 + 7] ^= 0xFF
    oback, orep = orc.recover(oa, ob, oc2, n, W, L, KEY, IV, mode=orc.MODE_FULL)
    ins = [to_dev(s[slice(*st["rec_in"][k])], dev) for k, s in zip("abc", (oa, ob, oc2))]
    out, rep = se.fragment_recover_stripe(*ins, n, W, L, KEY, IV, st["row_begin"], st["row_end"],
                                          st["rec_row0"], st["rec_rows"])
    assert np.array_equal(out.cpu().numpy(), oback[st["byte_begin"]: st["byte_end"]])
    first, bad = rep.cpu().tolist()
    assert (first + st["block_offset"], bad) == orep if orep[1] else (first, bad) == (-1, 0)
    # a window without its halo is refused
    with pytest.raises(se.SEError):
        se.fragment_recover_stripe(*ins, n, W, L, KEY, IV, st["row_begin"], st["row_end"],
                                   st["row_begin"], st["row_end"] - st["row_begin"])


def _fuzz_cases(k=12, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(k):
        W = 8 * int(rng.integers(1, 200))
        rows = int(rng.integers(1, 90))
        n = max(1, W * rows - int(rng.integers(0, W)))
        out.append((n, W, int(rng.integers(1, 4))))
    return out


@pytest.mark.parametrize("n,W,L", _fuzz_cases())
def test_full_streaming_fuzz(dev, orc, n, W, L):
    """Seeded random shapes for the streaming FULL transform (column groups of
    30 / 28 chunks, row segments with halos, ragged tails): coefficients
    bit-exact and the round trip exact."""
    x = synth.random_bytes(n, n ^ W)
    coef = se.dwt_fwd(to_dev(x, dev), W, L, mode=FULL)
    assert np.array_equal(coef.cpu().numpy().astype(np.int32), orc.dwt_fwd(x, W, L, orc.MODE_FULL))
    assert np.array_equal(se.dwt_inv(coef, n, W, L, mode=FULL).cpu().numpy(), x)


@pytest.mark.parametrize("seg", [64, 128, 256])
@pytest.mark.parametrize("L", [1, 2, 3])
def test_full_segment_lengths(dev, orc, seg, L):
    """only 32-row segments were ever compared.  Force each
    segment length (se_full_segment_rows) on a matrix several segments tall
    with a ragged last segment: transform, inverse and FULL fragments equal
    the oracle."""
    n, W = 256 * 1000 - 77, 256                      # R = 1000 rows: 4 / 8 / 16 segments + ragged
    x = data(n, seg + L)
    prev = se.full_segment_rows(seg)
    try:
        coef = se.dwt_fwd(to_dev(x, dev), W, L, mode=FULL)
        ref = orc.dwt_fwd(x, W, L, orc.MODE_FULL)
        assert np.array_equal(coef.cpu().numpy().astype(np.int32), ref)
        assert np.array_equal(se.dwt_inv(coef, n, W, L, mode=FULL).cpu().numpy(), x)
        a, b, c = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV, mode=FULL)
        oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
        assert np.array_equal(a.cpu().numpy(), oa)
        assert np.array_equal(b.cpu().numpy(), ob)
        assert np.array_equal(c.cpu().numpy(), oc)
        back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, IV, mode=FULL)
        assert np.array_equal(back.cpu().numpy(), x) and rep.cpu().tolist() == [-1, 0]
    finally:
        se.full_segment_rows(prev)


def test_full_segment_knob_rejects_other_lengths(dev):
    with pytest.raises(se.SEError):
        se.full_segment_rows(48)
