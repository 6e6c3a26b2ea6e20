"""GPU parity of the persistent tile kernels (k_tile.cu), the single-file
BLOCK8 hot path: bulk-copy ("fast") tiles in both shared-memory layouts
(contiguous whole block rows; per-row runs), tiles spanning two block rows,
many tiles per CTA (the input and keystream rings wrap), ragged ends on the
per-thread path, widths that rule out bulk copies, all levels, masked and
PUBLIC_PLAIN, block offsets - every stream byte against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = bytes.fromhex("00112233445566778899aabbccddeef0")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    prev = se.kernel_choice(se.KERNEL_TILE)       # these cases are below the auto threshold
    yield torch.device("cuda:0")
    se.kernel_choice(prev)


def to_dev(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


# (n, W, L): TILE = 512 blocks (L = 2, 3), 256 (L = 1)
CASES = [
    (512 * 64 * 3, 1024, 2),                  # 3 whole tiles, contiguous layout (W/8 = 128 divides 512)
    (512 * 64 * 3 + 777, 1024, 2),            # + a ragged tile on the per-thread path
    (6144 * 8 * 9 + 5, 6144, 2),              # C2-like rows: 768 blocks per row, tiles span two rows (runs)
    (4096 * 8 * 6 + 4096 * 3, 4096, 3),       # one block row per tile (contiguous), partial last row
    (12288 * 8 * 2 + 1000, 12288, 2),         # 1536 blocks per row: three tiles per row (runs)
    (256 * 8 * 70 + 3, 256, 1),               # L = 1, TILE = 256, 8 block rows per tile
    (1032 * 8 * 80, 1032, 2),                 # W % 16 != 0: every tile on the per-thread path
    (512 * 64 * 7 + 64, 8, 2),                # W = 8: one block per row, per-thread path
    (64 * 8 * 512 + 96, 64, 3),               # 8 blocks per row, 64 rows per tile (contiguous)
]


@pytest.mark.parametrize("n,W,L", CASES)
@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
def test_tile_parity(dev, orc, n, W, L, flags):
    x = synth.random_bytes(n, n + W + L)
    boff = 16 * 128 * 3 if L != 1 else 128 * 7
    a, b, c = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV, flags=flags, block_offset=boff)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, flags=flags, block_offset=boff)
    assert np.array_equal(a.cpu().numpy(), oa), "A'"
    assert np.array_equal(b.cpu().numpy(), ob), "B'"
    assert np.array_equal(c.cpu().numpy(), oc), "C'"
    back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, IV, flags=flags, block_offset=boff)
    assert rep.cpu().tolist() == [-1, 0]
    assert np.array_equal(back.cpu().numpy(), x)


def test_tile_rings_wrap(dev, orc):
    """~1200 tiles over 148 CTAs: every CTA runs 8 tiles, so the two-stage
    input ring and the four-slot keystream ring each wrap several times."""
    n, W, L = 1200 * 512 * 64 + 4321, 1024, 2
    x = synth.random_bytes(n, 5)
    xt = to_dev(x, dev)
    for flags in (0, se.FLAG_PUBLIC_PLAIN):
        a, b, c = se.fragment_protect(xt, W, L, KEY, IV, flags=flags)
        lay = orc.layout(n, W, L)
        ha, hb, hc = a.cpu().numpy(), b.cpu().numpy(), c.cpu().numpy()
        rng = np.random.default_rng(flags)
        tiles = (lay["n_blocks"] + 511) // 512
        for t in sorted({0, 1, 147, 148, 149, 295, 296, tiles - 2, tiles - 1} | set(rng.integers(0, tiles, 6).tolist())):
            b0, b1 = t * 512, min(lay["n_blocks"], (t + 1) * 512)
            bufs = [np.zeros(lay[k], np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes")]
            orc.protect(x, W, L, KEY, IV, flags=flags, block_range=(b0, b1), out=bufs)
            for s, (got, ref, bits) in enumerate(zip((ha, hb, hc), bufs, (40, 124, 480))):
                lo, hi = b0 * bits // 8, -(-b1 * bits // 8)
                assert np.array_equal(got[lo:hi], ref[lo:hi]), ("tile", t, "stream", s)
        back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, IV, flags=flags)
        assert rep.cpu().tolist() == [-1, 0]
        assert torch.equal(back, xt)


def test_tile_report_matches_oracle(dev, orc):
    """Damage inside fast tiles and in the ragged tile: the recovered bytes and
    the report equal the oracle's."""
    n, W, L = 512 * 64 * 5 + 3000, 1024, 2
    x = synth.bitmap(-(-n // (3 * 512)), 512, 3, 9).reshape(-1)[:n]
    a, b, c = orc.protect(x, W, L, KEY, IV)
    a2, b2, c2 = a.copy(), b.copy(), c.copy()
    a2[640 * 9 + 1] ^= 0x40                   # tile 2 (fast)
    b2[-3] ^= 0x01                            # ragged tile
    c2[60 * 1500 + 7] ^= 0x80                 # tile 2
    back, rep = se.fragment_recover(to_dev(a2, dev), to_dev(b2, dev), to_dev(c2, dev), n, W, L, KEY, IV)
    oback, orep = orc.recover(a2, b2, c2, n, W, L, KEY, IV)
    assert np.array_equal(back.cpu().numpy(), oback)
    assert tuple(rep.cpu().tolist()) == orep
    bad_key = bytes([KEY[0] ^ 1]) + KEY[1:]
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c, dev), n, W, L, bad_key, IV)
    oback, orep = orc.recover(a, b, c, n, W, L, bad_key, IV)
    assert tuple(rep.cpu().tolist()) == orep and orep[1] > 0
    assert np.array_equal(back.cpu().numpy(), oback)


@pytest.mark.parametrize("L", [1, 2, 3])
def test_tile_plain_garbage_fragments(dev, orc, L):
    """PUBLIC_PLAIN recovery of random fragments: every field at arbitrary
    values, so the inverse transform reaches its extreme magnitudes and most
    blocks fail the [0, 255] range check (the only damage signal without
    masks).  Recovered bytes and report equal the oracle's."""
    n, W = 512 * 64 * 4 + 2000, 1024
    lay = orc.layout(n, W, L)
    rng = np.random.default_rng(40 + L)
    a, b, c = (rng.integers(0, 256, lay[k], dtype=np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes"))
    if L == 2:                                 # extreme fields: all ones / all zeros on some blocks
        c[:3000] = 0xFF
        b[:1000] = 0x00
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c, dev), n, W, L, KEY, IV,
                                    flags=se.FLAG_PUBLIC_PLAIN)
    oback, orep = orc.recover(a, b, c, n, W, L, KEY, IV, flags=se.FLAG_PUBLIC_PLAIN)
    assert tuple(rep.cpu().tolist()) == orep and orep[1] > 0
    assert np.array_equal(back.cpu().numpy(), oback)


def test_tile_streams_on_one_stream_back_to_back(dev, orc):
    """Protect then recover then protect again on one non-default stream with
    no host synchronisation in between (programmatic dependent launch: each
    kernel must wait for the previous one's writes before reading)."""
    n, W, L = 512 * 64 * 40, 1024, 2
    x = synth.random_bytes(n, 77)
    xt = to_dev(x, dev)
    s = torch.cuda.Stream()
    lay = se.fragment_layout(n, W, L)
    a, b, c = (se._empty(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
    out = se._empty(n, dev)
    rep = torch.empty(2, dtype=torch.int64, device=dev)
    with torch.cuda.stream(s):
        for i in range(5):
            se.fragment_protect(xt, W, L, KEY, IV, out=(a, b, c), stream=s)
            out.zero_()
            se.fragment_recover(a, b, c, n, W, L, KEY, IV, out=out, report=rep, stream=s)
            xt.copy_(out)                                 # the next protect reads what recover wrote
    s.synchronize()
    assert np.array_equal(out.cpu().numpy(), x) and rep.cpu().tolist() == [-1, 0]
    oa, _, _ = orc.protect(x, W, L, KEY, IV)
    assert np.array_equal(a.cpu().numpy(), oa)
