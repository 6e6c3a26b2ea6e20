"""GPU security-battery sums (se_stats_accumulate, row f2) equal the oracle's
exactly (integer sums), including accumulation across calls, y-only mode,
ragged widths, and the statistics of GPU-protected fragments."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def to_dev(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


@pytest.mark.parametrize("n,W", [(1, 8), (17, 8), (1000, 24), (4096, 64), (100003, 333), (1 << 20, 1024)])
def test_stats_sums_parity(dev, orc, n, W):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, n, dtype=np.uint8)
    y = synth.text_like(n, n + 1)
    st, jt = se.stats_accumulate(to_dev(y, dev), W, x=to_dev(x, dev))
    words, joint = orc.stats(y, W, x=x)
    assert np.array_equal(st.cpu().numpy().astype(np.uint64), words)
    assert np.array_equal(jt.cpu().numpy().astype(np.uint64), joint)
    sy, _ = se.stats_accumulate(to_dev(y, dev), W)
    wy, _ = orc.stats(y, W)
    assert np.array_equal(sy.cpu().numpy().astype(np.uint64), wy)


def test_stats_accumulate_across_calls(dev, orc):
    rng = np.random.default_rng(5)
    parts = [rng.integers(0, 256, k, dtype=np.uint8) for k in (1000, 2048, 777)]
    st, _ = se.stats_accumulate(to_dev(parts[0], dev), 64)
    for p in parts[1:]:
        st, _ = se.stats_accumulate(to_dev(p, dev), 64, stats=st)
    ref = sum(orc.stats(p, 64)[0].astype(np.int64) for p in parts)
    got = st.cpu().numpy()
    # histograms and moments add; n adds
    assert np.array_equal(got[:519], ref[:519])


def test_gpu_fragments_statistics(dev):
    W = 1024
    x = synth.bitmap(1024, 1024 // 3 + 1, 3, 12).reshape(-1)[: 1 << 20]
    xt = to_dev(x, dev)
    _, _, c = se.fragment_protect(xt, W, 2, synth.KEY, synth.iv_for(2))
    m = se.stats_metrics(*se.stats_accumulate(c, W, x=xt[: c.numel()]))
    assert m["entropy_y"] > 7.999 and 49.5 < m["dif_bits_pct"] < 50.5 and m["nmi"] < 0.01
    assert max(abs(m["rho_h"]), abs(m["rho_v"]), abs(m["rho_d"]), abs(m["r_xy"])) < 0.01
