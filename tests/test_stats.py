"""Security battery (NEXT row f2): the oracle's sums are pinned to numpy
re-derivations of the definitions, the product's host-side metric formulas
to numpy's own (entropy of a known PDF, np.corrcoef, bit counts), and the
protected fragments meet the paper's reported statistics (Table 5.1-5.4:
entropy of 1 MB protected chunks 7.9991-7.9995; Dif and KS ~50%,
P:2555; adjacent correlation ~0)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synth
import paper_1803_04880_b200 as se

KEY = synth.KEY
IV = synth.iv_for(2)


def numpy_sums(x, y, W):
    n = len(y)
    y64, x64 = y.astype(np.int64), x.astype(np.int64)
    out = [n] + list(np.bincount(x, minlength=256)) + list(np.bincount(y, minlength=256))
    out += [x64.sum(), y64.sum(), (x64 * x64).sum(), (y64 * y64).sum(), (x64 * y64).sum(),
            int(np.unpackbits(x ^ y).sum())]
    R = -(-n // W)
    pad = np.full(R * W, -1, dtype=np.int64)
    pad[:n] = y64
    M = pad.reshape(R, W)
    for a, b in ((M[:, :-1], M[:, 1:]), (M[:-1, :], M[1:, :]), (M[:-1, :-1], M[1:, 1:])):
        m = (a >= 0) & (b >= 0)
        a, b = a[m], b[m]
        out += [m.sum(), a.sum(), b.sum(), (a * a).sum(), (b * b).sum(), (a * b).sum()]
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("n,W", [(1, 8), (1000, 24), (4096, 64), (50000, 333)])
def test_oracle_sums_match_numpy(orc, n, W):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, n, dtype=np.uint8)
    y = synth.text_like(n, n)
    words, joint = orc.stats(y, W, x=x)
    assert np.array_equal(words, numpy_sums(x, y, W))
    ref = np.bincount(x.astype(np.int64) * 256 + y, minlength=65536)
    assert np.array_equal(joint, ref.astype(np.uint64))


def test_metric_formulas(orc):
    rng = np.random.default_rng(3)
    # uniform PDF: entropy exactly 8, chi^2 exactly 0
    y = np.repeat(np.arange(256, dtype=np.uint8), 40)
    m = se.stats_metrics(orc.stats(y, 64)[0])
    assert math.isclose(m["entropy_y"], 8.0) and m["chi2_y"] == 0
    # constant: entropy 0
    assert se.stats_metrics(orc.stats(np.full(1000, 7, np.uint8), 10)[0])["entropy_y"] == 0
    # r_xy against numpy; Dif of complement = 100 %, of itself = 0 %
    x = rng.integers(0, 256, 20000, dtype=np.uint8)
    y = (x // 2 + rng.integers(0, 100, 20000)).astype(np.uint8)
    words, joint = orc.stats(y, 100, x=x)
    m = se.stats_metrics(words, joint)
    assert math.isclose(m["r_xy"], np.corrcoef(x.astype(float), y.astype(float))[0, 1], rel_tol=1e-9)
    assert se.stats_metrics(orc.stats(~x, 100, x=x)[0])["dif_bits_pct"] == 100.0
    mi = se.stats_metrics(*orc.stats(x, 100, x=x))
    assert mi["dif_bits_pct"] == 0.0 and math.isclose(mi["nmi"], 1.0, rel_tol=1e-9)
    # adjacent correlation of a horizontal ramp matrix: rho_h = 1
    ramp = np.tile(np.arange(64, dtype=np.uint8), 64)
    assert math.isclose(se.stats_metrics(orc.stats(ramp, 64)[0])["rho_h"], 1.0, rel_tol=1e-9)


def test_protected_fragments_meet_paper_statistics(orc):
    """1 MiB bitmap-like chunk (the paper's chunk size), oracle fragments."""
    W = 1024
    x = synth.bitmap(1024, 1024 // 3 + 1, 3, 11).reshape(-1)[: 1 << 20]
    a, b, c = orc.protect(x, W, 2, KEY, IV)
    m = se.stats_metrics(*orc.stats(c, W, x=x[: c.size]))
    assert m["entropy_y"] > 7.999                       # Table 5.4: 7.9991-7.9995
    assert 49.5 < m["dif_bits_pct"] < 50.5              # Dif ~ 50 %
    assert abs(m["r_xy"]) < 0.01 and m["nmi"] < 0.01    # r_xy, NMI ~ 0
    assert max(abs(m["rho_h"]), abs(m["rho_v"]), abs(m["rho_d"])) < 0.01
    k2 = KEY[:3] + bytes([KEY[3] ^ 0x04]) + KEY[4:]
    _, _, c2 = orc.protect(x, W, 2, k2, IV)
    ks = se.stats_metrics(orc.stats(c2, W, x=c)[0])["dif_bits_pct"]
    assert 49.5 < ks < 50.5                             # KS ~ 50 %
    # the original bitmap is far from uniform: the battery discriminates
    mo = se.stats_metrics(orc.stats(x, W)[0])
    assert mo["entropy_y"] < 7.9 and mo["rho_h"] > 0.5
