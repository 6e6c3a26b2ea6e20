"""The integer recipes the CUDA kernels use in place of the textbook forms,
checked on the host against the oracle (which follows Eq. 5.1-5.2 as
written).  These are derivation checks: each function below transcribes one
kernel formula (se_device.cuh) with numpy's arithmetic shifts (the kernels'
SHF / LEA.HI floors), so a wrong identity in DESIGN.md §5.3 fails here
without a GPU; the GPU parity tests then compare the kernels themselves.

  lift_fwd_mix   d' = x_o + ((3 - x_l - x_r) >> 1) = d + 1,
                 s  = x_e + ((d'_l + d'_r) >> 2) (first: x_e + (d'_0 >> 1)) (Eq. 5.1-5.2)
  lift_inv_mix   x_e = s + ((1 - d_l - d_r) >> 2) (first: s + ((-d) >> 1)), x_o = d + ((x_l + x_r) >> 1)
  dwt8_fwd_mix   every band but the final LL leaves as v + 1
  out_of_range_pairs  (v_a + 2^16 v_b) & 0xff00ff00 != 0  <=>  v_a or v_b outside [0, 255]
                 for |v| < 2^15, and every inverse of <= 11-bit fields stays inside that
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle


def lift_fwd_mix(x):
    """se_device.cuh lift_fwd_mix, one 1-D lift of N = len(x) samples."""
    x = [int(v) for v in x]
    n_, h = len(x), len(x) // 2
    nn = [0] + [3 - x[2 * k] for k in range(1, h)]
    d = []
    for k in range(h):
        if 2 * k + 2 < n_:
            d.append(x[2 * k + 1] + ((-x[2 * k] + nn[k + 1]) >> 1))
        else:
            d.append(x[2 * k + 1] - x[2 * k] + 1)
    s = [x[0] + (d[0] >> 1) if k == 0 else x[2 * k] + ((d[k - 1] + d[k]) >> 2) for k in range(h)]
    return s + d


def lift_inv_mix(y):
    """se_device.cuh lift_inv_mix."""
    y = [int(v) for v in y]
    n_, h = len(y), len(y) // 2
    m = [1 - y[h + k] for k in range(h)]
    x = [0] * n_
    x[0] = y[0] + ((-y[h]) >> 1)                   # floor((1 - 2 d) / 4) = floor(-d / 2)
    for k in range(1, h):
        x[2 * k] = y[k] + ((-y[h + k - 1] + m[k]) >> 2)
    for k in range(h):
        if 2 * k + 2 < n_:
            x[2 * k + 1] = y[h + k] + ((x[2 * k] + x[2 * k + 2]) >> 1)
        else:
            x[2 * k + 1] = x[2 * k] + y[h + k]
    return x


def dwt8_mix(v, levels, inverse=False):
    """dwt2_level_lean<M, INV, 3> over the levels, rows then columns (forward)."""
    v = np.array(v, dtype=np.int64)
    sizes = [8 >> l for l in range(levels)]
    for m in (reversed(sizes) if inverse else sizes):
        order = ("cols", "rows") if inverse else ("rows", "cols")
        for pas in order:
            for a in range(m):
                t = v[a, :m] if pas == "rows" else v[:m, a]
                r = lift_inv_mix(t) if inverse else lift_fwd_mix(t)
                if pas == "rows":
                    v[a, :m] = r
                else:
                    v[:m, a] = r
    return v


def band_bias(levels):
    """+1 on every position outside the final LL."""
    b = np.ones((8, 8), dtype=np.int64)
    s = 8 >> levels
    b[:s, :s] = 0
    return b


@pytest.mark.parametrize("n", [2, 4, 8])
def test_lift_fwd_mix_is_oracle_plus_one_on_d(n):
    rng = np.random.default_rng(n)
    for _ in range(3000):
        x = rng.integers(-3000, 3000, n)
        ref = oracle.lift_fwd_1d(x.astype(np.int32)).astype(np.int64)
        got = np.array(lift_fwd_mix(x))
        h = n // 2
        assert np.array_equal(got[:h], ref[:h]), (x, got, ref)
        assert np.array_equal(got[h:], ref[h:] + 1), (x, got, ref)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_lift_inv_mix_inverts_the_oracle(n):
    rng = np.random.default_rng(10 + n)
    for _ in range(3000):
        y = rng.integers(-3000, 3000, n)
        ref = oracle.lift_inv_1d(y.astype(np.int32)).astype(np.int64)
        assert np.array_equal(np.array(lift_inv_mix(y)), ref), y


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_dwt8_mix_band_offsets(levels):
    """Forward 2-D mixed-pipe transform = oracle + 1 outside the final LL;
    the inverse of the exact coefficients is the oracle's inverse."""
    rng = np.random.default_rng(levels)
    for _ in range(300):
        blk = rng.integers(0, 256, (8, 8))
        ref = oracle.dwt2_fwd_region(blk.astype(np.int32), levels).astype(np.int64)
        got = dwt8_mix(blk, levels)
        assert np.array_equal(got, ref + band_bias(levels))
        assert np.array_equal(dwt8_mix(ref, levels, inverse=True), blk)


def out_of_range_pairs(va, vb):
    w = (va + (vb << 16)) & 0xFFFFFFFF
    return (w & 0xFF00FF00) != 0


def test_out_of_range_pairs_exact_for_15_bit_samples():
    edge = np.array([-(1 << 15), -(1 << 15) + 1, -257, -256, -255, -2, -1, 0, 1, 127, 128, 254, 255, 256,
                     257, 511, 512, 65535 >> 1, (1 << 15) - 1], dtype=np.int64)
    rng = np.random.default_rng(7)
    vals = np.unique(np.concatenate([edge, rng.integers(-(1 << 15), 1 << 15, 400)]))
    va, vb = np.meshgrid(vals, vals)
    want = (va < 0) | (va > 255) | (vb < 0) | (vb > 255)
    assert np.array_equal(out_of_range_pairs(va, vb), want)


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_inverse_of_any_fields_stays_below_2_15(levels):
    """The premise of out_of_range_pairs: recovering arbitrary (corrupted)
    fields never leaves |v| < 2^15.  Bound = the inverse's impulse-response
    L1 norm per output x the largest field magnitude (11-bit offset binary:
    1024; LL also carries +128) plus the floors' slack, and a search over
    extreme sign patterns."""
    scale = 1 << 12
    resp = np.zeros((64, 64))
    for k in range(64):
        e = np.zeros((8, 8), dtype=np.int32)
        e.flat[k] = scale
        resp[:, k] = oracle.dwt2_inv_region(e, levels).reshape(-1) / scale
    bound = np.abs(resp).sum(axis=1).max() * (1024 + 128) + 64
    assert bound < (1 << 15), bound
    rng = np.random.default_rng(levels)
    worst = 0
    for j in range(64):                     # the sign pattern that maximises output j
        f = (np.sign(resp[j]) * 1024).astype(np.int32).reshape(8, 8)
        worst = max(worst, int(np.abs(oracle.dwt2_inv_region(f, levels)).max()))
    for _ in range(200):
        f = rng.choice([-1024, 1023], (8, 8)).astype(np.int32)
        worst = max(worst, int(np.abs(oracle.dwt2_inv_region(f, levels)).max()))
    assert worst < (1 << 15)
