"""Hand-derived pins for the two DWT conventions the round-1 pins left open.

* Eq. 5.1-5.2's floor ("the largest integer not exceeding a") on
  predict and update sums that are negative and not divisible by 2 / 4
  (`golden/eq5_1_floor_negative_odd.txt`): truncation toward zero, the
  plausible C mistake, gives different integers.
* Rows before columns at every level ("first, in horizontal
  direction ... then ... vertical"; reading C5) on blocks where the two pass
  orders give different integers (`golden/pass_order_block.txt`).

Each expected value is derived by hand in the fixture's header from the
paper's equations; none comes from the oracle or the CUDA path.  The pins
are plain functions so `test_oracle_mutations.py` can run them against
deliberately broken builds of the oracle.
"""
from __future__ import annotations

import numpy as np

from conftest import golden_lines


def _ints(s):
    return np.array(s.split(), dtype=np.int32)


def pin_floor_1d(orc):
    for ln in golden_lines("eq5_1_floor_negative_odd.txt"):
        lhs, rhs = ln.split("|")
        x, y = _ints(lhs), _ints(rhs)
        assert np.array_equal(orc.lift_fwd_1d(x), y), (x, orc.lift_fwd_1d(x), y)
        assert np.array_equal(orc.lift_inv_1d(y), x), (y, orc.lift_inv_1d(y), x)


def _pass_order_cases():
    for ln in golden_lines("pass_order_block.txt"):
        head, inp, exp = ln.split("|")
        name, rows, cols, levels = head.split()
        rows, cols, levels = int(rows), int(cols), int(levels)
        yield name, levels, _ints(inp).reshape(rows, cols), _ints(exp).reshape(rows, cols)


def pin_pass_order_region(orc):
    """The level step on a region (the oracle's dyadic 2-D transform), both directions."""
    for name, levels, x, y in _pass_order_cases():
        got = orc.dwt2_fwd_region(x, levels)
        assert np.array_equal(got, y), (name, levels, got)
        assert np.array_equal(orc.dwt2_inv_region(y, levels), x), (name, levels)


def pin_pass_order_bytes(orc):
    """The same block through the byte-level BLOCK8 and FULL transforms
    (centering C8: byte = x + 128), both directions."""
    for name, levels, x, y in _pass_order_cases():
        if x.shape != (8, 8):
            continue
        data = (x + 128).astype(np.uint8).reshape(-1)
        for mode in (orc.MODE_BLOCK8, orc.MODE_FULL):
            coef = orc.dwt_fwd(data, 8, levels, mode)
            assert np.array_equal(coef, y), (name, levels, mode, coef)
            back, bad = orc.dwt_inv(y, 64, 8, levels, mode)
            assert bad == 0 and np.array_equal(back, data), (name, levels, mode)


PINS = [pin_floor_1d, pin_pass_order_region, pin_pass_order_bytes]


def test_floor_negative_odd_sums(orc):
    pin_floor_1d(orc)


def test_pass_order_region(orc):
    pin_pass_order_region(orc)


def test_pass_order_bytes(orc):
    pin_pass_order_bytes(orc)
