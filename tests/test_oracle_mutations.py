"""Mutation check of the oracle's DWT pins ("What's weak" 1).

Each case copies `oracle/*.c`, applies one plausible mistake to the lifting
code, builds the copy with gcc and runs the paper pins against it through
`oracle.library_override`.  A pin set that lets a mutant through is not
pinning that convention.  The two conventions round 1 left open -
Eq. 5.1's floor and rows-before-columns - must be caught
by the hand-derived pins of `test_oracle_pins.py` specifically; every other
mutant must be caught by at least one pin.
"""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

import test_oracle_dwt as dwt_pins
import test_oracle_pins as new_pins

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")

FWD_ROWS = """    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j) in[j] = a[(size_t)i * stride + j];
        oracle_lift_fwd_1d(in, out, cols);
        for (int j = 0; j < cols; ++j) a[(size_t)i * stride + j] = out[j];
    }
"""
FWD_COLS = """    for (int j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) in[i] = a[(size_t)i * stride + j];
        oracle_lift_fwd_1d(in, out, rows);
        for (int i = 0; i < rows; ++i) a[(size_t)i * stride + j] = out[i];
    }
"""
INV_COLS = FWD_COLS.replace("fwd", "inv")
INV_ROWS = FWD_ROWS.replace("fwd", "inv")

# name -> [(old, new, expected count)] applied to dwt53.c
MUTATIONS = {
    # Eq. 5.1 / 5.2 with C truncation instead of the floor (both directions)
    "predict_trunc": [("floor_div(xl + xr, 2)", "(xl + xr) / 2", 1),
                      ("floor_div(x[2 * k] + xr, 2)", "(x[2 * k] + xr) / 2", 1)],
    "update_trunc": [("floor_div(dm1 + d[k] + 2, 4)", "(dm1 + d[k] + 2) / 4", 2)],
    "floor_is_trunc": [("if ((a % b) != 0 && a < 0) q -= 1;", "", 1)],
    # columns before rows at every level (and the matching inverse)
    "cols_first": [(FWD_ROWS + FWD_COLS, FWD_COLS + FWD_ROWS, 1),
                   (INV_COLS + INV_ROWS, INV_ROWS + INV_COLS, 1)],
    # Eq. 5.2's printed '-' (reading C3)
    "update_sign_minus": [("s[k] = x[2 * k] + floor_div", "s[k] = x[2 * k] - floor_div", 1),
                          ("x[2 * k] = s[k] - floor_div", "x[2 * k] = s[k] + floor_div", 1)],
    # the +2 rounding offset of Eq. 5.2 dropped
    "update_no_offset": [("floor_div(dm1 + d[k] + 2, 4)", "floor_div(dm1 + d[k], 4)", 2)],
    # d(-1) = 0 instead of the symmetric d(-1) = d(0) (reading C2), both directions
    "edge_zero_detail": [("(k == 0) ? predict_at(x, n, -1) : d[k - 1]", "(k == 0) ? 0 : d[k - 1]", 1),
                         ("(k == 0) ? d[0] : d[k - 1]", "(k == 0) ? 0 : d[k - 1]", 1)],
    # [d | s] instead of [s | d] (reading C6)
    "detail_first": [("y[k] = s[k]; y[h + k] = d[k];", "y[k] = d[k]; y[h + k] = s[k];", 1),
                     ("const int32_t* s = y;\n    const int32_t* d = y + h;",
                      "const int32_t* d = y;\n    const int32_t* s = y + h;", 1)],
}
NAMED = {"predict_trunc", "cols_first", "update_trunc", "floor_is_trunc"}   # caught by the new hand pins


def build_mutant(tmp_path, name):
    src = os.path.join(tmp_path, "src")
    shutil.copytree(ORACLE, src, ignore=shutil.ignore_patterns("*.so", "__pycache__", "*.py"))
    path = os.path.join(src, "dwt53.c")
    text = open(path).read()
    for old, new, count in MUTATIONS[name]:
        assert text.count(old) == count, (name, old, text.count(old))
        text = text.replace(old, new)
    open(path, "w").write(text)
    so = os.path.join(tmp_path, f"liboracle_{name}.so")
    srcs = [os.path.join(src, f) for f in sorted(os.listdir(src)) if f.endswith(".c")]
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-w", "-o", so] + srcs + ["-lm"])
    return so


def _old_pins():
    return [dwt_pins.test_spec_hand_examples, dwt_pins.test_matrix_A_weights,
            dwt_pins.test_matrix_A_integer_exactness, dwt_pins.test_update_sign_is_plus,
            dwt_pins.test_level1_2d_is_separable_A, dwt_pins.test_eq_5_5_weights,
            dwt_pins.test_eq_5_5_integer_exactness, dwt_pins.test_impulse_block,
            dwt_pins.test_hand_ramp_block, dwt_pins.test_constant_blocks]


def failing(pins, orc):
    bad = []
    for pin in pins:
        try:
            pin(orc)
        except AssertionError:
            bad.append(pin.__name__)
    return bad


def test_unmutated_build_passes_every_pin(orc, tmp_path):
    """The harness itself: a copy built the same way passes all pins."""
    src = os.path.join(tmp_path, "src")
    shutil.copytree(ORACLE, src, ignore=shutil.ignore_patterns("*.so", "__pycache__", "*.py"))
    so = os.path.join(tmp_path, "liboracle_copy.so")
    srcs = [os.path.join(src, f) for f in sorted(os.listdir(src)) if f.endswith(".c")]
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-w", "-o", so] + srcs + ["-lm"])
    with orc.library_override(so):
        assert failing(new_pins.PINS + _old_pins(), orc) == []


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_pins_catch_mutation(orc, tmp_path, name):
    so = build_mutant(str(tmp_path), name)
    with orc.library_override(so):
        caught_new = failing(new_pins.PINS, orc)
        caught_all = caught_new + failing(_old_pins(), orc)
    assert caught_all, f"mutation {name} passes every DWT pin"
    if name in NAMED:
        assert caught_new, f"mutation {name} is not caught by the hand-derived convention pins"
