"""Pins for the oracle's integer 5/3 lifting DWT (rows a2-a4, a11).

Pinned to things other than the oracle itself:
  * the paper's matrix A: the oracle's exact 1st-level linear
    weights equal it entry for entry, and integer lifting equals IN.A
    exactly on inputs that make every floor exact;
  * the paper's 4x4 2nd-level matrix except its misprinted
    column 1, which must equal matrix A's own boundary stencil (column 3);
  * Eq. 5.5: all 25 printed weights of F(4,4), and exact
    integer agreement on bytes in {0, 64, 128, 192};
  * the printed range table, reproduced from the printed
    matrices; the true table and the paper's bit widths;
  * SPEC's hand examples and a hand-worked ramp block;
  * losslessness by round trip, and brute force on small inputs.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

from conftest import golden_lines, golden_matrix

IMP = 1 << 20   # impulse magnitude that makes every floor in 3 levels exact


def weights(orc, shape, levels):
    """Exact linear weights of the oracle's 2-D transform: W[out_r, out_c, in_r, in_c]."""
    R, C = shape
    W = np.zeros((R, C, R, C))
    for r in range(R):
        for c in range(C):
            x = np.zeros(shape, dtype=np.int32)
            x[r, c] = IMP
            W[:, :, r, c] = orc.dwt2_fwd_region(x, levels) / IMP
    return W


def weights_1d(orc, n):
    M = np.zeros((n, n))
    for r in range(n):
        x = np.zeros(n, dtype=np.int32)
        x[r] = IMP
        M[r] = orc.lift_fwd_1d(x) / IMP
    return M   # M[in, out]: same orientation as the paper's IN . A


# ---------------------------------------------------------------- 1-D pins

def test_spec_hand_examples(orc):
    for ln in golden_lines("spec_lifting_examples.txt"):
        lhs, rhs = ln.split("|")
        x = np.array(lhs.split(), dtype=np.int32)
        y = np.array(rhs.split(), dtype=np.int32)
        assert np.array_equal(orc.lift_fwd_1d(x), y)
        assert np.array_equal(orc.lift_inv_1d(y), x)


def test_matrix_A_weights(orc):
    A = golden_matrix("paper_matrix_A.txt")
    assert np.array_equal(weights_1d(orc, 8), A)


def test_matrix_A_integer_exactness(orc):
    """Integer lifting == IN.A exactly when centered inputs are multiples of 8."""
    A = golden_matrix("paper_matrix_A.txt")
    rng = np.random.default_rng(21)
    for _ in range(2000):
        x = rng.integers(-16, 16, size=8).astype(np.int32) * 8
        assert np.array_equal(orc.lift_fwd_1d(x), (x @ A).astype(np.int32))


def test_update_sign_is_plus(orc):
    """C3: the '-' printed in Eq. 5.2 would give low-band gain != 1 on a constant;
    the paper's matrix A columns 0-3 sum to 1 (DC preserved)."""
    A = golden_matrix("paper_matrix_A.txt")
    assert np.allclose(A[:, :4].sum(axis=0), 1.0)
    x = np.full(8, 100, dtype=np.int32)
    assert np.array_equal(orc.lift_fwd_1d(x), [100] * 4 + [0] * 4)


def test_4x4_matrix_except_misprinted_column(orc):
    P = golden_matrix("paper_matrix_4x4.txt")
    A = golden_matrix("paper_matrix_A.txt")
    M = weights_1d(orc, 4)
    for c in (0, 2, 3):
        assert np.array_equal(M[:, c], P[:, c]), c
    # column 1 (last low-pass output) has the boundary stencil of matrix A's
    # last low-pass column: rows 4..7 of A[:, 3]
    assert np.array_equal(M[:, 1], A[4:, 3])
    assert not np.array_equal(M[:, 1], P[:, 1])   # the misprint (reading C24)


@pytest.mark.parametrize("n", [2, 4, 6, 8, 16, 32])
def test_lift_round_trip_1d(orc, n):
    rng = np.random.default_rng(n)
    for _ in range(300):
        x = rng.integers(-2000, 2000, size=n).astype(np.int32)
        assert np.array_equal(orc.lift_inv_1d(orc.lift_fwd_1d(x)), x)


def test_two_sample_inverse_brute_force(orc):
    """N = 2: d = x1 - x0, s = x0 + floor((2d+2)/4); inverse exact on a dense grid."""
    vals = list(range(-512, 512, 3)) + [-512, -1, 0, 1, 511]
    for x0 in vals:
        for x1 in (-512, -511, -2, -1, 0, 1, 2, 510, 511, x0, -x0 - 1):
            x = np.array([x0, x1], dtype=np.int32)
            y = orc.lift_fwd_1d(x)
            assert y[1] == x1 - x0
            assert y[0] == x0 + math.floor((2 * (x1 - x0) + 2) / 4)
            assert np.array_equal(orc.lift_inv_1d(y), x)


# ---------------------------------------------------------------- 2-D pins

def test_level1_2d_is_separable_A(orc):
    """1st level = rows then columns with matrix A: F = A^T . IN . A."""
    A = golden_matrix("paper_matrix_A.txt")
    W = weights(orc, (8, 8), 1)
    expect = np.einsum("ri,cj->ijrc", A, A)     # A[r,i]*A[c,j] arranged [i,j,r,c]
    assert np.array_equal(W, expect)


def test_eq_5_5_weights(orc):
    W = weights(orc, (8, 8), 2)[3, 3]
    F = np.zeros((8, 8))
    for ln in golden_lines("paper_eq5_5_F44.txt"):
        r, c, w = ln.split()
        F[int(r), int(c)] = float(w)
    assert np.array_equal(W, F)
    assert math.isclose(np.abs(F).sum() * 128, 648.0)


def test_eq_5_5_integer_exactness(orc):
    F = np.zeros((8, 8))
    for ln in golden_lines("paper_eq5_5_F44.txt"):
        r, c, w = ln.split()
        F[int(r), int(c)] = float(w)
    rng = np.random.default_rng(22)
    blocks = rng.choice(np.array([0, 64, 128, 192], dtype=np.uint8), size=(500, 8, 8))
    data = blocks.transpose(1, 0, 2).reshape(8, 500 * 8)     # 500 blocks side by side
    coef = orc.dwt_fwd(data.reshape(-1), 500 * 8, 2)
    for b in range(500):
        x = blocks[b].astype(np.int64) - 128
        assert coef[3, 8 * b + 3] == int((F * x).sum())


def test_impulse_block(orc):
    data = np.full(64, 128, dtype=np.uint8)
    data[4 * 8 + 4] = 192
    coef = orc.dwt_fwd(data, 8, 2)
    assert coef[3, 3] == 49          # 0.765625 * 64 (Eq. 5.5, IN[4,4])


def test_hand_ramp_block(orc):
    data = np.array([[8 * i + j for j in range(8)] for i in range(8)], dtype=np.uint8)
    expect = np.array([[int(t) for t in ln.split()] for ln in golden_lines("hand_ramp_block.txt")])
    assert np.array_equal(orc.dwt_fwd(data.reshape(-1), 8, 2), expect)


def test_constant_blocks(orc):
    assert not orc.dwt_fwd(np.full(64, 128, np.uint8), 8, 2).any()     # all-128 -> zero
    for L in (1, 2, 3):
        for v in (0, 77, 255):
            coef = orc.dwt_fwd(np.full(64, v, np.uint8), 8, L)
            s = 8 >> L
            assert np.all(coef[:s, :s] == v - 128)
            low = np.zeros((8, 8), bool)
            low[:s, :s] = True
            assert not coef[~low].any()


def range_table(M8, M4):
    """max |coef| over inputs in [-128,128] of the 2-level map (rounding ignored),
    built from a 1-D level-1 matrix (8x8) and level-2 matrix (4x4), as P:2217-2233."""
    L1 = M8[:, :4]                     # low-pass outputs of level 1
    comp = L1 @ M4                     # 8 inputs -> 4 level-2 outputs (1-D)
    # 2-D separable: coef(i,j) weights = comp[:, i] (rows) x comp[:, j] (cols)
    T = np.zeros((4, 4))
    for i in range(4):
        for j in range(4):
            T[i, j] = np.abs(np.outer(comp[:, i], comp[:, j])).sum() * 128
    return np.ceil(T - 1e-9).astype(int)


def test_printed_range_table_reproduced_from_printed_matrices():
    A = golden_matrix("paper_matrix_A.txt")
    P4 = golden_matrix("paper_matrix_4x4.txt")
    printed = golden_matrix("paper_range_table.txt").astype(int)
    assert np.array_equal(range_table(A, P4), printed)


def test_true_range_table_and_widths(orc):
    W = weights(orc, (8, 8), 2)
    T = np.ceil(np.abs(W[:4, :4]).sum(axis=(2, 3)) * 128 - 1e-9).astype(int)
    printed = golden_matrix("paper_range_table.txt").astype(int)
    assert T.tolist() == [[338, 260, 468, 468], [260, 200, 360, 360],
                          [468, 360, 648, 648], [468, 360, 648, 648]]
    mask = np.ones((4, 4), bool)
    mask[1, :] = mask[:, 1] = False          # entries untouched by the misprint
    assert np.array_equal(T[mask], printed[mask])
    # widths: only the four 648 (HH2) entries need 11 bits
    need11 = T > 511
    assert need11.sum() == 4 and need11[2:, 2:].all()


def test_level1_bounds(orc):
    """|H| <= 255, |L| <= 192 after rows; |HH1| <= 511 -> 10 bits."""
    W = weights(orc, (8, 8), 1)
    lin = np.abs(W).sum(axis=(2, 3)) * 128
    assert lin[4:, 4:].max() == 512 and lin[:4, 4:].max() <= 384 and lin[4:, :4].max() <= 384
    # exact extremes by adversarial sign patterns (floors included)
    worst = {}
    for (i, j) in itertools.product(range(8), range(8)):
        for sgn in (1, -1):
            x = np.where(sgn * W[i, j] > 0, 255, 0).astype(np.uint8)
            v = orc.dwt_fwd(x.reshape(-1), 8, 1)[i, j]
            worst[(i, j)] = max(worst.get((i, j), 0), abs(int(v)))
    assert max(worst[(i, j)] for i in range(4, 8) for j in range(4, 8)) == 510
    assert max(v for v in worst.values()) <= 511


@pytest.mark.parametrize("L", [1, 2, 3])
def test_random_blocks_within_bounds_and_lossless(orc, L):
    rng = np.random.default_rng(100 + L)
    n_blocks = 40000
    data = rng.integers(0, 256, size=(8, 8 * n_blocks), dtype=np.uint8)
    data[:, : 8 * 64] = rng.choice(np.array([0, 255], np.uint8), size=(8, 8 * 64))   # extremes
    coef = orc.dwt_fwd(data.reshape(-1), 8 * n_blocks, L)
    assert np.abs(coef).max() <= (646 if L == 2 else 738 if L == 3 else 510)
    back, bad = orc.dwt_inv(coef, data.size, 8 * n_blocks, L)
    assert bad == 0 and np.array_equal(back, data.reshape(-1))


# ---------------------------------------------------------------- FULL mode (a11)

def test_full_mode_single_block_equals_block8(orc):
    rng = np.random.default_rng(31)
    for L in (1, 2, 3):
        x = rng.integers(0, 256, size=64, dtype=np.uint8)
        assert np.array_equal(orc.dwt_fwd(x, 8, L, orc.MODE_FULL), orc.dwt_fwd(x, 8, L))


def test_full_mode_interior_stencil_is_matrix_A(orc):
    """Interior level-1 FULL coefficients use matrix A's interior stencils
    (low: column 1, high: column 5) in both directions."""
    A = golden_matrix("paper_matrix_A.txt")
    lo_taps = A[2:7, 2]          # s2: the interior low-pass stencil
    hi_taps = A[2:5, 5]          # d1: the interior high-pass stencil
    assert np.count_nonzero(A[:, 2]) == 5 and np.count_nonzero(A[:, 5]) == 3
    W = weights(orc, (16, 16), 1)
    # coefficient LL1 (3,3) is the low output centred on input row/col 6
    k = np.zeros((16, 16))
    k[4:9, 4:9] = np.outer(lo_taps, lo_taps)
    assert np.array_equal(W[3, 3], k)
    # HH1 (8+3, 8+3) is centred on input 7 (odd)
    k = np.zeros((16, 16))
    k[6:9, 6:9] = np.outer(hi_taps, hi_taps)
    assert np.array_equal(W[11, 11], k)


@pytest.mark.parametrize("L", [1, 2, 3])
def test_full_mode_round_trip(orc, L):
    rng = np.random.default_rng(40 + L)
    for (n, w) in [(64 * 64, 64), (1000, 32), (24 * 40, 40)]:
        x = rng.integers(0, 256, size=n, dtype=np.uint8)
        coef = orc.dwt_fwd(x, w, L, orc.MODE_FULL)
        back, bad = orc.dwt_inv(coef, n, w, L, orc.MODE_FULL)
        assert bad == 0 and np.array_equal(back, x)


def test_full_mode_bounds_fit_widths(orc):
    """C23: FULL widths (B fields 11 bits) hold the whole-matrix bounds."""
    W = weights(orc, (64, 64), 3)
    lin = np.abs(W).sum(axis=(2, 3)) * 128
    assert lin.max() < 1024
    W2 = weights(orc, (32, 32), 2)
    lin2 = np.abs(W2).sum(axis=(2, 3)) * 128
    assert lin2[:8, :8].max() <= 511                        # LL2: 10 bits
    assert 512 < lin2[:8, 8:16].max() <= 520                # HL2 exceeds 10 bits
    assert 512 < lin2[8:16, 8:16].max() <= 800              # HH2
