"""Pins of the Chapter 4 DCT selective-encryption oracle (NEXT row f3,
oracle/dct.c) against things other than itself: the matrix the paper prints
(Eq. 4.6), scipy's orthonormal DCT-II (a library routine the definition
reduces to), the closed forms of Eq. 4.4 and Parseval, the value ranges the
paper states, the storage figure, the paper's worked block
(P:1525-1550), the PSNR the paper reports (Table 4.2), the multi-round
behaviour, and independent re-derivations of the fragments with
`cryptography` (AES-CTR) and hashlib (SHA-512)."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest
import scipy.fft

import synth
from conftest import golden_matrix
from dct_helpers import SEL, blocks, psnr, records, unblocks

KEY = synth.KEY
IV = synth.iv_for(6)


def aes_ctr(key, iv, ctr_offset, data):
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    ctr = (int.from_bytes(iv, "big") + ctr_offset) % (1 << 128)
    enc = Cipher(algorithms.AES(key), modes.CTR(ctr.to_bytes(16, "big"))).encryptor()
    return np.frombuffer(enc.update(bytes(data)) + enc.finalize(), np.uint8)


# ---------------------------------------------------------------- the transform


def test_basis_equals_printed_matrix(orc):
    """Eq. 4.6 as printed (5 decimals) == alpha(u) cos(pi(2x+1)u/16) at [x][u] (D2)."""
    assert np.allclose(orc.dct_basis(), golden_matrix("paper_eq4_6_dct_matrix.txt"), atol=6e-6)


@pytest.mark.parametrize("seed", range(4))
def test_dct8_equals_scipy_orthonormal_dct2(orc, seed):
    """Eq. 4.1/4.2 == the orthonormal DCT-II / DCT-III, axis 0 = x = row (D1)."""
    f = np.random.default_rng(seed).integers(-128, 128, (8, 8)).astype(float)
    c = orc.dct8_fwd(f)
    assert np.allclose(c, scipy.fft.dctn(f, type=2, norm="ortho"), atol=1e-9)
    assert np.allclose(orc.dct8_inv(c), scipy.fft.idctn(c, type=2, norm="ortho"), atol=1e-9)
    assert np.allclose(orc.dct8_inv(c), f, atol=1e-9)                         # exact inverse
    assert np.isclose((f ** 2).sum(), (c ** 2).sum())                          # Parseval


@pytest.mark.parametrize("W,H,C", [(16, 8, 1), (24, 16, 3)])
def test_image_transform_equals_scipy(orc, W, H, C):
    """The whole-image DCT (Table 4.1's operation) = scipy per block of
    (x - 128), coefficients in pixel layout; the inverse rebuilds x exactly."""
    img = synth.bitmap(H, W, C, 31).reshape(-1)
    got = orc.dct_image_fwd(img, W, H, C)
    blk = blocks(img, W, H, C).astype(float) - 128
    ref = unblocks(scipy.fft.dctn(blk, type=2, norm="ortho", axes=(1, 2)), W, H, C)
    assert np.allclose(got, ref, atol=1e-9)
    assert np.array_equal(orc.dct_image_inv(got, W, H, C), img)


def test_dc_is_eight_times_the_mean(orc):
    """Eq. 4.4: C(0,0) = alpha(0)^2 sum f = 8 * mean; all AC of a flat block vanish."""
    f = np.full((8, 8), 37.0)
    c = orc.dct8_fwd(f)
    assert np.isclose(c[0, 0], 8 * 37.0) and np.allclose(c.flat[1:], 0, atol=1e-9)
    # an asymmetric basis image (u, v) = (1, 2) has a single coefficient: catches transposes
    m = orc.dct_basis()
    b = np.outer(m[:, 1], m[:, 2])
    c = orc.dct8_fwd(b)
    assert np.isclose(c[1, 2], 1.0) and np.isclose(np.abs(c).sum(), 1.0)


def test_coefficient_ranges_stated_by_the_paper(orc):
    """centered DC in [-1024, 1024], every AC within [-1023, 1023]."""
    m = orc.dct_basis()
    for u in range(8):
        for v in range(8):
            w = np.outer(m[:, u], m[:, v])
            hi = 127 * w[w > 0].sum() - 128 * w[w < 0].sum()
            lo = -128 * w[w > 0].sum() + 127 * w[w < 0].sum()
            if (u, v) == (0, 0):
                assert np.isclose(lo, -1024) and np.isclose(hi, 1016)
            else:
                assert max(hi, -lo) <= 1023


# ---------------------------------------------------------------- the fragments


def test_layout_storage(orc):
    """66 extra bits per 8x8 block = 12.9 % of 512 bits."""
    lay = orc.dct_layout(4800, 4800, 1)
    assert lay["bits"] == 66 and lay["records"] == 600 * 600
    assert lay["a_bytes"] == 600 * 600 * 66 // 8 and lay["p_bytes"] == 4800 * 4800
    assert round(100 * 66 / 512, 1) == 12.9
    for bad in [(0, 8, 1), (12, 8, 1), (8, 12, 1), (8, 8, 2)]:
        with pytest.raises(ValueError):
            orc.dct_layout(*bad)


@pytest.mark.parametrize("W,H,C", [(64, 48, 1), (32, 16, 3), (16, 16, 4)])
@pytest.mark.parametrize("level", [1, 2])
def test_fragments_rederived_independently(orc, W, H, C, level):
    """Fragment 1 = AES-CTR(rint of the scipy coefficients, 11-bit store);
    Fragment 2 = clamp(rint(iDCT with DC 1024 and 5 AC 0)) [^ SHA-512(rec9)]."""
    img = synth.bitmap(H, W, C, W + H + C).reshape(-1)
    a, p, pr = orc.dct_protect(img, W, H, C, level, KEY, IV, real=True)
    blk = blocks(img, W, H, C).astype(float) - 128
    n = blk.shape[0]
    coef = scipy.fft.dctn(blk, type=2, norm="ortho", axes=(1, 2))
    sel = np.stack([coef[:, u, v] for u, v in SEL], 1)
    sel[:, 0] = blk.sum((1, 2)) / 8                                           # Eq. 4.4
    assert np.allclose(orc.dct_select(img, W, H, C), sel, atol=1e-9)
    plain = aes_ctr(KEY, IV, 0, a)
    q = records(plain, n)
    assert np.array_equal(q, np.clip(np.rint(sel), -1023, 1023).astype(int))
    pad = coef.copy()
    for u, v in SEL[1:]:
        pad[:, u, v] = 0
    pad[:, 0, 0] = 1024
    g = scipy.fft.idctn(pad, type=2, norm="ortho", axes=(1, 2)).reshape(n, 64)
    assert np.allclose(pr, g, atol=1e-9)
    pb = np.clip(np.rint(g), 0, 255).astype(np.uint8)
    if level == 2:
        bits = np.unpackbits(plain)[: 66 * n].reshape(n, 66)
        rec9 = np.packbits(np.concatenate([bits, np.zeros((n, 6), np.uint8)], 1), axis=1)
        dig = np.stack([np.frombuffer(hashlib.sha512(bytes(r)).digest(), np.uint8) for r in rec9])
        pb ^= dig
    assert np.array_equal(unblocks(pb, W, H, C), p)


def test_keyed_level2_framing(orc):
    """Flag KEYED: message K || IV || be64(block_offset + r) || rec9 (D9)."""
    W, H = 16, 8
    img = synth.bitmap(H, W, 1, 3).reshape(-1)
    off = 64 * 5
    a1, p1 = orc.dct_protect(img, W, H, 1, 1, KEY, IV, block_offset=off)
    a2, p2 = orc.dct_protect(img, W, H, 1, 2, KEY, IV, flags=orc.DCT_KEYED, block_offset=off)
    assert np.array_equal(a1, a2)
    plain = aes_ctr(KEY, IV, off * 66 // 128, a1)
    bits = np.unpackbits(plain)[:132].reshape(2, 66)
    for r in range(2):
        rec9 = np.packbits(np.concatenate([bits[r], np.zeros(6, np.uint8)]))
        d = np.frombuffer(hashlib.sha512(KEY + IV + (off + r).to_bytes(8, "big") + bytes(rec9)).digest(), np.uint8)
        got = blocks(p1 ^ p2, W, H, 1)[r].reshape(-1)
        assert np.array_equal(got, d)
    with pytest.raises(ValueError):                   # CTR offset must be whole AES blocks (D8)
        orc.dct_protect(img, W, H, 1, 1, KEY, IV, block_offset=3)


def test_eleven_bit_store_saturation(orc):
    """All-zero block: DC = -1024 stored as -1023 (D5); recovery still exact."""
    img = np.zeros(64, np.uint8)
    a, p = orc.dct_protect(img, 8, 8, 1, 1, KEY, IV)
    assert records(aes_ctr(KEY, IV, 0, a), 1).tolist() == [[-1023, 0, 0, 0, 0, 0]]
    assert np.all(p == 128)                                                   # mean 128
    assert np.array_equal(orc.dct_recover(a, p, 8, 8, 1, 1, KEY, IV), img)
    img = np.full(64, 255, np.uint8)
    a, p = orc.dct_protect(img, 8, 8, 1, 2, KEY, IV)
    assert records(aes_ctr(KEY, IV, 0, a), 1).tolist() == [[1016, 0, 0, 0, 0, 0]]
    assert np.array_equal(orc.dct_recover(a, p, 8, 8, 1, 2, KEY, IV), img)


# ---------------------------------------------------------------- recovery


@pytest.mark.parametrize("level", [1, 2])
def test_recover_rederived_independently(orc, level):
    """out = clamp(rint(iDCT(DCT(P) with the 6 stored values) + 128)) via scipy."""
    W, H, C = 32, 24, 3
    img = synth.bitmap(H, W, C, 9).reshape(-1)
    a, p = orc.dct_protect(img, W, H, C, level, KEY, IV)
    out, orl = orc.dct_recover(a, p, W, H, C, level, KEY, IV, real=True)
    n = W * H * C // 64
    q = records(aes_ctr(KEY, IV, 0, a), n)
    a1, p1 = orc.dct_protect(img, W, H, C, 1, KEY, IV)
    pb = blocks(p1, W, H, C).astype(float)                                    # unmasked Fragment 2
    c = scipy.fft.dctn(pb, type=2, norm="ortho", axes=(1, 2))
    for k, (u, v) in enumerate(SEL):
        c[:, u, v] = q[:, k]
    g = scipy.fft.idctn(c, type=2, norm="ortho", axes=(1, 2)).reshape(n, 64) + 128
    assert np.allclose(orl, g, atol=1e-9)
    assert np.array_equal(out, unblocks(np.clip(np.rint(g), 0, 255).astype(np.uint8), W, H, C))


def test_paper_worked_block(orc):
    """the rebuilt block differs from the original in a few pixels,
    each by exactly 1 (the paper shows 3; positions depend on its float pipeline)."""
    x = golden_matrix("paper_dct_block_example.txt").astype(np.uint8).reshape(-1)
    for level in (1, 2):
        a, p = orc.dct_protect(x, 8, 8, 1, level, KEY, IV)
        y = orc.dct_recover(a, p, 8, 8, 1, level, KEY, IV)
        d = np.abs(y.astype(int) - x)
        assert d.max() == 1 and 1 <= (d > 0).sum() <= 8


@pytest.mark.parametrize("H,W,C", [(256, 256, 1), (96, 128, 3)])
def test_psnr_and_changed_pixels(orc, H, W, C):
    """Table 4.2: PSNR after protect + recover ~ 62.8 dB on photos; the
    synthetic proxy (noise sigma 2 in every block, no flat areas) gives
    ~60.3 dB: the two roundings the paper names each leave <= 0.5.
    Pixels change by at most 1 and < 10 % of them change (paper: ~3 %)."""
    x = synth.bitmap(H, W, C, 7).reshape(-1)
    for level in (1, 2):
        a, p = orc.dct_protect(x, W, H, C, level, KEY, IV)
        y = orc.dct_recover(a, p, W, H, C, level, KEY, IV)
        assert psnr(x, y) > 59.5
        assert np.abs(y.astype(int) - x).max() == 1 and np.mean(x != y) < 0.10


def test_repeated_rounds_converge(orc):
    """P:1563, Figs 4.12-4.14: over 15 protect/rebuild rounds PSNR and the share
    of changed pixels stop changing after a few rounds (paper: final PSNR
    60.7-61.8 dB, < 5 % changed, on photos)."""
    H = W = 64
    x = synth.bitmap(H, W, 1, 21).reshape(-1)
    z, hist = x.copy(), []
    for _ in range(15):
        a, p = orc.dct_protect(z, W, H, 1, 1, KEY, IV)
        z = orc.dct_recover(a, p, W, H, 1, 1, KEY, IV)
        hist.append((psnr(x, z), np.mean(x != z)))
    assert hist[-1] == hist[-2] == hist[-3]                      # fixed point reached
    assert hist[-1][0] > 57.0 and hist[-1][0] <= hist[0][0]


def test_level2_public_fragment_statistics(orc):
    """P:1643, Fig. 4.15: the level-2 public fragment's PDF is close to uniform
    and differs from the original's; level 1 leaves it image-like."""
    H, W = 256, 256
    x = synth.bitmap(H, W, 1, 5).reshape(-1)
    _, p2 = orc.dct_protect(x, W, H, 1, 2, KEY, IV)
    _, p1 = orc.dct_protect(x, W, H, 1, 1, KEY, IV)

    def entropy(v):
        h = np.bincount(v, minlength=256) / v.size
        h = h[h > 0]
        return float(-(h * np.log2(h)).sum())
    assert entropy(p2) > 7.99 and entropy(p1) < 7.0
