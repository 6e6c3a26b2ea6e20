"""Pins for the oracle's split / pack / protect / recover (rows a1, a5-a10).

Pinned to:
  * the paper's storage accounting (tests/golden/paper_storage.txt: 40/124/480
    bits, 644 total, 164 local, 7.8/24.2/93.8 %, k = 4);
  * a second, test-side implementation of readings C9-C17 built from numpy
    bit arrays, hashlib (SHA-2) and OpenSSL (AES-CTR via ``cryptography``),
    fed with the oracle's DWT coefficients (the DWT is pinned separately in
    test_oracle_dwt.py);
  * losslessness, error confinement and key
    sensitivity (Table 5.1 "KS" ~50%).
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import synth
from conftest import golden_lines

KEY = synth.KEY
IV = bytes.fromhex("f0f1f2f3f4f5f6f7f8f9fafbfcfdfe00")


# ---------------------------------------------------------------- layout

def test_storage_accounting_matches_paper(orc):
    g = {ln.split()[0]: float(ln.split()[1]) for ln in golden_lines("paper_storage.txt")}
    lay = orc.layout(64, 8, 2)
    assert lay["a_bits"] == g["a_bits"] and lay["b_bits"] == g["b_bits"] and lay["c_bits"] == g["c_bits"]
    assert lay["a_bits"] + lay["b_bits"] + lay["c_bits"] == g["total_bits"]
    assert lay["a_bits"] + lay["b_bits"] == g["local_bits"]
    for k, s in (("a", "a_percent"), ("b", "b_percent"), ("c", "c_percent")):
        assert round(100 * lay[k + "_bits"] / 512, 1) == g[s]
    assert len(orc.record_fields(2, 0, 0)) == g["k"]


def expected_fields(L, mode):
    """Readings C10, C21-C23 written independently of the oracle."""
    def band(level, b, w):
        s = 8 >> level
        return [(level, b, i, j, w) for i in range(s) for j in range(s)]
    A = band(L, 0, 10)
    B = []
    for lev in range(L, 1, -1):
        wd = 11 if mode == 1 else 10
        B += band(lev, 1, wd) + band(lev, 2, wd) + band(lev, 3, 11)
    C = band(1, 1, 10) + band(1, 2, 10) + band(1, 3, 10)
    return [A, B, C]


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_record_fields(orc, L, mode):
    exp = expected_fields(L, mode)
    for s in range(3):
        assert orc.record_fields(L, mode, s) == exp[s]
    bits = [sum(f[4] for f in e) for e in exp]
    want = {(1, 0): [160, 0, 480], (2, 0): [40, 124, 480], (3, 0): [10, 155, 480],
            (1, 1): [160, 0, 480], (2, 1): [40, 132, 480], (3, 1): [10, 165, 480]}
    assert bits == want[(L, mode)]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_layouts(orc, cfg):
    c = synth.CONFIGS[cfg]
    lay = orc.layout(c["n_bytes"], c["width"], c["levels"])
    table = {1: (1024, 20480, 0, 61440), 2: (196608, 983040, 3047424, 11796480),
             3: (1048576, 1310720, 20316160, 62914560), 4: (16777216, 80 << 20, 248 << 20, 960 << 20)}
    assert (lay["n_blocks"], lay["a_bytes"], lay["b_bytes"], lay["c_bytes"]) == table[cfg]


# ---------------------------------------------------------------- test-side re-derivation

def coef_of(coef, mode, R, W, br, bc, f):
    level, b, i, j, _ = f
    if mode == 0:
        s = 8 >> level
        ro = s if b in (2, 3) else 0
        co = s if b in (1, 3) else 0
        return int(coef[8 * br + ro + i, 8 * bc + co + j])
    ro = (R >> level) if b in (2, 3) else 0
    co = (W >> level) if b in (1, 3) else 0
    return int(coef[ro + ((8 * br) >> level) + i, co + ((8 * bc) >> level) + j])


def bits_of(v, w):
    return [(v >> (w - 1 - k)) & 1 for k in range(w)]


def reference_protect(orc, data, W, L, key, iv, mode=0, flags=0, block_offset=0):
    """Independent implementation of C9-C17 (numpy bits + hashlib + OpenSSL)."""
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    coef = orc.dwt_fwd(data, W, L, mode)
    R = coef.shape[0]
    fl = expected_fields(L, mode)
    streams = [[], [], []]
    for blk in range((R // 8) * (W // 8)):
        br, bc = divmod(blk, W // 8)
        rec = []
        for s in range(3):
            bits = []
            for f in fl[s]:
                bits += bits_of(coef_of(coef, mode, R, W, br, bc, f) + (1 << (f[4] - 1)), f[4])
            rec.append(np.array(bits, dtype=np.uint8))
        if not flags & 1:
            gb = (block_offset + blk).to_bytes(8, "big")
            def packed(b):
                return np.packbits(b).tobytes()
            if len(rec[1]):
                dB = np.unpackbits(np.frombuffer(hashlib.sha256(key + iv + gb + packed(rec[0])).digest(), np.uint8))
                rec[1] = rec[1] ^ dB[: len(rec[1])]
                src = rec[1]
            else:
                src = rec[0]
            dC = np.unpackbits(np.frombuffer(hashlib.sha512(key + iv + gb + packed(src)).digest(), np.uint8))
            rec[2] = rec[2] ^ dC[: len(rec[2])]
        for s in range(3):
            streams[s].append(rec[s])
    out = [np.packbits(np.concatenate(s)) if len(s) and sum(map(len, s)) else np.zeros(0, np.uint8)
           for s in streams]
    a_plain = out[0].tobytes()
    abits = sum(f[4] for f in fl[0])
    start = block_offset * abits // 8
    ctr = int.from_bytes(iv, "big") + start // 16
    enc = Cipher(algorithms.AES(key), modes.CTR((ctr % (1 << 128)).to_bytes(16, "big"))).encryptor()
    ks = enc.update(bytes(start % 16 + len(a_plain)))[start % 16:]
    out[0] = np.frombuffer(bytes(x ^ y for x, y in zip(a_plain, ks)), np.uint8)
    return out


@pytest.mark.parametrize("L,mode,n,W", [(1, 0, 256 * 24, 256), (2, 0, 40 * 33 + 5, 40), (3, 0, 64 * 17, 64),
                                        (2, 1, 64 * 16, 64), (3, 1, 32 * 24, 32), (1, 1, 16 * 16, 16)])
def test_protect_matches_independent_derivation(orc, L, mode, n, W):
    rng = np.random.default_rng(L * 10 + mode)
    data = rng.integers(0, 256, size=n, dtype=np.uint8)
    for flags in (0, 1):
        got = orc.protect(data, W, L, KEY, IV, mode=mode, flags=flags, block_offset=256)
        exp = reference_protect(orc, data, W, L, KEY, IV, mode=mode, flags=flags, block_offset=256)
        for s in range(3):
            assert np.array_equal(got[s], exp[s]), ("stream", s, "flags", flags)


# ---------------------------------------------------------------- invariants

CASES = [(0, 8, 2), (1, 8, 2), (63, 8, 1), (64, 8, 3), (65, 8, 2), (511, 16, 2), (1000, 24, 3),
         (4096, 64, 1), (5000, 128, 2), (64 * 64 * 3 + 17, 192, 3)]


@pytest.mark.parametrize("n,W,L", CASES)
@pytest.mark.parametrize("mode", [0, 1])
def test_round_trip(orc, n, W, L, mode):
    rng = np.random.default_rng(n + W + L)
    data = rng.integers(0, 256, size=n, dtype=np.uint8)
    for flags in (0, 1):
        a, b, c = orc.protect(data, W, L, KEY, IV, mode=mode, flags=flags, block_offset=7 * 128)
        back, rep = orc.recover(a, b, c, n, W, L, KEY, IV, mode=mode, flags=flags, block_offset=7 * 128)
        assert np.array_equal(back, data)
        assert rep == (-1, 0)


def test_extreme_inputs_round_trip(orc):
    for data in (np.zeros(4096, np.uint8), np.full(4096, 255, np.uint8),
                 (np.indices((64, 64)).sum(0) % 2 * 255).astype(np.uint8).reshape(-1)):
        for L in (1, 2, 3):
            a, b, c = orc.protect(data, 64, L, KEY, IV)
            back, rep = orc.recover(a, b, c, data.size, 64, L, KEY, IV)
            assert np.array_equal(back, data) and rep == (-1, 0)


def test_ranges_compose(orc):
    """Processing block ranges separately reproduces the whole-file streams."""
    data = synth.random_bytes(64 * 1024, 9)
    W, L = 64, 2
    whole = orc.protect(data, W, L, KEY, IV)
    lay = orc.layout(data.size, W, L)
    bufs = [np.zeros(lay[k], np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes")]
    cuts = [0, 128, 384, 512, lay["n_blocks"]]
    for b0, b1 in zip(cuts[:-1], cuts[1:]):
        orc.protect(data, W, L, KEY, IV, block_range=(b0, b1), out=bufs)
    for s in range(3):
        assert np.array_equal(bufs[s], whole[s])


def test_stripe_shards_equal_slices(orc):
    """A row stripe processed as its own input with block_offset equals the
    corresponding slice of the whole-file streams (the multi-GPU invariant, §8.6)."""
    W, L = 1024, 2
    data = synth.random_bytes(W * 8 * 4, 10)           # 4 block-rows of 128 blocks
    whole = orc.protect(data, W, L, KEY, IV)
    per_row = [5 * 128, 124 * 128 // 8, 60 * 128]
    for r0, r1 in [(0, 1), (1, 3), (3, 4)]:
        part = data[r0 * 8 * W: r1 * 8 * W]
        got = orc.protect(part, W, L, KEY, IV, block_offset=r0 * 128)
        for s in range(3):
            assert np.array_equal(got[s], whole[s][r0 * per_row[s]: r1 * per_row[s]])


def test_error_confinement(orc):
    """a bit error in the 2nd public fragment gives exactly a 1-bit error
    in that fragment after unmasking and stays inside its 8x8 block."""
    W, L = 64, 2
    data = synth.bitmap(64, 64, 1, 3).reshape(-1)
    a, b, c = orc.protect(data, W, L, KEY, IV)
    rng = np.random.default_rng(5)
    for _ in range(20):
        blk = int(rng.integers(0, 64))
        bit = blk * 480 + int(rng.integers(0, 480))
        c2 = c.copy()
        c2[bit // 8] ^= 0x80 >> (bit % 8)
        back, rep = orc.recover(a, b, c2, data.size, W, L, KEY, IV)
        diff = np.nonzero(back != data)[0]
        br, bc = blk // 8, blk % 8
        assert all((i // W) // 8 == br and (i % W) // 8 == bc for i in diff)
        # unmasked C differs in exactly one bit: compare with PUBLIC_PLAIN run
        p_a, p_b, p_c = orc.protect(back, W, L, KEY, IV, flags=1) if rep[1] == 0 else (None,) * 3
        if p_c is not None:
            q_a, q_b, q_c = orc.protect(data, W, L, KEY, IV, flags=1)
            x = np.unpackbits(p_c) ^ np.unpackbits(q_c)
            assert x.sum() == 1
    # a flipped bit in B' or A' also stays inside its block
    for stream in ("a", "b"):
        blk = 37
        a2, b2 = a.copy(), b.copy()
        if stream == "a":
            a2[(blk * 40 + 3) // 8] ^= 0x80 >> ((blk * 40 + 3) % 8)
        else:
            b2[(blk * 124 + 5) // 8] ^= 0x80 >> ((blk * 124 + 5) % 8)
        back, _ = orc.recover(a2, b2, c, data.size, W, L, KEY, IV)
        diff = np.nonzero(back != data)[0]
        assert len(diff) > 0
        assert all((i // W) // 8 == blk // 8 and (i % W) // 8 == blk % 8 for i in diff)


def test_wrong_key_flags_corruption(orc):
    data = synth.bitmap(64, 128, 1, 4).reshape(-1)
    a, b, c = orc.protect(data, 128, 2, KEY, IV)
    bad_key = bytes([KEY[0] ^ 1]) + KEY[1:]
    back, rep = orc.recover(a, b, c, data.size, 128, 2, bad_key, IV)
    assert rep[0] >= 0 and rep[1] > 32       # most of the 128 blocks out of [0,255]


def test_key_sensitivity_about_half(orc):
    """P:2592 / Table 5.1 'KS': one key bit flipped changes ~50% of the public bits."""
    data = synth.bitmap(128, 128, 1, 6).reshape(-1)
    _, b1, c1 = orc.protect(data, 128, 2, KEY, IV)
    k2 = KEY[:5] + bytes([KEY[5] ^ 0x10]) + KEY[6:]
    _, b2, c2 = orc.protect(data, 128, 2, k2, IV)
    for x, y in ((b1, b2), (c1, c2)):
        frac = (np.unpackbits(x) != np.unpackbits(y)).mean()
        assert 0.47 < frac < 0.53, frac


def test_identical_blocks_get_distinct_masks(orc):
    """C16 / P:2576 nonce: identical blocks do not give identical public fragments."""
    data = np.full(64 * 16, 99, dtype=np.uint8)
    _, b, c = orc.protect(data, 64, 2, KEY, IV)
    recs = {c[i * 60:(i + 1) * 60].tobytes() for i in range(16)}
    assert len(recs) == 16
