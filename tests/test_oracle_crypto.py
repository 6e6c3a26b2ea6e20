"""Pins for the oracle's AES-128 / CTR / SHA-2 (rows a6-a8 primitives).

Pinned to: FIPS-197 App. B and C.1 vectors, SP 800-38A F.5.1, FIPS 180-4
example digests (tests/golden/), the FIPS-197 §5.1.1 S-box worked example,
and randomised equivalence with two third-party implementations (hashlib /
OpenSSL via ``cryptography``).
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_lines

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def test_aes128_fips197_vectors(orc):
    for ln in golden_lines("fips197_aes128.txt"):
        k, p, c = (bytes.fromhex(t) for t in ln.split())
        assert orc.aes128_encrypt_block(k, p) == c


def test_aes_sbox_definition_examples(orc):
    s = orc.aes128_sbox()
    # FIPS-197 §5.1.1: "if s1,1 = {53}, then ... s'1,1 = {ed}"
    assert s[0x53] == 0xED
    assert s[0x00] == 0x63           # inverse of 0 is 0, affine constant 0x63
    assert sorted(s.tolist()) == list(range(256))   # a permutation
    assert not np.any(s == np.arange(256))          # no fixed points (AES design property)


def test_ctr_sp800_38a(orc):
    lines = golden_lines("sp800_38a_ctr.txt")
    key = bytes.fromhex(lines[0].split()[1])
    ctr = bytes.fromhex(lines[1].split()[1])
    pt = b"".join(bytes.fromhex(ln.split()[0]) for ln in lines[2:])
    ct = b"".join(bytes.fromhex(ln.split()[1]) for ln in lines[2:])
    assert orc.aes128_ctr(key, ctr, pt).tobytes() == ct
    # ctr_offset: starting at block 2 reproduces the tail of the stream
    assert orc.aes128_ctr(key, ctr, pt[32:], ctr_offset=2).tobytes() == ct[32:]


def test_ctr_random_vs_openssl(orc):
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    rng = np.random.default_rng(11)
    for trial in range(20):
        key = rng.bytes(16)
        iv = rng.bytes(16)
        if trial % 8 == 0:     # carry out of the low 64 bits of the counter
            iv = bytes(8) + b"\xff" * 8
        elif trial % 8 == 4:   # wrap of the whole 128-bit counter
            iv = b"\xff" * 16
        n = int(rng.integers(0, 300))
        data = rng.bytes(n)
        enc = Cipher(algorithms.AES(key), modes.CTR(iv)).encryptor()
        assert orc.aes128_ctr(key, iv, data).tobytes() == enc.update(data) + enc.finalize()


@pytest.mark.parametrize("offset", [3, (1 << 64) - 2, (1 << 64) - 1])
def test_ctr_offset_is_128_bit(orc, offset):
    """SP 800-38A: counter = IV + j mod 2^128, also when IV + offset + j crosses 2^64."""
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    key = bytes(range(16))
    iv = bytes.fromhex("f0f1f2f3f4f5f6f7f8f9fafbfcfdfeff")
    start = ((int.from_bytes(iv, "big") + offset) % (1 << 128)).to_bytes(16, "big")
    data = bytes(range(200))
    enc = Cipher(algorithms.AES(key), modes.CTR(start)).encryptor()
    assert orc.aes128_ctr(key, iv, data, ctr_offset=offset).tobytes() == enc.update(data)


def test_sha_fips180_vectors(orc):
    for ln in golden_lines("fips180_4_sha.txt"):
        alg, msg, dig = ln.split()
        f = orc.sha256 if alg == "sha256" else orc.sha512
        assert f(msg.encode()).hex() == dig


@pytest.mark.parametrize("alg", ["sha256", "sha512"])
def test_sha_random_lengths_vs_hashlib(orc, alg):
    rng = np.random.default_rng(12)
    f = getattr(orc, alg)
    # every length across the one/two-block padding boundaries, then random
    lengths = list(range(0, 260)) + [int(x) for x in rng.integers(0, 2000, size=40)]
    for n in lengths:
        m = rng.bytes(n)
        assert f(m) == getattr(hashlib, alg)(m).digest(), n
