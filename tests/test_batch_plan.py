"""fragment_batch_plan (host side of the batch entry points): CTA assignment,
validation, and the per-file derived constants, checked without a GPU."""
from __future__ import annotations

import ctypes as C
import hashlib
import struct

import pytest

import synth
import paper_1803_04880_b200 as se


@pytest.fixture(scope="module")
def lib():
    se.build()
    return se.lib()


def make_jobs(sizes, widths, ivs, offsets=None):
    jobs = (se.Job * len(sizes))()
    for i, (n, w, iv) in enumerate(zip(sizes, widths, ivs)):
        j = jobs[i]
        j.in_, j.out, j.a, j.b, j.c = 0x1000, 0x2000, 0x3000, 0x4000, 0x5000
        j.n_bytes, j.width = n, w
        j.block_offset = offsets[i] if offsets else 0
        j.iv[:] = list(iv)
    return jobs


def test_job_struct_layout():
    assert C.sizeof(se.Job) == 616
    assert se.Job.cta_begin.offset == 80 and se.Job.derived.offset == 88


def test_plan_assigns_ctas(lib, orc):
    sizes = [1, 64 * 1024, 0, 5 * 1024 * 1024 + 3, 777]
    widths = [synth.width_rule(n) for n in sizes]
    ivs = [synth.iv_for(5, i) for i in range(len(sizes))]
    jobs = make_jobs(sizes, widths, ivs)
    total = lib.fragment_batch_plan(jobs, len(sizes), 2, synth.KEY)
    expect, acc = [], 0
    for n, w in zip(sizes, widths):
        expect.append(acc)
        acc += -(-orc.layout(n, w, 2)["n_blocks"] // 128)
    assert total == acc
    assert [j.cta_begin for j in jobs] == expect
    # derived: counter base = IV (block_offset 0), K||IV words for the hash framing (C13, C15)
    d = list(jobs[3].derived)
    assert struct.pack(">4I", *d[0:4]) == ivs[3]
    assert struct.pack(">8I", *d[4:12]) == synth.KEY + ivs[3]


def test_plan_midstate_is_sha256_of_prefix(lib):
    """The SHA-256 midstate equals the state after compressing K||IV, checked
    by completing the hash on the host with a pure-Python finish (rounds 8..63
    of FIPS 180-4 over a message whose first 32 bytes are K||IV)."""
    jobs = make_jobs([4096], [64], [bytes(range(16, 32))])
    assert lib.fragment_batch_plan(jobs, 1, 2, synth.KEY) == 1
    mid = list(jobs[0].derived)[12:20]
    # FIPS 180-4 constants from the oracle-independent definition (cube roots), computed here
    def frac_root(p, k, bits):
        lo, hi = 0, 1 << (bits + 10)
        n = p << (bits * k)
        while lo < hi:
            m = (lo + hi + 1) // 2
            if m ** k <= n:
                lo = m
            else:
                hi = m - 1
        return lo & ((1 << bits) - 1)
    primes = [p for p in range(2, 400) if all(p % q for q in range(2, int(p ** 0.5) + 1))][:64]
    K = [frac_root(p, 3, 32) for p in primes]
    H0 = [frac_root(p, 2, 32) for p in primes[:8]]
    msg = synth.KEY + bytes(range(16, 32)) + b"tail of message!"   # 48 bytes -> one block
    block = msg + b"\x80" + bytes(55 - len(msg)) + (len(msg) * 8).to_bytes(8, "big")
    W = list(struct.unpack(">16I", block))
    for t in range(16, 64):
        r = lambda x, n: ((x >> n) | (x << (32 - n))) & 0xFFFFFFFF
        s0 = r(W[t - 15], 7) ^ r(W[t - 15], 18) ^ (W[t - 15] >> 3)
        s1 = r(W[t - 2], 17) ^ r(W[t - 2], 19) ^ (W[t - 2] >> 10)
        W.append((W[t - 16] + s0 + W[t - 7] + s1) & 0xFFFFFFFF)
    a, b, c, d_, e, f, g, h = mid
    for t in range(8, 64):
        r = lambda x, n: ((x >> n) | (x << (32 - n))) & 0xFFFFFFFF
        S1 = r(e, 6) ^ r(e, 11) ^ r(e, 25)
        ch = (e & f) ^ (~e & g)
        t1 = (h + S1 + ch + K[t] + W[t]) & 0xFFFFFFFF
        S0 = r(a, 2) ^ r(a, 13) ^ r(a, 22)
        mj = (a & b) ^ (a & c) ^ (b & c)
        h, g, f, e, d_, c, b, a = g, f, e, (d_ + t1) & 0xFFFFFFFF, c, b, a, (t1 + S0 + mj) & 0xFFFFFFFF
    digest = struct.pack(">8I", *[(x + y) & 0xFFFFFFFF for x, y in zip(H0, [a, b, c, d_, e, f, g, h])])
    assert digest == hashlib.sha256(msg).digest()


def test_plan_rejects_bad_jobs(lib):
    ivs = [bytes(16)]
    assert lib.fragment_batch_plan(make_jobs([100], [12], ivs), 1, 2, synth.KEY) == se.SE_EINVAL   # width % 8
    assert lib.fragment_batch_plan(make_jobs([100], [8], ivs, [3]), 1, 2, synth.KEY) == se.SE_EINVAL  # CTR align
    assert lib.fragment_batch_plan(make_jobs([100], [8], ivs), 1, 4, synth.KEY) == se.SE_EINVAL   # levels
    jobs = make_jobs([100], [8], ivs)
    jobs[0].a = 0
    assert lib.fragment_batch_plan(jobs, 1, 2, synth.KEY) == se.SE_EINVAL                         # null stream
    assert lib.fragment_batch_plan(make_jobs([100], [8], ivs, [16]), 1, 2, synth.KEY) == 1       # 16*40 % 128 == 0
