"""Host-resident streaming entry points (row f1): fragment_protect_host /
fragment_recover_host cut the input into block-row chunks and pipeline
H2D -> fused kernel -> D2H on several streams.  Outputs must be byte-identical
to the oracle for any chunking, and the merged corruption report must equal
the whole-file report."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = bytes.fromhex("0102030405060708090a0b0c0d0e0f10")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def host(x):
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("chunk,streams", [(0, 0), (64 * 1024, 3), (200 * 1024, 1), (8 * 1024, 4)])
def test_host_streaming_parity(dev, orc, L, chunk, streams):
    n, W = 1024 * 8 * 37 + 1234, 1024
    x = synth.random_bytes(n, 17 + L)
    a, b, c = se.fragment_protect_host(host(x), W, L, KEY, IV, chunk_bytes=chunk, n_streams=streams)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV)
    assert np.array_equal(a.numpy(), oa) and np.array_equal(b.numpy(), ob) and np.array_equal(c.numpy(), oc)
    back, rep = se.fragment_recover_host(a, b, c, n, W, L, KEY, IV, chunk_bytes=chunk, n_streams=streams)
    assert np.array_equal(back.numpy(), x) and rep == (-1, 0)


def test_host_streaming_report_across_chunks(dev, orc):
    n, W, L = 512 * 8 * 40, 512, 2
    x = synth.bitmap(8 * 40, 512 // 3 + 1, 3, 8).reshape(-1)[:n]
    oa, ob, oc = orc.protect(x, W, L, KEY, IV)
    oc2 = oc.copy()
    for blk in (5, 64 * 17 + 3, 64 * 33):                # three blocks in different chunks
        oc2[blk * 60] ^= 0xFF
    back, rep = se.fragment_recover_host(host(oa), host(ob), host(oc2), n, W, L, KEY, IV, chunk_bytes=64 * 1024)
    oback, orep = orc.recover(oa, ob, oc2, n, W, L, KEY, IV)
    assert np.array_equal(back.numpy(), oback) and rep == orep


def test_host_streaming_full_mode(dev, orc):
    n, W, L = 256 * 136, 256, 2
    x = synth.random_bytes(n, 3)
    a, b, c = se.fragment_protect_host(host(x), W, L, KEY, IV, mode=se.MODE_FULL)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, mode=orc.MODE_FULL)
    assert np.array_equal(a.numpy(), oa) and np.array_equal(b.numpy(), ob) and np.array_equal(c.numpy(), oc)
    back, rep = se.fragment_recover_host(a, b, c, n, W, L, KEY, IV, mode=se.MODE_FULL)
    assert np.array_equal(back.numpy(), x) and rep == (-1, 0)


def test_host_pageable_buffers(dev, orc):
    """Pageable host memory works too (driver-staged copies)."""
    n, W = 300000, 512
    x = synth.random_bytes(n, 5)
    xt = torch.from_numpy(x.copy())
    a, b, c = se.fragment_protect_host(xt, W, 2, KEY, IV, chunk_bytes=32 * 1024)
    oa, ob, oc = orc.protect(x, W, 2, KEY, IV)
    assert np.array_equal(c.numpy(), oc) and np.array_equal(a.numpy(), oa)


def test_graph_replay_reads_new_contents(dev, orc):
    """Repeated calls with the same buffers and arguments replay a cached CUDA
    graph (se_host.cu): new contents of the same host buffers must be read,
    and a different key or chunking must not reuse the graph."""
    n, W, L = 1024 * 8 * 24, 1024, 2
    hx = host(np.zeros(n, np.uint8))
    lay = se.fragment_layout(n, W, L)
    frag = tuple(se._host_empty(lay[k]) for k in ("a_bytes", "b_bytes", "c_bytes"))
    out = se._host_empty(n)
    for i, (key, chunk) in enumerate([(KEY, 64 * 1024), (KEY, 64 * 1024), (KEY, 64 * 1024),
                                      (bytes(16), 64 * 1024), (KEY, 96 * 1024)]):
        x = synth.random_bytes(n, 100 + i)
        hx.copy_(torch.from_numpy(x))
        se.fragment_protect_host(hx, W, L, key, IV, out=frag, chunk_bytes=chunk, n_streams=3)
        oa, ob, oc = orc.protect(x, W, L, key, IV)
        assert np.array_equal(frag[0].numpy(), oa) and np.array_equal(frag[2].numpy(), oc), i
        _, rep = se.fragment_recover_host(*frag, n, W, L, key, IV, out=out, chunk_bytes=chunk, n_streams=3)
        assert np.array_equal(out.numpy(), x) and rep == (-1, 0), i
    # a corrupted replay still reports (the report copies are part of the graph)
    frag[2][60 * 7] ^= 0xFF
    _, rep = se.fragment_recover_host(*frag, n, W, L, KEY, IV, out=out, chunk_bytes=96 * 1024, n_streams=3)
    assert rep == orc.recover(frag[0].numpy(), frag[1].numpy(), frag[2].numpy(), n, W, L, KEY, IV)[1]


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
def test_host_mapped_zero_copy(dev, orc, L, flags):
    """SE_FLAG_HOST_MAPPED: the kernels read and write the page-locked host
    buffers directly (no staging copies): same bytes as the oracle, same report."""
    n, W = 1024 * 8 * 21 + 777, 1024
    x = synth.random_bytes(n, 40 + L)
    fl = flags | se.FLAG_HOST_MAPPED
    a, b, c = se.fragment_protect_host(host(x), W, L, KEY, IV, flags=fl)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, flags=flags)
    assert np.array_equal(a.numpy(), oa) and np.array_equal(b.numpy(), ob) and np.array_equal(c.numpy(), oc)
    back, rep = se.fragment_recover_host(a, b, c, n, W, L, KEY, IV, flags=fl)
    assert np.array_equal(back.numpy(), x) and rep == (-1, 0)
    c2 = c.clone().pin_memory()                                       # mapped mode needs page-locked buffers
    c2[60 * 9 + 4] ^= 0xFF
    back, rep = se.fragment_recover_host(a, b, c2, n, W, L, KEY, IV, flags=fl)
    oback, orep = orc.recover(oa, ob, c2.numpy(), n, W, L, KEY, IV, flags=flags)
    assert np.array_equal(back.numpy(), oback) and rep == orep


def test_host_mapped_needs_pinned(dev):
    x = torch.from_numpy(synth.random_bytes(4096, 1))              # pageable
    with pytest.raises(se.SEError):
        se.fragment_protect_host(x, 64, 2, KEY, IV, flags=se.FLAG_HOST_MAPPED)


@pytest.mark.parametrize("offset", [0, 4])
@pytest.mark.parametrize("W", [1032, 1024])
def test_host_hybrid_staging(dev, orc, W, offset):
    """Protect's hybrid staging (the fused kernel writes the fragments into the
    page-locked host buffers) on chunks of whole 128-block groups — W = 1032
    has 129 blocks per block row, so chunks span 128 block rows — and, with
    the output views 4 bytes into their buffers (not 16-byte aligned), the
    staged fallback: both byte-identical to the oracle."""
    n, L = W * 8 * 300 + 77, 2
    x = synth.random_bytes(n, W + offset)
    lay = se.fragment_layout(n, W, L)
    outs = []
    for key in ("a_bytes", "b_bytes", "c_bytes"):
        buf = torch.empty(lay[key] + 16, dtype=torch.uint8).pin_memory()
        outs.append(buf[offset:offset + lay[key]])
    a, b, c = se.fragment_protect_host(host(x), W, L, KEY, IV, out=tuple(outs), chunk_bytes=256 * 1024,
                                       n_streams=3)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV)
    assert np.array_equal(a.numpy(), oa) and np.array_equal(b.numpy(), ob) and np.array_equal(c.numpy(), oc)
    back, rep = se.fragment_recover_host(a, b, c, n, W, L, KEY, IV, chunk_bytes=256 * 1024, n_streams=3)
    assert np.array_equal(back.numpy(), x) and rep == (-1, 0)


@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
@pytest.mark.parametrize("n,W,L,chunk", [(1024 * 8 * 37 + 1234, 1024, 2, 64 * 1024), (6144 * 2048, 6144, 2, 0),
                                         (4096 * 8 * 300, 4096, 3, 1 << 20)])
def test_host_async_round_trip(dev, orc, n, W, L, chunk, flags):
    """fragment_protect_host_async then fragment_recover_host_async chunk by
    chunk after it: fragments equal the oracle's (and the blocking call's),
    bytes round-trip, the report is clean."""
    x = synth.random_bytes(n, n % 97)
    hx = host(x)
    (a, b, c), tp = se.fragment_protect_host_async(hx, W, L, KEY, IV, flags=flags, chunk_bytes=chunk, n_streams=3)
    out, tr = se.fragment_recover_host_async(a, b, c, n, W, L, KEY, IV, flags=flags, chunk_bytes=chunk,
                                             n_streams=3, after=tp)
    assert tr.wait() == (-1, 0)
    tp.wait()
    assert np.array_equal(out.numpy(), x)
    oa, ob, oc = orc.protect(x, W, L, KEY, IV, flags=flags)
    assert np.array_equal(a.numpy(), oa) and np.array_equal(b.numpy(), ob) and np.array_equal(c.numpy(), oc)


def test_host_async_report_and_back_to_back(dev, orc):
    """Two protects in a row (the second settles the first), a recover of
    damaged fragments: the report equals the oracle's."""
    n, W, L = 1024 * 8 * 64, 1024, 2
    x1, x2 = synth.random_bytes(n, 1), synth.random_bytes(n, 2)
    (a1, b1, c1), t1 = se.fragment_protect_host_async(host(x1), W, L, KEY, IV, chunk_bytes=128 * 1024)
    (a2, b2, c2), t2 = se.fragment_protect_host_async(host(x2), W, L, KEY, IV, chunk_bytes=128 * 1024)
    t2.wait()
    t1.wait()
    oa, ob, oc = orc.protect(x1, W, L, KEY, IV)
    assert np.array_equal(a1.numpy(), oa) and np.array_equal(c1.numpy(), oc)
    c1[60 * 300 + 2] ^= 0x20
    a1[5 * 1000] ^= 0x01
    out, tr = se.fragment_recover_host_async(a1, b1, c1, n, W, L, KEY, IV, chunk_bytes=128 * 1024)
    rep = tr.wait()
    oback, orep = orc.recover(a1.numpy(), b1.numpy(), c1.numpy(), n, W, L, KEY, IV)
    assert rep == orep and orep[1] > 0
    assert np.array_equal(out.numpy(), oback)
