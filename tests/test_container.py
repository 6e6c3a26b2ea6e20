"""Row f4: fragment containers and dispersion layouts (host-only C ABI,
include/se_container.h) — no GPU needed.

Pinned to: hashlib (the content digest), an independent struct-based
encoder of the documented SEFR v1 layout, the paper's storage figures
(164 b local / 480 b remote per block, 644 b total "about 26 %
more"; 7.8 % local), and the oracle's fragments, which must
survive every layout and rebuild the input; a transmission error in a remote
container is detected by its digest, and when forced through it stays inside
its block."""
from __future__ import annotations

import hashlib
import struct

import numpy as np
import pytest

import synth
import paper_1803_04880_b200 as se

KEY = synth.KEY
IV = synth.iv_for(2)


@pytest.fixture(scope="module")
def lib():
    se.build()
    return se.lib()


@pytest.mark.parametrize("n", [0, 1, 55, 56, 63, 64, 65, 119, 120, 200, 1000, 100003])
def test_sha256_matches_hashlib(lib, n):
    d = synth.random_bytes(n, n)
    assert se.sha256(d) == hashlib.sha256(d.tobytes()).digest()


def reference_container(info, streams: dict) -> bytes:
    """SEFR v1 written out with struct, from the header comment of se_container.h."""
    ids = sorted(streams)
    hdr = struct.pack("<4sHHIIIIIIQQ16sII", b"SEFR", 1, 72, info.scheme, info.flags, info.levels, info.width,
                      info.height, info.channels, info.n_bytes, info.block_offset, bytes(info.iv), len(ids), 0)
    off = 72 + 56 * len(ids)
    entries, body = b"", b""
    for sid in ids:
        data = bytes(streams[sid])
        pad = (-off) % 8
        body += b"\0" * pad
        off += pad
        entries += struct.pack("<IIQQ", sid, 0, off, len(data)) + hashlib.sha256(data).digest()
        body += data
        off += len(data)
    return hdr + entries + body


def dwt_fragments(orc, n=64 * 1024 + 77, W=256, L=2, seed=1):
    x = synth.bitmap(-(-n // (3 * 64)) + 1, 64, 3, seed).reshape(-1)[:n]
    a, b, c = orc.protect(x, W, L, KEY, IV)
    info = se.container_info(se.SCHEME_DWT_BLOCK8, n, W, L, IV)
    return x, info, {se.STREAM_A: a, se.STREAM_B: b, se.STREAM_C: c}


def test_format_equals_documented_layout(lib, orc):
    _, info, st = dwt_fragments(orc, n=5000, W=64)
    for mask in ([0], [1], [2], [0, 1], [1, 2], [0, 1, 2]):
        sub = {i: st[i] for i in mask}
        assert se.container_pack(info, sub).tobytes() == reference_container(info, sub)


@pytest.mark.parametrize("layout", [se.LAYOUT_A_LOCAL, se.LAYOUT_AB_LOCAL])
def test_dispersion_round_trip(lib, orc, layout):
    x, info, st = dwt_fragments(orc)
    parts = se.disperse(info, st, layout)
    assert len(parts["remote"]) == (2 if layout == se.LAYOUT_A_LOCAL else 1)
    merged = {}
    for c in [parts["local"]] + parts["remote"]:
        got_info, streams = se.container_open(c)
        assert bytes(got_info) == bytes(info)
        assert not (set(streams) & set(merged))
        merged.update(streams)
    assert sorted(merged) == [0, 1, 2]
    back, rep = orc.recover(merged[0], merged[1], merged[2], x.size, info.width, info.levels, KEY, IV)
    assert np.array_equal(back, x) and rep == (-1, 0)
    local_sids = set(se.container_open(parts["local"])[1])
    assert local_sids == ({0} if layout == se.LAYOUT_A_LOCAL else {0, 1})
    for c in parts["remote"]:                                  # the private fragment never leaves
        assert se.STREAM_A not in se.container_open(c)[1]
    for c in [parts["local"]] + parts["remote"]:               # no key material anywhere
        assert KEY not in c.tobytes()


def test_dct_dispersion_round_trip(lib, orc):
    W, H, C = 64, 32, 3
    img = synth.bitmap(H, W, C, 4).reshape(-1)
    a, p = orc.dct_protect(img, W, H, C, 2, KEY, IV)
    info = se.container_info(se.SCHEME_DCT, img.size, W, 2, IV, height=H, channels=C)
    parts = se.disperse(info, {se.STREAM_A: a, se.STREAM_P: p}, se.LAYOUT_A_LOCAL)
    (_, loc), (_, rem) = se.container_open(parts["local"]), se.container_open(parts["remote"][0])
    assert set(loc) == {se.STREAM_A} and set(rem) == {se.STREAM_P}
    back = orc.dct_recover(loc[se.STREAM_A], rem[se.STREAM_P], W, H, C, 2, KEY, IV)
    assert np.array_equal(back, orc.dct_recover(a, p, W, H, C, 2, KEY, IV))
    with pytest.raises(se.SEError):                               # two parts, one layout
        se.disperse_plan(se.LAYOUT_AB_LOCAL, se.SCHEME_DCT)


def test_storage_footprint_matches_paper(lib):
    """C2-sized file: A-local keeps 40/512 = 7.8 % local, A+B-local 164/512 =
    32.0 %; both total 644/512 = 125.8 % ("about 26 % more");
    72 + 56 e header bytes per container are the only overhead."""
    n = 6144 * 2048
    info = se.container_info(se.SCHEME_DWT_BLOCK8, n, 6144, 2, IV)
    lo, to = se.storage_footprint(info, se.LAYOUT_A_LOCAL)
    assert abs(lo - 40 / 512) < 1e-4 and abs(to - 644 / 512) < 1e-4
    lo, to = se.storage_footprint(info, se.LAYOUT_AB_LOCAL)
    assert abs(lo - 164 / 512) < 1e-4 and abs(to - 644 / 512) < 1e-4
    assert round(100 * 40 / 512, 1) == 7.8 and round(100 * (644 - 512) / 512) == 26
    dinfo = se.container_info(se.SCHEME_DCT, 4800 * 4800, 4800, 2, IV, height=4800)
    lo, to = se.storage_footprint(dinfo, se.LAYOUT_A_LOCAL)
    assert abs(lo - 66 / 512) < 1e-4 and abs(to - 578 / 512) < 1e-4        # 12.9 % extra


def test_transmission_error_detected_then_confined(lib, orc):
    """A-B local layout: one bit flipped in the remote C container.
    Verification names stream C; forced through, the unmasked C differs in
    exactly that bit and the damage stays in its 8x8 block."""
    x, info, st = dwt_fragments(orc, n=128 * 64, W=128)
    parts = se.disperse(info, st, se.LAYOUT_AB_LOCAL)
    remote = parts["remote"][0].copy()
    _, rem = se.container_open(remote)
    off = rem[se.STREAM_C].ctypes.data - remote.ctypes.data
    blk, bit = 9, 9 * 480 + 123
    remote[off + bit // 8] ^= 0x80 >> (bit % 8)
    with pytest.raises(se.SEError) as e:
        se.container_open(remote)
    assert e.value.status == se.SE_EINTEGRITY and e.value.bad_mask == 1 << se.STREAM_C
    _, rem = se.container_open(remote, verify=False)
    _, loc = se.container_open(parts["local"])
    back, rep = orc.recover(loc[0], loc[1], rem[2], x.size, 128, 2, KEY, IV)
    diff = np.nonzero(back != x)[0]
    assert len(diff) and all((i // 128) // 8 == blk // 16 and (i % 128) // 8 == blk % 16 for i in diff)
    if rep[1] == 0:        # no clipping: the PUBLIC_PLAIN (unmasked) C of the rebuilt bytes is off by one bit
        c_back = orc.protect(back, 128, 2, KEY, IV, flags=1)[2]
        c_true = orc.protect(x, 128, 2, KEY, IV, flags=1)[2]
        assert (np.unpackbits(c_back) ^ np.unpackbits(c_true)).sum() == 1


def test_format_errors(lib, orc):
    _, info, st = dwt_fragments(orc, n=4096, W=64)
    good = se.container_pack(info, st)

    def status(buf):
        with pytest.raises(se.SEError) as e:
            se.container_open(buf)
        return e.value.status
    bad = good.copy(); bad[0] ^= 1
    assert status(bad) == se.SE_EFORMAT                                   # magic
    bad = good.copy(); bad[4] = 2
    assert status(bad) == se.SE_EFORMAT                                   # version
    assert status(good[:100]) == se.SE_EFORMAT                            # truncated
    bad = good.copy(); bad[20] = 12                                       # width 12: invalid geometry
    assert status(bad) == se.SE_EFORMAT
    bad = good.copy(); bad[72 + 56 + 8] ^= 8                              # entry 1 offset overlaps entry 0
    assert status(bad) == se.SE_EFORMAT
    bad = good.copy(); bad[72 + 16] ^= 1                                  # entry 0 length != layout
    assert status(bad) == se.SE_EFORMAT
    bad = good.copy(); bad[72] = 3                                        # stream P in a DWT container
    assert status(bad) == se.SE_EFORMAT
    with pytest.raises(se.SEError):
        se.container_pack(info, {se.STREAM_P: st[0]})                    # foreign stream id
    with pytest.raises(ValueError):
        se.container_pack(info, {se.STREAM_A: st[0][:-1]})               # wrong length
    with pytest.raises(se.SEError):
        se.disperse_plan(7, se.SCHEME_DWT_BLOCK8)
