"""CPU oracle for the Chapter 5 agnostic SE path (arxiv/paper_1803_04880).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product (``paper_1803_04880_b200``, ``libse.so``) never imports
it, and it never imports the product.  See ``oracle/oracle.h`` for the
readings and citations; this file only marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SOURCES = ["dwt53.c", "aes128.c", "sha2.c", "protect.c", "stats.c", "dct.c"]

MODE_BLOCK8 = 0
MODE_FULL = 1
FLAG_PUBLIC_PLAIN = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -O2, no intrinsics)."""
    srcs = [os.path.join(_HERE, s) for s in SOURCES]
    hdr = os.path.join(_HERE, "oracle.h")
    if not force and os.path.exists(LIB_PATH):
        newest = max(os.path.getmtime(p) for p in srcs + [hdr])
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
           "-o", tmp] + srcs + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None

_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = _load(LIB_PATH)
    return _lib


@contextlib.contextmanager
def library_override(path: str):
    """Run this module's functions against another build of the oracle's C
    sources (test infrastructure: tests/test_oracle_mutations.py builds
    deliberately mutated copies and checks that the paper pins reject them)."""
    global _lib
    saved = lib()
    _lib = _load(path)
    try:
        yield
    finally:
        _lib = saved


def _load(path: str):
    L = C.CDLL(path)
    u64, u32 = C.c_uint64, C.c_uint32
    L.oracle_layout.argtypes = [u64, u32, u32, u32, _u64p]
    L.oracle_lift_fwd_1d.argtypes = [_i32p, _i32p, C.c_int]
    L.oracle_lift_inv_1d.argtypes = [_i32p, _i32p, C.c_int]
    L.oracle_dwt_fwd.argtypes = [_u8p, u64, u32, u32, u32, _i32p]
    L.oracle_dwt_inv.argtypes = [_i32p, u64, u32, u32, u32, _u8p]
    L.oracle_dwt_inv.restype = C.c_int64
    L.oracle_aes128_sbox.argtypes = [_u8p]
    L.oracle_aes128_encrypt_block.argtypes = [_u8p, _u8p, _u8p]
    L.oracle_aes128_ctr.argtypes = [_u8p, _u8p, u64, _u8p, _u8p, u64]
    L.oracle_sha256.argtypes = [_u8p, u64, _u8p]
    L.oracle_sha512.argtypes = [_u8p, u64, _u8p]
    L.oracle_protect_range.argtypes = [u64, u32, u32, u32, u32, u64, _u8p, _u8p,
                                       _u8p, _u8p, _u8p, _u8p, u64, u64]
    L.oracle_recover_range.argtypes = [u64, u32, u32, u32, u32, u64, _u8p, _u8p,
                                       _u8p, _u8p, _u8p, _u8p, _i64p, u64, u64]
    L.oracle_dwt2_fwd_region.argtypes = [_i32p, C.c_size_t, C.c_int, C.c_int, C.c_int]
    L.oracle_dwt2_inv_region.argtypes = [_i32p, C.c_size_t, C.c_int, C.c_int, C.c_int]
    L.oracle_stats.argtypes = [_u8p, _u8p, u64, u32, _u64p, _u64p]
    _f64p = C.POINTER(C.c_double)
    L.oracle_dct_basis.argtypes = [_f64p]
    L.oracle_dct8_fwd.argtypes = [_f64p, _f64p]
    L.oracle_dct8_inv.argtypes = [_f64p, _f64p]
    L.oracle_dct_layout.argtypes = [u32, u32, u32, _u64p]
    L.oracle_dct_select.argtypes = [u32, u32, u32, _u8p, _f64p]
    L.oracle_dct_image_fwd.argtypes = [u32, u32, u32, _u8p, _f64p]
    L.oracle_dct_image_inv.argtypes = [u32, u32, u32, _f64p, _u8p]
    L.oracle_dct_protect.argtypes = [u32, u32, u32, u32, u32, u64, _u8p, _u8p, _u8p, _u8p, _u8p, _f64p]
    L.oracle_dct_recover.argtypes = [u32, u32, u32, u32, u32, u64, _u8p, _u8p, _u8p, _u8p, _u8p, _f64p]
    L.oracle_record_fields.argtypes = [u32, u32, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p]
    return L


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _u8(x) -> np.ndarray:
    a = np.ascontiguousarray(np.frombuffer(bytes(x), dtype=np.uint8) if isinstance(x, (bytes, bytearray)) else x,
                             dtype=np.uint8)
    if a.size == 0:
        a = np.zeros(1, dtype=np.uint8)[:0]
    return a


def layout(n_bytes: int, width: int, levels: int, mode: int = MODE_BLOCK8) -> dict:
    out = np.zeros(8, dtype=np.uint64)
    rc = lib().oracle_layout(n_bytes, width, levels, mode, _p(out, _u64p))
    if rc:
        raise ValueError(f"invalid geometry n={n_bytes} W={width} L={levels} mode={mode}")
    keys = ["rows", "n_blocks", "a_bits", "b_bits", "c_bits", "a_bytes", "b_bytes", "c_bytes"]
    return {k: int(v) for k, v in zip(keys, out)}


def lift_fwd_1d(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.zeros_like(x)
    lib().oracle_lift_fwd_1d(_p(x, _i32p), _p(y, _i32p), x.size)
    return y


def lift_inv_1d(y) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.int32)
    x = np.zeros_like(y)
    lib().oracle_lift_inv_1d(_p(y, _i32p), _p(x, _i32p), y.size)
    return x


def dwt2_fwd_region(a, levels: int) -> np.ndarray:
    """In-place-style dyadic transform of a whole int32 2-D array (copy returned)."""
    a = np.array(a, dtype=np.int32, order="C", copy=True)
    lib().oracle_dwt2_fwd_region(_p(a, _i32p), a.shape[1], a.shape[0], a.shape[1], levels)
    return a


def dwt2_inv_region(a, levels: int) -> np.ndarray:
    a = np.array(a, dtype=np.int32, order="C", copy=True)
    lib().oracle_dwt2_inv_region(_p(a, _i32p), a.shape[1], a.shape[0], a.shape[1], levels)
    return a


def dwt_fwd(data, width: int, levels: int, mode: int = MODE_BLOCK8) -> np.ndarray:
    d = _u8(data)
    lay = layout(d.size, width, levels, mode)
    coef = np.zeros((lay["rows"], width), dtype=np.int32)
    buf = d if d.size else np.zeros(1, np.uint8)
    rc = lib().oracle_dwt_fwd(_p(buf, _u8p), d.size, width, levels, mode, _p(coef, _i32p))
    assert rc == 0
    return coef


def dwt_inv(coef, n_bytes: int, width: int, levels: int, mode: int = MODE_BLOCK8):
    coef = np.ascontiguousarray(coef, dtype=np.int32)
    out = np.zeros(max(n_bytes, 1), dtype=np.uint8)
    bad = lib().oracle_dwt_inv(_p(coef, _i32p), n_bytes, width, levels, mode, _p(out, _u8p))
    return out[:n_bytes], int(bad)


def aes128_sbox() -> np.ndarray:
    s = np.zeros(256, dtype=np.uint8)
    lib().oracle_aes128_sbox(_p(s, _u8p))
    return s


def aes128_encrypt_block(key: bytes, block: bytes) -> bytes:
    k, b = _u8(key), _u8(block)
    out = np.zeros(16, dtype=np.uint8)
    lib().oracle_aes128_encrypt_block(_p(k, _u8p), _p(b, _u8p), _p(out, _u8p))
    return out.tobytes()


def aes128_ctr(key: bytes, iv: bytes, data, ctr_offset: int = 0) -> np.ndarray:
    k, v, d = _u8(key), _u8(iv), _u8(data)
    out = np.zeros(max(d.size, 1), dtype=np.uint8)
    buf = d if d.size else np.zeros(1, np.uint8)
    lib().oracle_aes128_ctr(_p(k, _u8p), _p(v, _u8p), ctr_offset, _p(buf, _u8p), _p(out, _u8p), d.size)
    return out[:d.size]


def sha256(msg: bytes) -> bytes:
    m = _u8(msg) if len(msg) else np.zeros(1, np.uint8)
    out = np.zeros(32, dtype=np.uint8)
    lib().oracle_sha256(_p(m, _u8p), len(msg), _p(out, _u8p))
    return out.tobytes()


def sha512(msg: bytes) -> bytes:
    m = _u8(msg) if len(msg) else np.zeros(1, np.uint8)
    out = np.zeros(64, dtype=np.uint8)
    lib().oracle_sha512(_p(m, _u8p), len(msg), _p(out, _u8p))
    return out.tobytes()


def record_fields(levels: int, mode: int, stream: int):
    arrs = [np.zeros(64, dtype=np.int32) for _ in range(5)]
    n = lib().oracle_record_fields(levels, mode, stream, *[_p(a, _i32p) for a in arrs])
    return [tuple(int(a[k]) for a in arrs) for k in range(n)]


def _streams(lay):
    return [np.zeros(max(lay[k], 1), dtype=np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes")]


def protect(data, width: int, levels: int, key: bytes, iv: bytes, mode: int = MODE_BLOCK8,
            flags: int = 0, block_offset: int = 0, block_range=None, out=None):
    """Returns (A', B', C') byte streams.  ``block_range=(b0, b1)`` processes
    only those local blocks into ``out`` (or fresh zeroed streams)."""
    d = _u8(data)
    lay = layout(d.size, width, levels, mode)
    a, b, c = out if out is not None else _streams(lay)
    k, v = _u8(key), _u8(iv)
    b0, b1 = block_range if block_range is not None else (0, lay["n_blocks"])
    buf = d if d.size else np.zeros(1, np.uint8)
    rc = lib().oracle_protect_range(d.size, width, levels, mode, flags, block_offset,
                                    _p(k, _u8p), _p(v, _u8p), _p(buf, _u8p),
                                    _p(a, _u8p), _p(b, _u8p), _p(c, _u8p), b0, b1)
    if rc:
        raise ValueError(f"oracle_protect failed rc={rc}")
    return a[:lay["a_bytes"]], b[:lay["b_bytes"]], c[:lay["c_bytes"]]


def recover(a, b, c, n_bytes: int, width: int, levels: int, key: bytes, iv: bytes,
            mode: int = MODE_BLOCK8, flags: int = 0, block_offset: int = 0, block_range=None,
            out=None):
    """Returns (bytes, (first_bad_block, bad_blocks))."""
    lay = layout(n_bytes, width, levels, mode)
    streams = []
    for s, key_ in zip((a, b, c), ("a_bytes", "b_bytes", "c_bytes")):
        s = _u8(s)
        assert s.size >= lay[key_], (key_, s.size, lay[key_])
        streams.append(s if s.size else np.zeros(1, np.uint8))
    o = out if out is not None else np.zeros(max(n_bytes, 1), dtype=np.uint8)
    rep = np.zeros(2, dtype=np.int64)
    k, v = _u8(key), _u8(iv)
    b0, b1 = block_range if block_range is not None else (0, lay["n_blocks"])
    rc = lib().oracle_recover_range(n_bytes, width, levels, mode, flags, block_offset,
                                    _p(k, _u8p), _p(v, _u8p), *[_p(s, _u8p) for s in streams],
                                    _p(o, _u8p), _p(rep, _i64p), b0, b1)
    if rc:
        raise ValueError(f"oracle_recover failed rc={rc}")
    return o[:n_bytes], (int(rep[0]), int(rep[1]))


STATS_WORDS = 1 + 256 + 256 + 6 + 18


def stats(y, width: int, x=None, joint: bool = True):
    """The security-battery sums (oracle/stats.c): (words uint64[STATS_WORDS], joint uint64[65536] or None)."""
    yy = _u8(y)
    xx = _u8(x) if x is not None else None
    n = yy.size if xx is None else min(xx.size, yy.size)
    out = np.zeros(STATS_WORDS, dtype=np.uint64)
    jt = np.zeros(65536, dtype=np.uint64) if (joint and xx is not None) else None
    lib().oracle_stats(_p(xx, _u8p) if xx is not None else None, _p(yy, _u8p), n, width, _p(out, _u64p),
                       _p(jt, _u64p) if jt is not None else None)
    return out, jt


# ---------------------------------------------------------------- Chapter 4 DCT SE (NEXT row f3, dct.c)

DCT_KEYED = 1
_f64p = C.POINTER(C.c_double)


def dct_basis() -> np.ndarray:
    """Eq. 4.6 layout: m[x, u] = alpha(u) cos(pi (2x+1) u / 16)."""
    m = np.zeros((8, 8))
    lib().oracle_dct_basis(_p(m, _f64p))
    return m


def dct8_fwd(f) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64).reshape(8, 8)
    c = np.zeros((8, 8))
    lib().oracle_dct8_fwd(_p(f, _f64p), _p(c, _f64p))
    return c


def dct8_inv(c) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.float64).reshape(8, 8)
    f = np.zeros((8, 8))
    lib().oracle_dct8_inv(_p(c, _f64p), _p(f, _f64p))
    return f


def dct_layout(width: int, height: int, channels: int = 1) -> dict:
    out = np.zeros(4, dtype=np.uint64)
    if lib().oracle_dct_layout(width, height, channels, _p(out, _u64p)):
        raise ValueError(f"invalid DCT geometry {width}x{height}x{channels}")
    return dict(zip(["records", "bits", "a_bytes", "p_bytes"], (int(v) for v in out)))


def dct_select(img, width: int, height: int, channels: int = 1) -> np.ndarray:
    """(records, 6) real coefficients [0,0],[0,1],[1,0],[2,0],[1,1],[0,2]."""
    lay = dct_layout(width, height, channels)
    x = _u8(img)
    assert x.size == lay["p_bytes"]
    out = np.zeros((lay["records"], 6))
    assert lib().oracle_dct_select(width, height, channels, _p(x, _u8p), _p(out, _f64p)) == 0
    return out


def dct_protect(img, width: int, height: int, channels: int, level: int, key: bytes, iv: bytes,
                flags: int = 0, block_offset: int = 0, real: bool = False):
    """Returns (a, p) or (a, p, p_real[records, 64]) — p_real before rounding and masking."""
    lay = dct_layout(width, height, channels)
    x = _u8(img)
    assert x.size == lay["p_bytes"]
    a = np.zeros(max(lay["a_bytes"], 1), dtype=np.uint8)
    p = np.zeros(lay["p_bytes"], dtype=np.uint8)
    pr = np.zeros((lay["records"], 64)) if real else None
    k, v = _u8(key), _u8(iv)
    rc = lib().oracle_dct_protect(width, height, channels, level, flags, block_offset, _p(k, _u8p), _p(v, _u8p),
                                  _p(x, _u8p), _p(a, _u8p), _p(p, _u8p), _p(pr, _f64p) if real else None)
    if rc:
        raise ValueError(f"oracle_dct_protect failed rc={rc}")
    return (a[:lay["a_bytes"]], p, pr) if real else (a[:lay["a_bytes"]], p)


def dct_recover(a, p, width: int, height: int, channels: int, level: int, key: bytes, iv: bytes,
                flags: int = 0, block_offset: int = 0, real: bool = False):
    """Returns out or (out, out_real[records, 64]) — out_real before rounding."""
    lay = dct_layout(width, height, channels)
    aa, pp = _u8(a), _u8(p)
    assert aa.size >= lay["a_bytes"] and pp.size == lay["p_bytes"]
    if aa.size == 0:
        aa = np.zeros(1, np.uint8)
    out = np.zeros(lay["p_bytes"], dtype=np.uint8)
    orl = np.zeros((lay["records"], 64)) if real else None
    k, v = _u8(key), _u8(iv)
    rc = lib().oracle_dct_recover(width, height, channels, level, flags, block_offset, _p(k, _u8p), _p(v, _u8p),
                                  _p(aa, _u8p), _p(pp, _u8p), _p(out, _u8p), _p(orl, _f64p) if real else None)
    if rc:
        raise ValueError(f"oracle_dct_recover failed rc={rc}")
    return (out, orl) if real else out


def dct_image_fwd(img, width: int, height: int, channels: int = 1) -> np.ndarray:
    """Full DCT 8x8 of (img - 128), coefficients in pixel layout (float64, img's shape)."""
    lay = dct_layout(width, height, channels)
    x = _u8(img)
    assert x.size == lay["p_bytes"]
    out = np.zeros(lay["p_bytes"])
    assert lib().oracle_dct_image_fwd(width, height, channels, _p(x, _u8p), _p(out, _f64p)) == 0
    return out


def dct_image_inv(coef, width: int, height: int, channels: int = 1) -> np.ndarray:
    lay = dct_layout(width, height, channels)
    c = np.ascontiguousarray(coef, dtype=np.float64).reshape(-1)
    assert c.size == lay["p_bytes"]
    out = np.zeros(lay["p_bytes"], np.uint8)
    assert lib().oracle_dct_image_inv(width, height, channels, _p(c, _f64p), _p(out, _u8p)) == 0
    return out
