"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
symbol include/se.h declares; host-only entry points (layout, validation)
behave as documented.  No compute calls (no GPU here)."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

import paper_1803_04880_b200 as se


@pytest.fixture(scope="module")
def lib():
    se.build()
    return se.lib()


def declared_functions():
    inc = os.path.join(ROOT, "include")
    src = "".join(open(os.path.join(inc, h)).read() for h in sorted(os.listdir(inc)) if h.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ["fragment_layout", "fragment_protect", "fragment_recover", "fragment_protect_batch",
              "fragment_recover_batch", "dwt_fwd", "dwt_inv", "cipher_encrypt", "cipher_decrypt",
              "se_strerror", "dct_layout", "dct_protect", "dct_recover", "dct_select"]:
        assert n in names, n


def test_every_declared_symbol_is_exported(lib):
    for n in declared_functions():
        assert hasattr(lib, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", se.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for n in declared_functions():
        assert n in exported, n


def test_binding_names_match_header():
    for n in declared_functions():
        assert n in se.SYMBOLS, n


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", se.LIB_PATH], text=True)
    assert "sm_100a" in out


@pytest.mark.parametrize("n,W,L,expect", [
    (6144 * 2048, 6144, 2, (2048, 196608, 983040, 3047424, 11796480)),
    (1 << 26, 1024, 3, (65536, 1048576, 1310720, 20316160, 62914560)),
    (65536, 256, 1, (256, 1024, 20480, 0, 61440)),
    (1, 8, 2, (8, 1, 5, 16, 60)),
    (0, 8, 2, (0, 0, 0, 0, 0)),
])
def test_layout_host(lib, n, W, L, expect, orc):
    lay = se.fragment_layout(n, W, L)
    assert (lay["rows"], lay["n_blocks"], lay["a_bytes"], lay["b_bytes"], lay["c_bytes"]) == expect
    o = orc.layout(n, W, L)
    assert all(lay[k] == o[k] for k in o)


def test_layout_full_mode_widths(lib):
    lay = se.fragment_layout(64 * 64, 64, 2, mode=se.MODE_FULL)
    assert (lay["a_bits"], lay["b_bits"], lay["c_bits"], lay["halo_rows"]) == (40, 132, 480, 6)


@pytest.mark.parametrize("W,L,mode,flags", [(0, 2, 0, 0), (12, 2, 0, 0), (8, 0, 0, 0), (8, 4, 0, 0),
                                            (8, 2, 2, 0), (8, 2, 0, 4)])
def test_layout_rejects_bad_geometry(lib, W, L, mode, flags):
    with pytest.raises(se.SEError) as e:
        se.fragment_layout(64, W, L, mode, flags)
    assert e.value.status == se.SE_EINVAL


def test_validation_before_any_device_work(lib):
    """Argument errors are reported synchronously without touching the GPU."""
    g = se.Geom(64, 8, 2, 0, 0, 0)
    key = bytes(16)
    # null pointers
    assert lib.fragment_protect(C.byref(g), key, key, None, None, None, None, None) == se.SE_EINVAL
    # misaligned device pointers (never dereferenced: validation fails first)
    assert lib.fragment_protect(C.byref(g), key, key, C.c_void_p(0x1001), C.c_void_p(0x2000),
                                C.c_void_p(0x3000), C.c_void_p(0x4000), None) == se.SE_EALIGN
    # block_offset that does not align the CTR counter (40 * 3 bits is not a multiple of 128)
    g2 = se.Geom(64, 8, 2, 0, 0, 3)
    assert lib.fragment_protect(C.byref(g2), key, key, C.c_void_p(0x1000), C.c_void_p(0x2000),
                                C.c_void_p(0x3000), C.c_void_p(0x4000), None) == se.SE_EINVAL
    # n_bytes == 0 is a no-op
    g0 = se.Geom(0, 8, 2, 0, 0, 0)
    assert lib.fragment_protect(C.byref(g0), key, key, None, None, None, None, None) == se.SE_OK
    assert lib.cipher_encrypt(key, key, 0, None, None, 0, None) == se.SE_OK
    assert lib.cipher_encrypt(None, key, 0, None, None, 16, None) == se.SE_EINVAL
    assert se.lib().se_strerror(se.SE_EALIGN).decode().startswith("device pointer")


@pytest.mark.parametrize("W,H,C", [(4800, 4800, 1), (1600, 1200, 1), (64, 48, 3), (16, 8, 4)])
def test_dct_layout_host(lib, orc, W, H, C):
    lay = se.dct_layout(W, H, C, 2)
    o = orc.dct_layout(W, H, C)
    assert (lay["records"], lay["a_bits"], lay["a_bytes"], lay["p_bytes"]) == \
        (o["records"], o["bits"], o["a_bytes"], o["p_bytes"])


@pytest.mark.parametrize("W,H,C,level,flags,off", [(0, 8, 1, 1, 0, 0), (12, 8, 1, 1, 0, 0), (8, 12, 1, 1, 0, 0),
                                                   (8, 8, 2, 1, 0, 0), (8, 8, 1, 3, 0, 0), (8, 8, 1, 2, 2, 0),
                                                   (8, 8, 1, 1, 0, 3)])
def test_dct_layout_rejects_bad_geometry(lib, W, H, C, level, flags, off):
    with pytest.raises(se.SEError) as e:
        se.dct_layout(W, H, C, level, flags, off)
    assert e.value.status == se.SE_EINVAL


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libse.so the package raises instead of
    computing anything (run in a subprocess so the loaded library is untouched)."""
    import sys
    code = ("import paper_1803_04880_b200 as se\n"
            "try:\n    se.lib()\nexcept RuntimeError as e:\n    print('raised', e)\n")
    env = dict(os.environ, SE_LIB_PATH=str(tmp_path / "missing.so"), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert "raised" in out.stdout and "not built" in out.stdout


def test_product_never_imports_the_oracle():
    """The product package and its sources do not reference oracle/ (the
    oracle is test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_1803_04880_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "oracle.h" not in src and "liboracle" not in src, f
