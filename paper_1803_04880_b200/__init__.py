"""paper_1803_04880_b200 — B200-native agnostic selective encryption.

Thin ctypes binding over ``libse.so`` (the C ABI in ``include/se.h``): every
function here only marshals arguments — torch tensors supply device memory
and the current CUDA stream; all work runs in the library's sm_100a kernels.
There is no CPU fallback: if ``libse.so`` is missing or no CUDA device is
present, calls raise.

Names follow the C ABI and the paper's problem statement: protect
maps a chunk D_i to its fragments (D_iA, D_iB, D_iC); recover maps them back.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libse.so")
CSRC = os.path.join(_HERE, "csrc")
SOURCES = ["se_api.cu", "k_block8.cu", "k_tile.cu", "k_full.cu", "k_cipher.cu", "k_stats.cu", "se_host.cu",
           "k_dct.cu", "se_dct_api.cu", "se_container.cpp"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]

SE_OK, SE_EINVAL, SE_EALIGN, SE_ECUDA, SE_ENOTSUP = 0, -1, -2, -3, -4
SE_EFORMAT, SE_EINTEGRITY = -5, -6
MODE_BLOCK8, MODE_FULL = 0, 1
FLAG_PUBLIC_PLAIN = 1
FLAG_HOST_MAPPED = 2      # *_host calls: kernels access the pinned host buffers directly (zero-copy)


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile libse.so in-tree for sm_100a (nvcc cross-compiles without a GPU).
    ``defines``/``out`` build a tuning variant (e.g. ("SE_MIN_CTAS=5",)) to
    another in-tree path, selectable at load time with SE_LIB_PATH."""
    target = out or LIB_PATH
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps += [os.path.join(_ROOT, "include", h) for h in ("se.h", "se_dct.h", "se_container.h")]
    if not force and os.path.exists(target):
        if os.path.getmtime(target) >= max(os.path.getmtime(p) for p in deps):
            return target
    # compile translation units in parallel, then link the shared library
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + f".{os.getpid()}.o")
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            print(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        return obj

    with ThreadPoolExecutor(max_workers=len(sources())) as ex:
        futs = [ex.submit(compile_one, src) for src in sources()]
    errors = [f.exception() for f in futs if f.exception() is not None]
    if errors:
        for f in futs:
            if f.exception() is None and os.path.exists(f.result()):
                os.remove(f.result())
        raise errors[0]
    objs = [f.result() for f in futs]
    tmp = target + f".tmp{os.getpid()}"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    for o in objs:
        os.remove(o)
    os.replace(tmp, target)
    return target


class Geom(C.Structure):
    _fields_ = [("n_bytes", C.c_uint64), ("width", C.c_uint32), ("levels", C.c_uint32),
                ("mode", C.c_uint32), ("flags", C.c_uint32), ("block_offset", C.c_uint64)]


class Layout(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("n_blocks", C.c_uint64), ("a_bytes", C.c_uint64),
                ("b_bytes", C.c_uint64), ("c_bytes", C.c_uint64), ("a_bits", C.c_uint32),
                ("b_bits", C.c_uint32), ("c_bits", C.c_uint32), ("halo_rows", C.c_uint32)]


class Job(C.Structure):
    _fields_ = [("in_", C.c_void_p), ("out", C.c_void_p), ("a", C.c_void_p), ("b", C.c_void_p),
                ("c", C.c_void_p), ("n_bytes", C.c_uint64), ("block_offset", C.c_uint64),
                ("width", C.c_uint32), ("reserved0", C.c_uint32), ("iv", C.c_uint8 * 16),
                ("cta_begin", C.c_uint64), ("derived", C.c_uint32 * 132)]


SYMBOLS = ["fragment_layout", "fragment_protect", "fragment_recover", "fragment_batch_plan",
           "fragment_protect_batch", "fragment_recover_batch", "fragment_protect_host",
           "fragment_recover_host", "dwt_fwd", "dwt_inv", "cipher_encrypt", "cipher_decrypt",
           "se_stats_accumulate", "se_strerror", "se_launch_count",
           "dct_layout", "dct_protect", "dct_recover", "dct_select", "dct8_forward", "dct8_inverse",
           "se_container_streams", "se_container_size", "se_container_pack", "se_container_open",
           "se_disperse_plan", "se_storage_footprint", "se_sha256",
           "fragment_protect_stripe", "fragment_recover_stripe", "fragment_workspace_size",
           "fragment_protect_ws", "fragment_recover_ws", "se_kernel_choice", "se_full_segment_rows",
           "fragment_protect_host_async", "fragment_recover_host_async", "se_host_wait"]


class Stripe(C.Structure):
    _fields_ = [("row_begin", C.c_uint64), ("row_end", C.c_uint64), ("src_row0", C.c_uint64),
                ("src_rows", C.c_uint64)]


class ContainerInfo(C.Structure):
    _fields_ = [("scheme", C.c_uint32), ("flags", C.c_uint32), ("levels", C.c_uint32), ("width", C.c_uint32),
                ("height", C.c_uint32), ("channels", C.c_uint32), ("n_bytes", C.c_uint64),
                ("block_offset", C.c_uint64), ("iv", C.c_uint8 * 16)]


class DctGeom(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("channels", C.c_uint32),
                ("level", C.c_uint32), ("flags", C.c_uint32), ("reserved", C.c_uint32),
                ("block_offset", C.c_uint64)]


class DctLayout(C.Structure):
    _fields_ = [("records", C.c_uint64), ("a_bytes", C.c_uint64), ("p_bytes", C.c_uint64),
                ("a_bits", C.c_uint32), ("reserved", C.c_uint32)]

_lib = None


def lib():
    """Load libse.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SE_LIB_PATH", LIB_PATH)
        if not os.path.exists(path):
            raise RuntimeError(f"libse.so not built ({path}); run __graft_entry__.build()")
        L = C.CDLL(path)
        vp, u8p = C.c_void_p, C.c_char_p
        gp = C.POINTER(Geom)
        L.fragment_layout.argtypes = [gp, C.POINTER(Layout)]
        L.fragment_protect.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, vp]
        L.fragment_recover.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, vp, vp]
        L.fragment_batch_plan.argtypes = [C.POINTER(Job), C.c_uint32, C.c_uint32, u8p]
        L.fragment_batch_plan.restype = C.c_int64
        L.fragment_protect_batch.argtypes = [C.c_uint32, vp, C.c_uint64, C.c_uint32, C.c_uint32, u8p, vp]
        L.fragment_recover_batch.argtypes = [C.c_uint32, vp, C.c_uint64, C.c_uint32, C.c_uint32, u8p, vp, vp]
        L.fragment_protect_host.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, C.c_uint64, C.c_uint32]
        L.fragment_recover_host.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, vp, C.c_uint64, C.c_uint32]
        L.fragment_protect_host_async.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, C.c_uint64, C.c_uint32,
                                                  C.POINTER(C.c_void_p)]
        L.fragment_recover_host_async.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, C.c_uint64, C.c_uint32, vp,
                                                  C.POINTER(C.c_void_p)]
        L.se_host_wait.argtypes = [vp, vp]
        L.dwt_fwd.argtypes = [gp, vp, vp, vp]
        L.dwt_inv.argtypes = [gp, vp, vp, vp]
        L.cipher_encrypt.argtypes = [u8p, u8p, C.c_uint64, vp, vp, C.c_uint64, vp]
        L.cipher_decrypt.argtypes = [u8p, u8p, C.c_uint64, vp, vp, C.c_uint64, vp]
        L.se_stats_accumulate.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, vp, vp]
        dg = C.POINTER(DctGeom)
        L.dct_layout.argtypes = [dg, C.POINTER(DctLayout)]
        L.dct_protect.argtypes = [dg, u8p, u8p, vp, vp, vp, vp]
        L.dct_recover.argtypes = [dg, u8p, u8p, vp, vp, vp, vp]
        L.dct_select.argtypes = [dg, vp, vp, vp]
        L.dct8_forward.argtypes = [dg, vp, vp, vp]
        L.dct8_inverse.argtypes = [dg, vp, vp, vp]
        cip = C.POINTER(ContainerInfo)
        L.se_container_streams.argtypes = [cip, C.POINTER(C.c_uint64)]
        L.se_container_size.argtypes = [cip, C.c_uint32, C.POINTER(C.c_uint64)]
        L.se_container_pack.argtypes = [cip, C.c_uint32, C.POINTER(C.c_void_p), vp, C.c_uint64,
                                        C.POINTER(C.c_uint64)]
        L.se_container_open.argtypes = [vp, C.c_uint64, C.c_int, cip, C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_uint32)]
        L.se_disperse_plan.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.se_storage_footprint.argtypes = [cip, C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.se_sha256.argtypes = [vp, C.c_uint64, vp]
        L.se_sha256.restype = None
        sp = C.POINTER(Stripe)
        L.fragment_protect_stripe.argtypes = [gp, sp, u8p, u8p, vp, vp, vp, vp, vp, C.c_uint64, vp]
        L.fragment_recover_stripe.argtypes = [gp, sp, u8p, u8p, vp, vp, vp, vp, vp, vp, C.c_uint64, vp]
        L.fragment_workspace_size.argtypes = [gp, sp, C.POINTER(C.c_uint64)]
        L.fragment_protect_ws.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, vp, C.c_uint64, vp]
        L.fragment_recover_ws.argtypes = [gp, u8p, u8p, vp, vp, vp, vp, vp, vp, C.c_uint64, vp]
        L.se_strerror.argtypes = [C.c_int]
        L.se_strerror.restype = C.c_char_p
        L.se_full_segment_rows.argtypes = [C.c_int]
        L.se_kernel_choice.argtypes = [C.c_int]
        L.se_kernel_choice.restype = C.c_int
        L.se_launch_count.argtypes = [C.c_int]
        L.se_launch_count.restype = C.c_uint64
        _lib = L
    return _lib


class SEError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {lib().se_strerror(status).decode()} ({status})")
        self.status = status


def _check(rc: int, what: str):
    if rc != SE_OK:
        raise SEError(rc, what)


def _geom(n_bytes, width, levels, mode=MODE_BLOCK8, flags=0, block_offset=0) -> Geom:
    return Geom(int(n_bytes), int(width), int(levels), int(mode), int(flags), int(block_offset))


def _bytes16(x, name) -> bytes:
    b = bytes(x)
    if len(b) != 16:
        raise ValueError(f"{name} must be 16 bytes")
    return b


def _stream(stream):
    import torch
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def fragment_layout(n_bytes: int, width: int, levels: int, mode: int = MODE_BLOCK8,
                    flags: int = 0, block_offset: int = 0) -> dict:
    g = _geom(n_bytes, width, levels, mode, flags, block_offset)
    out = Layout()
    _check(lib().fragment_layout(C.byref(g), C.byref(out)), "fragment_layout")
    return {k: int(getattr(out, k)) for k, _ in Layout._fields_}


def _empty(n, device):
    import torch
    return torch.empty(max(int(n), 1), dtype=torch.uint8, device=device)[: int(n)] if n else \
        torch.empty(16, dtype=torch.uint8, device=device)[:0]


def fragment_workspace_size(n_bytes: int, width: int, levels: int, mode: int = MODE_BLOCK8, stripe=None) -> int:
    """Device workspace bytes a FULL-mode call needs (0 in BLOCK8); stripe =
    (row_begin, row_end, src_row0, src_rows) for the stripe calls."""
    g = _geom(n_bytes, width, levels, mode)
    st = Stripe(*[int(v) for v in stripe]) if stripe is not None else None
    out = C.c_uint64()
    _check(lib().fragment_workspace_size(C.byref(g), C.byref(st) if st is not None else None, C.byref(out)),
           "fragment_workspace_size")
    return int(out.value)


def _workspace(nbytes: int, device, stream):
    """A caller-side workspace tensor (torch's caching allocator; kept alive
    for the stream's use of it with record_stream)."""
    import torch
    if nbytes == 0:
        return None
    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    if stream is not None and hasattr(stream, "cuda_stream"):
        ws.record_stream(stream)
    return ws


def fragment_protect(x, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8, flags: int = 0,
                     block_offset: int = 0, out=None, stream=None, workspace=None):
    """x: 1-D uint8 CUDA tensor (n bytes).  Returns device tensors (A', B', C').
    FULL mode uses `workspace` (a uint8 CUDA tensor of fragment_workspace_size
    bytes) or allocates one through torch."""
    lay = fragment_layout(x.numel(), width, levels, mode, flags, block_offset)
    a, b, c = out if out is not None else (_empty(lay["a_bytes"], x.device), _empty(lay["b_bytes"], x.device),
                                           _empty(lay["c_bytes"], x.device))
    g = _geom(x.numel(), width, levels, mode, flags, block_offset)
    if mode == MODE_FULL:
        ws = workspace if workspace is not None else \
            _workspace(fragment_workspace_size(x.numel(), width, levels, mode), x.device, stream)
        _check(lib().fragment_protect_ws(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(x), _ptr(a),
                                         _ptr(b) if b.numel() else None, _ptr(c), _ptr(ws),
                                         ws.numel() if ws is not None else 0, _stream(stream)), "fragment_protect_ws")
        return a, b, c
    _check(lib().fragment_protect(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(x), _ptr(a),
                                  _ptr(b) if b.numel() else None, _ptr(c), _stream(stream)), "fragment_protect")
    return a, b, c


def fragment_recover(a, b, c, n_bytes: int, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8,
                     flags: int = 0, block_offset: int = 0, out=None, report=None, stream=None, workspace=None):
    """Returns (bytes tensor, report tensor int64[2] = [first_bad_block, bad_blocks])."""
    import torch
    dev = a.device
    o = out if out is not None else _empty(n_bytes, dev)
    rep = report if report is not None else torch.empty(2, dtype=torch.int64, device=dev)
    g = _geom(n_bytes, width, levels, mode, flags, block_offset)
    bb = _ptr(b) if b is not None and b.numel() else None
    if mode == MODE_FULL:
        ws = workspace if workspace is not None else \
            _workspace(fragment_workspace_size(n_bytes, width, levels, mode), dev, stream)
        _check(lib().fragment_recover_ws(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(a), bb, _ptr(c),
                                         _ptr(o), _ptr(rep), _ptr(ws), ws.numel() if ws is not None else 0,
                                         _stream(stream)), "fragment_recover_ws")
        return o, rep
    _check(lib().fragment_recover(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(a), bb, _ptr(c),
                                  _ptr(o), _ptr(rep), _stream(stream)), "fragment_recover")
    return o, rep


def fragment_protect_stripe(src, n_bytes: int, width: int, levels: int, key, iv, row_begin: int, row_end: int,
                            src_row0: int, flags: int = 0, block_offset: int = 0, out=None, stream=None,
                            workspace=None):
    """FULL-mode stripe: `src` = input bytes of rows [src_row0, ...) (the stripe
    plus halo rows).  Returns the stripe's (A', B', C') slices (device)."""
    lay = fragment_layout(n_bytes, width, levels, MODE_FULL, flags, block_offset)
    nb = (row_end - row_begin) // 8 * (width // 8)
    sizes = [-(-nb * lay[k] // 8) for k in ("a_bits", "b_bits", "c_bits")]
    a, b, c = out if out is not None else tuple(_empty(n, src.device) for n in sizes)
    src_rows = -(-src.numel() // width)
    st = Stripe(int(row_begin), int(row_end), int(src_row0), int(min(src_rows, lay["rows"] - src_row0)))
    g = _geom(n_bytes, width, levels, MODE_FULL, flags, block_offset)
    ws = workspace if workspace is not None else _workspace(
        fragment_workspace_size(n_bytes, width, levels, MODE_FULL, (st.row_begin, st.row_end, st.src_row0,
                                                                    st.src_rows)), src.device, stream)
    _check(lib().fragment_protect_stripe(C.byref(g), C.byref(st), _bytes16(key, "key"), _bytes16(iv, "iv"),
                                         _ptr(src), _ptr(a), _ptr(b) if b.numel() else None, _ptr(c),
                                         _ptr(ws), ws.numel(), _stream(stream)),
           "fragment_protect_stripe")
    return a, b, c


def fragment_recover_stripe(a, b, c, n_bytes: int, width: int, levels: int, key, iv, row_begin: int, row_end: int,
                            src_row0: int, src_rows: int, flags: int = 0, block_offset: int = 0, out=None,
                            report=None, stream=None, workspace=None):
    """FULL-mode stripe recovery from the fragments of block rows [src_row0/8,
    (src_row0+src_rows)/8).  Returns (stripe bytes, report[2])."""
    import torch
    dev = a.device
    nbytes = max(0, min(n_bytes, row_end * width) - row_begin * width)
    o = out if out is not None else _empty(nbytes, dev)
    rep = report if report is not None else torch.empty(2, dtype=torch.int64, device=dev)
    st = Stripe(int(row_begin), int(row_end), int(src_row0), int(src_rows))
    g = _geom(n_bytes, width, levels, MODE_FULL, flags, block_offset)
    ws = workspace if workspace is not None else _workspace(
        fragment_workspace_size(n_bytes, width, levels, MODE_FULL, (row_begin, row_end, src_row0, src_rows)),
        dev, stream)
    _check(lib().fragment_recover_stripe(C.byref(g), C.byref(st), _bytes16(key, "key"), _bytes16(iv, "iv"),
                                         _ptr(a), _ptr(b) if b is not None and b.numel() else None, _ptr(c),
                                         _ptr(o), _ptr(rep), _ptr(ws), ws.numel(), _stream(stream)),
           "fragment_recover_stripe")
    return o, rep


def dwt_fwd(x, width: int, levels: int, mode: int = MODE_BLOCK8, out=None, stream=None):
    """Returns the R x W int16 coefficient matrix (device)."""
    import torch
    lay = fragment_layout(x.numel(), width, levels, mode)
    coef = out if out is not None else torch.empty((lay["rows"], width), dtype=torch.int16, device=x.device)
    g = _geom(x.numel(), width, levels, mode)
    _check(lib().dwt_fwd(C.byref(g), _ptr(x), _ptr(coef), _stream(stream)), "dwt_fwd")
    return coef


def dwt_inv(coef, n_bytes: int, width: int, levels: int, mode: int = MODE_BLOCK8, out=None, stream=None):
    o = out if out is not None else _empty(n_bytes, coef.device)
    g = _geom(n_bytes, width, levels, mode)
    _check(lib().dwt_inv(C.byref(g), _ptr(coef), _ptr(o), _stream(stream)), "dwt_inv")
    return o


def cipher_encrypt(key, iv, x, ctr_block_offset: int = 0, out=None, stream=None):
    o = out if out is not None else _empty(x.numel(), x.device)
    _check(lib().cipher_encrypt(_bytes16(key, "key"), _bytes16(iv, "iv"), int(ctr_block_offset), _ptr(x),
                                _ptr(o), x.numel(), _stream(stream)), "cipher_encrypt")
    return o


def cipher_decrypt(key, iv, x, ctr_block_offset: int = 0, out=None, stream=None):
    o = out if out is not None else _empty(x.numel(), x.device)
    _check(lib().cipher_decrypt(_bytes16(key, "key"), _bytes16(iv, "iv"), int(ctr_block_offset), _ptr(x),
                                _ptr(o), x.numel(), _stream(stream)), "cipher_decrypt")
    return o


# ---------------------------------------------------------------- Chapter 4 DCT SE (row f3, se_dct.h)

DCT_KEYED = 1


def _dgeom(width, height, channels, level, flags=0, block_offset=0) -> DctGeom:
    return DctGeom(int(width), int(height), int(channels), int(level), int(flags), 0, int(block_offset))


def dct_layout(width: int, height: int, channels: int = 1, level: int = 1, flags: int = 0,
               block_offset: int = 0) -> dict:
    out = DctLayout()
    _check(lib().dct_layout(C.byref(_dgeom(width, height, channels, level, flags, block_offset)), C.byref(out)),
           "dct_layout")
    return {k: int(getattr(out, k)) for k, _ in DctLayout._fields_ if k != "reserved"}


def dct_protect(img, width: int, height: int, channels: int, level: int, key, iv, flags: int = 0,
                block_offset: int = 0, out=None, stream=None):
    """img: uint8 CUDA tensor of W*H*channels pixels.  Returns (A', P) device tensors."""
    lay = dct_layout(width, height, channels, level, flags, block_offset)
    a, p = out if out is not None else (_empty(lay["a_bytes"], img.device), _empty(lay["p_bytes"], img.device))
    g = _dgeom(width, height, channels, level, flags, block_offset)
    _check(lib().dct_protect(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(img), _ptr(a), _ptr(p),
                             _stream(stream)), "dct_protect")
    return a, p


def dct_recover(a, p, width: int, height: int, channels: int, level: int, key, iv, flags: int = 0,
                block_offset: int = 0, out=None, stream=None):
    """Returns the rebuilt image (uint8 device tensor)."""
    lay = dct_layout(width, height, channels, level, flags, block_offset)
    o = out if out is not None else _empty(lay["p_bytes"], p.device)
    g = _dgeom(width, height, channels, level, flags, block_offset)
    _check(lib().dct_recover(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(a), _ptr(p), _ptr(o),
                             _stream(stream)), "dct_recover")
    return o


def dct_select(img, width: int, height: int, channels: int = 1, out=None, stream=None):
    """The 6 selected fp32 coefficients per record: (records, 6) device tensor."""
    import torch
    lay = dct_layout(width, height, channels)
    o = out if out is not None else torch.empty((lay["records"], 6), dtype=torch.float32, device=img.device)
    g = _dgeom(width, height, channels, 1)
    _check(lib().dct_select(C.byref(g), _ptr(img), _ptr(o), _stream(stream)), "dct_select")
    return o


# ---------------------------------------------------------------- containers / dispersion (row f4, se_container.h)

SCHEME_DWT_BLOCK8, SCHEME_DWT_FULL, SCHEME_DCT = 1, 2, 3
STREAM_A, STREAM_B, STREAM_C, STREAM_P = 0, 1, 2, 3
LAYOUT_A_LOCAL, LAYOUT_AB_LOCAL = 0, 1


def container_info(scheme: int, n_bytes: int, width: int, levels: int, iv, flags: int = 0, block_offset: int = 0,
                   height: int = 0, channels: int = 1) -> ContainerInfo:
    info = ContainerInfo(int(scheme), int(flags), int(levels), int(width), int(height), int(channels),
                         int(n_bytes), int(block_offset))
    info.iv[:] = list(_bytes16(iv, "iv"))
    return info


def _host_bytes(x):
    import numpy as np
    if hasattr(x, "cpu"):
        x = x.cpu().numpy()
    return np.ascontiguousarray(np.frombuffer(bytes(x), np.uint8) if isinstance(x, (bytes, bytearray)) else x,
                                dtype=np.uint8)


def container_streams(info: ContainerInfo) -> list:
    lens = (C.c_uint64 * 4)()
    _check(lib().se_container_streams(C.byref(info), lens), "se_container_streams")
    return [int(v) for v in lens]


def container_pack(info: ContainerInfo, streams: dict):
    """streams: {stream id: host bytes / numpy / tensor}.  Returns the container (numpy uint8)."""
    import numpy as np
    mask = 0
    keep = {}
    ptrs = (C.c_void_p * 4)()
    for sid, data in streams.items():
        mask |= 1 << sid
        keep[sid] = _host_bytes(data)
        ptrs[sid] = keep[sid].ctypes.data if keep[sid].size else None
    size = C.c_uint64()
    _check(lib().se_container_size(C.byref(info), mask, C.byref(size)), "se_container_size")
    lens = container_streams(info)
    for sid, a in keep.items():
        if a.size != lens[sid]:
            raise ValueError(f"stream {sid}: {a.size} bytes, layout says {lens[sid]}")
    out = np.zeros(size.value, np.uint8)
    written = C.c_uint64()
    _check(lib().se_container_pack(C.byref(info), mask, ptrs, out.ctypes.data, out.size, C.byref(written)),
           "se_container_pack")
    return out


def container_open(buf, verify: bool = True):
    """Returns (info, {stream id: numpy view into buf}).  Raises SEError
    (status SE_EFORMAT / SE_EINTEGRITY; .bad_mask = failing stream ids)."""
    import numpy as np
    b = _host_bytes(buf)
    info = ContainerInfo()
    mask = C.c_uint32()
    bad = C.c_uint32()
    ptrs = (C.c_void_p * 4)()
    rc = lib().se_container_open(b.ctypes.data if b.size else None, b.size, 1 if verify else 0, C.byref(info),
                                 C.byref(mask), ptrs, C.byref(bad))
    if rc != SE_OK:
        err = SEError(rc, "se_container_open")
        err.bad_mask = int(bad.value)
        raise err
    lens = container_streams(info)
    base = b.ctypes.data
    streams = {sid: b[ptrs[sid] - base: ptrs[sid] - base + lens[sid]] if lens[sid] else np.zeros(0, np.uint8)
               for sid in range(4) if (mask.value >> sid) & 1}
    return info, streams


def disperse_plan(layout: int, scheme: int):
    """(local stream mask, [remote mask 0, remote mask 1]) of a placement layout."""
    lm = C.c_uint32()
    rm = (C.c_uint32 * 2)()
    _check(lib().se_disperse_plan(int(layout), int(scheme), C.byref(lm), rm), "se_disperse_plan")
    return int(lm.value), [int(rm[0]), int(rm[1])]


def disperse(info: ContainerInfo, streams: dict, layout: int) -> dict:
    """Pack the fragments into the layout's containers: {"local": c, "remote": [c, ...]}."""
    lm, rms = disperse_plan(layout, info.scheme)

    def pick(mask):
        return {sid: streams[sid] for sid in range(4) if (mask >> sid) & 1}
    return {"local": container_pack(info, pick(lm)), "remote": [container_pack(info, pick(m)) for m in rms if m]}


def storage_footprint(info: ContainerInfo, layout: int):
    """(local bytes / n, total bytes / n) for a layout, headers included."""
    lo, to = C.c_double(), C.c_double()
    _check(lib().se_storage_footprint(C.byref(info), int(layout), C.byref(lo), C.byref(to)), "se_storage_footprint")
    return lo.value, to.value


def sha256(data) -> bytes:
    b = _host_bytes(data)
    out = (C.c_uint8 * 32)()
    lib().se_sha256(b.ctypes.data if b.size else None, b.size, out)
    return bytes(out)


def dct8_forward(img, width: int, height: int, channels: int = 1, out=None, stream=None):
    """DCT 8x8 (Eq. 4.1) of (img - 128), fp32 coefficients in pixel layout (device tensor)."""
    import torch
    lay = dct_layout(width, height, channels)
    o = out if out is not None else torch.empty(lay["p_bytes"], dtype=torch.float32, device=img.device)
    _check(lib().dct8_forward(C.byref(_dgeom(width, height, channels, 1)), _ptr(img), _ptr(o), _stream(stream)),
           "dct8_forward")
    return o


def dct8_inverse(coef, width: int, height: int, channels: int = 1, out=None, stream=None):
    """iDCT 8x8 (Eq. 4.2) + 128, rounded to bytes in [0, 255] (device tensor)."""
    lay = dct_layout(width, height, channels)
    o = out if out is not None else _empty(lay["p_bytes"], coef.device)
    _check(lib().dct8_inverse(C.byref(_dgeom(width, height, channels, 1)), _ptr(coef), _ptr(o), _stream(stream)),
           "dct8_inverse")
    return o


KERNEL_AUTO, KERNEL_TILE, KERNEL_CTA = 0, 1, 2


def kernel_choice(choice: int = -1) -> int:
    """Set (0 auto, 1 tile, 2 per-CTA) or query (-1) which kernels serve
    single-file BLOCK8 calls; returns the previous choice."""
    return int(lib().se_kernel_choice(int(choice)))


def full_segment_rows(rows: int) -> int:
    """Test knob: rows per segment of the FULL-mode streaming transform (0 = auto)."""
    r = int(lib().se_full_segment_rows(int(rows)))
    if r < 0:
        raise SEError(r, "se_full_segment_rows")
    return r


def launch_count(reset: bool = False) -> int:
    return int(lib().se_launch_count(1 if reset else 0))


# ---------------------------------------------------------------- batches of files (C5)

class Batch:
    """Device-resident job table for fragment_protect_batch / fragment_recover_batch.

    files: list of 1-D uint8 CUDA tensors (inputs); widths: per-file W; ivs:
    per-file 16-byte IVs.  Allocates the fragment streams (and recover
    outputs) and plans the launch with fragment_batch_plan."""

    def __init__(self, files, widths, ivs, levels: int, key, flags: int = 0, block_offsets=None):
        import torch
        self.levels, self.flags, self.key = int(levels), int(flags), _bytes16(key, "key")
        self.files = list(files)
        n = len(self.files)
        dev = self.files[0].device if n else torch.device("cuda")
        self.jobs = (Job * max(n, 1))()
        self.outs, self.streams = [], []
        for i, (x, w, iv) in enumerate(zip(self.files, widths, ivs)):
            lay = fragment_layout(x.numel(), w, levels)
            a, b, c = _empty(lay["a_bytes"], dev), _empty(lay["b_bytes"], dev), _empty(lay["c_bytes"], dev)
            o = _empty(x.numel(), dev)
            self.streams.append((a, b, c))
            self.outs.append(o)
            j = self.jobs[i]
            j.in_, j.out = x.data_ptr(), o.data_ptr()
            j.a, j.b, j.c = a.data_ptr(), (b.data_ptr() if b.numel() else 0), c.data_ptr()
            j.n_bytes, j.width = x.numel(), int(w)
            j.block_offset = int(block_offsets[i]) if block_offsets is not None else 0
            j.iv[:] = list(_bytes16(iv, "iv"))
        total = lib().fragment_batch_plan(self.jobs, n, self.levels, self.key)
        if total < 0:
            raise SEError(int(total), "fragment_batch_plan")
        self.total_ctas = int(total)
        self.n = n
        raw = bytes(C.string_at(C.addressof(self.jobs), C.sizeof(Job) * max(n, 1)))
        self.d_jobs = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
        self.reports = torch.empty((max(n, 1), 2), dtype=torch.int64, device=dev)

    def protect(self, stream=None):
        _check(lib().fragment_protect_batch(self.n, _ptr(self.d_jobs), self.total_ctas, self.levels, self.flags,
                                            self.key, _stream(stream)), "fragment_protect_batch")
        return self.streams

    def recover(self, stream=None):
        _check(lib().fragment_recover_batch(self.n, _ptr(self.d_jobs), self.total_ctas, self.levels, self.flags,
                                            self.key, _ptr(self.reports), _stream(stream)), "fragment_recover_batch")
        return self.outs, self.reports[: self.n]


# ---------------------------------------------------------------- host-resident streaming (f1)

class Report(C.Structure):
    _fields_ = [("first_bad_block", C.c_int64), ("bad_blocks", C.c_uint64)]


def _host_empty(n, pin=True):
    import torch
    t = torch.empty(max(int(n), 1), dtype=torch.uint8)
    if pin:
        t = t.pin_memory()
    return t[: int(n)]


def fragment_protect_host(x, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8, flags: int = 0,
                          block_offset: int = 0, out=None, chunk_bytes: int = 0, n_streams: int = 0):
    """x: 1-D uint8 CPU tensor (pinned for overlap).  Returns CPU tensors (A', B', C')."""
    lay = fragment_layout(x.numel(), width, levels, mode, flags, block_offset)
    a, b, c = out if out is not None else (_host_empty(lay["a_bytes"]), _host_empty(lay["b_bytes"]),
                                           _host_empty(lay["c_bytes"]))
    g = _geom(x.numel(), width, levels, mode, flags, block_offset)
    _check(lib().fragment_protect_host(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(x), _ptr(a),
                                       _ptr(b) if b.numel() else None, _ptr(c), int(chunk_bytes), int(n_streams)),
           "fragment_protect_host")
    return a, b, c


def fragment_recover_host(a, b, c, n_bytes: int, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8,
                          flags: int = 0, block_offset: int = 0, out=None, chunk_bytes: int = 0, n_streams: int = 0):
    """Returns (CPU uint8 tensor, (first_bad_block, bad_blocks))."""
    o = out if out is not None else _host_empty(n_bytes)
    rep = Report()
    g = _geom(n_bytes, width, levels, mode, flags, block_offset)
    _check(lib().fragment_recover_host(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(a),
                                       _ptr(b) if b is not None and b.numel() else None, _ptr(c), _ptr(o),
                                       C.byref(rep), int(chunk_bytes), int(n_streams)), "fragment_recover_host")
    return o, (int(rep.first_bad_block), int(rep.bad_blocks))


class HostTicket:
    """An asynchronous host call in flight (fragment_*_host_async); wait()
    blocks until its work is done and returns the recover report (or None)."""

    def __init__(self, handle, keep):
        self._h = handle
        self._keep = keep            # host tensors the call reads / writes
        self.report = None

    def wait(self):
        if self._h is None:
            return self.report
        rep = Report()
        st = lib().se_host_wait(self._h, C.byref(rep))
        self._h = None
        self._keep = None
        _check(st, "se_host_wait")
        self.report = (int(rep.first_bad_block), int(rep.bad_blocks))
        return self.report


def fragment_protect_host_async(x, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8, flags: int = 0,
                                block_offset: int = 0, out=None, chunk_bytes: int = 0, n_streams: int = 0):
    """Enqueue fragment_protect_host; returns ((A', B', C') host tensors, HostTicket)."""
    lay = fragment_layout(x.numel(), width, levels, mode, flags, block_offset)
    a, b, c = out if out is not None else (_host_empty(lay["a_bytes"]), _host_empty(lay["b_bytes"]),
                                           _host_empty(lay["c_bytes"]))
    g = _geom(x.numel(), width, levels, mode, flags, block_offset)
    h = C.c_void_p()
    _check(lib().fragment_protect_host_async(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(x), _ptr(a),
                                             _ptr(b) if b.numel() else None, _ptr(c), int(chunk_bytes),
                                             int(n_streams), C.byref(h)), "fragment_protect_host_async")
    return (a, b, c), HostTicket(h, (x, a, b, c))


def fragment_recover_host_async(a, b, c, n_bytes: int, width: int, levels: int, key, iv, mode: int = MODE_BLOCK8,
                                flags: int = 0, block_offset: int = 0, out=None, chunk_bytes: int = 0,
                                n_streams: int = 0, after=None):
    """Enqueue fragment_recover_host, chunk by chunk after the protect ticket
    `after` (if given); returns (host bytes tensor, HostTicket)."""
    o = out if out is not None else _host_empty(n_bytes)
    g = _geom(n_bytes, width, levels, mode, flags, block_offset)
    h = C.c_void_p()
    _check(lib().fragment_recover_host_async(C.byref(g), _bytes16(key, "key"), _bytes16(iv, "iv"), _ptr(a),
                                             _ptr(b) if b is not None and b.numel() else None, _ptr(c), _ptr(o),
                                             int(chunk_bytes), int(n_streams),
                                             after._h if after is not None else None, C.byref(h)),
           "fragment_recover_host_async")
    return o, HostTicket(h, (a, b, c, o))


# ---------------------------------------------------------------- security battery (f2)

STATS_WORDS = 1 + 256 + 256 + 6 + 18          # se_stats as uint64 words


def stats_accumulate(y, width: int, x=None, stats=None, joint=None, stream=None):
    """One pass of se_stats_accumulate over device byte tensors x (optional) and y.
    Returns (stats int64 tensor of STATS_WORDS, joint int32 tensor of 65536 or None);
    pass the returned tensors back in to accumulate more data."""
    import torch
    dev = y.device
    st = stats if stats is not None else torch.zeros(STATS_WORDS, dtype=torch.int64, device=dev)
    jt = joint if joint is not None else (torch.zeros(65536, dtype=torch.int32, device=dev) if x is not None else None)
    n = y.numel() if x is None else min(x.numel(), y.numel())
    _check(lib().se_stats_accumulate(_ptr(x), _ptr(y), n, int(width), _ptr(st), _ptr(jt), _stream(stream)),
           "se_stats_accumulate")
    return st, jt


def stats_metrics(stats, joint=None) -> dict:
    """The paper's metrics from the exact sums (host arithmetic):
    entropy Eq. 5.6 and chi^2 of y's byte PDF, r_xy Eq. 5.8, bit difference
    Dif (= KS when x, y are fragments under two keys),
    adjacent-pair correlation of y (h, v, d), NMI as
    I(X;Y) / sqrt(H(X) H(Y))."""
    import math
    s = [int(v) for v in (stats.tolist() if hasattr(stats, "tolist") else stats)]
    n = s[0]
    hx, hy = s[1:257], s[257:513]
    sx, sy, sxx, syy, sxy, diff = s[513:519]
    adj = [s[519 + 6 * d: 525 + 6 * d] for d in range(3)]

    def ent(h):
        t = sum(h)
        return -sum(c / t * math.log2(c / t) for c in h if c) if t else 0.0

    def corr(cnt, a, b, aa, bb, ab):
        if cnt == 0:
            return float("nan")
        ea, eb = a / cnt, b / cnt
        da, db = aa / cnt - ea * ea, bb / cnt - eb * eb
        cov = ab / cnt - ea * eb
        return cov / math.sqrt(da * db) if da > 0 and db > 0 else float("nan")
    m = {"n": n, "entropy_y": ent(hy), "entropy_x": ent(hx) if any(hx) else None,
         "chi2_y": sum((c - n / 256) ** 2 / (n / 256) for c in hy) if n else None,
         "r_xy": corr(n, sx, sy, sxx, syy, sxy) if any(hx) else None,
         "dif_bits_pct": 100.0 * diff / (8 * n) if n and any(hx) else None,
         "rho_h": corr(*adj[0]), "rho_v": corr(*adj[1]), "rho_d": corr(*adj[2])}
    if joint is not None:
        j = [int(v) for v in joint.tolist()]
        tot = sum(j)
        mi = 0.0
        for xi in range(256):
            px = hx[xi] / tot if tot else 0
            if not px:
                continue
            for yi in range(256):
                c = j[xi * 256 + yi]
                if c:
                    pxy = c / tot
                    mi += pxy * math.log2(pxy / (px * hy[yi] / tot))
        hxe, hye = ent(hx), ent(hy)
        m["nmi"] = mi / math.sqrt(hxe * hye) if hxe > 0 and hye > 0 else 0.0
    return m
