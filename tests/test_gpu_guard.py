"""Out-of-bounds guard bands (compute-sanitizer is closed on this pool): every
device buffer an entry point reads or writes is a view into a larger
allocation whose 4 KiB before and after the view hold a known pattern.
After each call the guard bytes must be unchanged and the inputs untouched,
so a kernel that writes past the end of a ragged stream, a stripe, the
recovered bytes or a workspace - or before its start - fails here even where
the caching allocator's rounding would otherwise hide it.  Results are also
checked (round trip / oracle), so the views are the real buffers."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = bytes.fromhex("0f0e0d0c0b0a09080706050403020100")
G = 4096                                   # guard bytes on each side (keeps 16-byte alignment)
PAT = 0xA5


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


class Guarded:
    """A uint8 (or other dtype) view of `n` elements with guard bands."""

    def __init__(self, n, dev, dtype=torch.uint8, fill=None):
        esz = torch.empty(0, dtype=dtype).element_size()
        self.raw = torch.full((2 * G + n * esz,), PAT, dtype=torch.uint8, device=dev)
        self.n, self.esz = n, esz
        self.view = self.raw[G:G + n * esz].view(dtype)
        if fill is not None:
            self.view.copy_(fill)

    def guards_ok(self):
        torch.cuda.synchronize()
        lo = self.raw[:G]
        hi = self.raw[G + self.n * self.esz:]
        return bool((lo == PAT).all()) and bool((hi == PAT).all())


def gin(x_np, dev):
    return Guarded(x_np.size, dev, fill=torch.from_numpy(x_np).to(dev))


def gout(n, dev, dtype=torch.uint8):
    return Guarded(n, dev, dtype=dtype)


def check_all(*bufs):
    for i, b in enumerate(bufs):
        assert b.guards_ok(), f"guard band of buffer {i} overwritten"


def test_guard_detects_overwrites(dev):
    """The detector itself: one byte written just past the view (by a device
    copy, as a kernel would) or just before it is reported."""
    g = gout(100, dev)
    assert g.guards_ok()
    g.raw[G + 100: G + 101].copy_(torch.zeros(1, dtype=torch.uint8, device=dev))
    assert not g.guards_ok()
    h = gout(100, dev)
    h.raw[G - 1: G].fill_(0)
    assert not h.guards_ok()


CASES = [
    (1, 8, 2), (777, 24, 1), (128 * 64 * 2 + 77, 1024, 2), (6144 * 8 * 3 + 5, 6144, 2),
    (512 * 64 * 3 + 999, 1024, 3), (1032 * 8 * 20 + 1, 1032, 2),
]


@pytest.mark.parametrize("n,W,L", CASES)
@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("kernel", ["auto", "tile", "cta"])
def test_block8_protect_recover_guards(dev, n, W, L, flags, kernel):
    choice = {"auto": se.KERNEL_AUTO, "tile": se.KERNEL_TILE, "cta": se.KERNEL_CTA}[kernel]
    prev = se.kernel_choice(choice)
    try:
        x_np = synth.random_bytes(n, n + W)
        x = gin(x_np, dev)
        lay = se.fragment_layout(n, W, L, flags=flags)
        a, b, c = (gout(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
        se.fragment_protect(x.view, W, L, KEY, IV, flags=flags, out=(a.view, b.view, c.view))
        out = gout(n, dev)
        rep = gout(2, dev, torch.int64)
        se.fragment_recover(a.view, b.view, c.view, n, W, L, KEY, IV, flags=flags, out=out.view, report=rep.view)
        check_all(x, a, b, c, out, rep)
        assert np.array_equal(x.view.cpu().numpy(), x_np), "input modified"
        assert torch.equal(out.view, x.view) and rep.view.cpu().tolist() == [-1, 0]
    finally:
        se.kernel_choice(prev)


@pytest.mark.parametrize("n,W,L", [(32768 * 8 * 3 + 100, 32768, 2), (4096 * 40 + 3, 4096, 3), (999, 16, 1)])
def test_full_mode_guards(dev, n, W, L):
    x_np = synth.random_bytes(n, 3 * n)
    x = gin(x_np, dev)
    lay = se.fragment_layout(n, W, L, se.MODE_FULL)
    a, b, c = (gout(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
    ws = gout(se.fragment_workspace_size(n, W, L, se.MODE_FULL), dev)
    se.fragment_protect(x.view, W, L, KEY, IV, mode=se.MODE_FULL, out=(a.view, b.view, c.view), workspace=ws.view)
    out = gout(n, dev)
    rep = gout(2, dev, torch.int64)
    ws2 = gout(se.fragment_workspace_size(n, W, L, se.MODE_FULL), dev)
    se.fragment_recover(a.view, b.view, c.view, n, W, L, KEY, IV, mode=se.MODE_FULL, out=out.view,
                        report=rep.view, workspace=ws2.view)
    check_all(x, a, b, c, ws, out, rep, ws2)
    assert torch.equal(out.view, x.view) and rep.view.cpu().tolist() == [-1, 0]


@pytest.mark.parametrize("n,W,L", [(128 * 64 * 2 + 77, 1024, 2), (5000, 128, 3)])
def test_transform_and_cipher_guards(dev, n, W, L):
    x_np = synth.random_bytes(n, 7 * n)
    x = gin(x_np, dev)
    for mode in (se.MODE_BLOCK8, se.MODE_FULL):
        lay = se.fragment_layout(n, W, L, mode)
        coef = gout(lay["rows"] * W, dev, torch.int16)
        se.dwt_fwd(x.view, W, L, mode=mode, out=coef.view.view(lay["rows"], W))
        back = gout(n, dev)
        se.dwt_inv(coef.view.view(lay["rows"], W), n, W, L, mode=mode, out=back.view)
        check_all(x, coef, back)
        assert torch.equal(back.view, x.view)
    for off in (0, 5, (1 << 64) - 3):
        e = gout(n, dev)
        se.cipher_encrypt(KEY, IV, x.view, ctr_block_offset=off, out=e.view)
        d = gout(n, dev)
        se.cipher_decrypt(KEY, IV, e.view, ctr_block_offset=off, out=d.view)
        check_all(x, e, d)
        assert torch.equal(d.view, x.view)


def test_batch_guards(dev):
    sizes = [1, 0, 5000, 70001, 1 << 20, 3 * 1024 * 1024 + 9]
    files = [gin(synth.random_bytes(s, 50 + i), dev) if s else Guarded(0, dev) for i, s in enumerate(sizes)]
    widths = [synth.width_rule(max(s, 1)) for s in sizes]
    ivs = [synth.iv_for(5, 700 + i) for i in range(len(sizes))]
    batch = se.Batch([f.view for f in files], widths, ivs, 2, KEY)
    # point the jobs' fragment and output buffers at guarded views
    gs, go = [], []
    for i, s in enumerate(sizes):
        lay = se.fragment_layout(s, widths[i], 2)
        g3 = tuple(gout(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
        o = gout(s, dev)
        gs.append(g3)
        go.append(o)
        j = batch.jobs[i]
        j.a, j.b, j.c = g3[0].view.data_ptr(), (g3[1].view.data_ptr() if g3[1].n else 0), g3[2].view.data_ptr()
        j.out = o.view.data_ptr()
    batch.streams = [tuple(g.view for g in g3) for g3 in gs]
    batch.outs = [o.view for o in go]
    import ctypes
    raw = bytes(ctypes.string_at(ctypes.addressof(batch.jobs), ctypes.sizeof(batch.jobs)))
    batch.d_jobs = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
    batch.protect()
    outs, reps = batch.recover()
    check_all(*files, *[g for g3 in gs for g in g3], *go)
    for f, o in zip(files, outs):
        assert torch.equal(o, f.view)
    assert (reps.cpu().numpy() == np.array([-1, 0])).all()


@pytest.mark.parametrize("level", [1, 2])
def test_dct_guards(dev, level):
    Wd, Hd = 136, 40
    img_np = synth.bitmap(Hd, Wd, 1, 5).reshape(-1)
    img = gin(img_np, dev)
    lay = se.dct_layout(Wd, Hd, 1, level)
    a, p = gout(lay["a_bytes"], dev), gout(lay["p_bytes"], dev)
    se.dct_protect(img.view, Wd, Hd, 1, level, KEY, IV, out=(a.view, p.view))
    o = gout(lay["p_bytes"], dev)
    se.dct_recover(a.view, p.view, Wd, Hd, 1, level, KEY, IV, out=o.view)
    f = gout(lay["p_bytes"], dev, torch.float32)
    se.dct8_forward(img.view, Wd, Hd, 1, out=f.view)
    i8 = gout(lay["p_bytes"], dev)
    se.dct8_inverse(f.view, Wd, Hd, 1, out=i8.view)
    check_all(img, a, p, o, f, i8)
    assert int((o.view.int() - img.view.int()).abs().max()) <= 8       # lossy by design (~60 dB)
    assert int((i8.view.int() - img.view.int()).abs().max()) <= 1


@pytest.mark.parametrize("n,W,L,world", [(256 * 256 + 77, 256, 2, 3), (1024 * 200, 1024, 3, 2)])
def test_full_stripe_guards(dev, n, W, L, world):
    """FULL-mode stripes with halo rows: each stripe's source window, slices,
    workspace and recovered bytes are guarded; the stripes reassemble the file."""
    from paper_1803_04880_b200 import shard
    x_np = synth.random_bytes(n, 11 * n)
    plan = [s for s in shard.plan_full_stripes(n, W, L, world) if s is not None]
    frags = {k: [] for k in "abc"}
    for st in plan:
        src = gin(x_np[st["src_byte_begin"]: st["src_byte_end"]], dev)
        sizes = [st["out"][k][1] - st["out"][k][0] for k in "abc"]
        outs = [gout(s, dev) for s in sizes]
        stripe = (st["row_begin"], st["row_end"], st["src_row0"], min(-(-src.n // W), st["src_rows"]))
        ws = gout(se.fragment_workspace_size(n, W, L, se.MODE_FULL, stripe), dev)
        se.fragment_protect_stripe(src.view, n, W, L, KEY, IV, st["row_begin"], st["row_end"], st["src_row0"],
                                   out=tuple(o.view for o in outs), workspace=ws.view)
        check_all(src, ws, *outs)
        for k, o in zip("abc", outs):
            frags[k].append(o.view.cpu().numpy())
    whole = {k: np.concatenate(v) for k, v in frags.items()}
    back = []
    for st in plan:
        ins = [gin(whole[k][slice(*st["rec_in"][k])], dev) for k in "abc"]
        nb = st["byte_end"] - st["byte_begin"]
        out, rep = gout(nb, dev), gout(2, dev, torch.int64)
        stripe = (st["row_begin"], st["row_end"], st["rec_row0"], st["rec_rows"])
        ws = gout(se.fragment_workspace_size(n, W, L, se.MODE_FULL, stripe), dev)
        se.fragment_recover_stripe(*(i.view for i in ins), n, W, L, KEY, IV, st["row_begin"], st["row_end"],
                                   st["rec_row0"], st["rec_rows"], out=out.view, report=rep.view, workspace=ws.view)
        check_all(*ins, out, rep, ws)
        assert rep.view.cpu().tolist() == [-1, 0]
        back.append(out.view.cpu().numpy())
    assert np.array_equal(np.concatenate(back), x_np)


class HostGuarded:
    """A pinned host uint8 view of n bytes with guard bands (16-byte aligned)."""

    def __init__(self, n, fill=None):
        self.raw = torch.full((2 * G + n,), PAT, dtype=torch.uint8).pin_memory()
        self.n = n
        self.view = self.raw[G:G + n]
        if fill is not None:
            self.view.copy_(torch.from_numpy(fill))

    def guards_ok(self):
        torch.cuda.synchronize()
        return bool((self.raw[:G] == PAT).all()) and bool((self.raw[G + self.n:] == PAT).all())


@pytest.mark.parametrize("n,W,chunk", [(300000, 512, 64 * 1024), (6144 * 8 * 9 + 5, 6144, 0), (999, 8, 0)])
@pytest.mark.parametrize("asyn", [False, True])
def test_host_api_guards(dev, n, W, chunk, asyn):
    """Host streaming (staged chunks; protect's kernels write the fragments
    straight into the pinned buffers): nothing outside the host views changes."""
    L = 2
    x_np = synth.random_bytes(n, 5 * n + 1)
    x = HostGuarded(n, x_np)
    lay = se.fragment_layout(n, W, L)
    a, b, c = (HostGuarded(lay[k]) for k in ("a_bytes", "b_bytes", "c_bytes"))
    y = HostGuarded(n)
    kw = dict(chunk_bytes=chunk, n_streams=3)
    if asyn:
        _, t1 = se.fragment_protect_host_async(x.view, W, L, KEY, IV, out=(a.view, b.view, c.view), **kw)
        _, t2 = se.fragment_recover_host_async(a.view, b.view, c.view, n, W, L, KEY, IV, out=y.view, after=t1, **kw)
        rep = t2.wait()
        t1.wait()
    else:
        se.fragment_protect_host(x.view, W, L, KEY, IV, out=(a.view, b.view, c.view), **kw)
        _, rep = se.fragment_recover_host(a.view, b.view, c.view, n, W, L, KEY, IV, out=y.view, **kw)
    for i, h in enumerate((x, a, b, c, y)):
        assert h.guards_ok(), f"host guard band of buffer {i} overwritten"
    assert np.array_equal(x.view.numpy(), x_np) and np.array_equal(y.view.numpy(), x_np)
    assert tuple(rep) == (-1, 0)
