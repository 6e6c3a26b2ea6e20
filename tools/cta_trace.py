"""CTA timeline of the fused kernels (diagnostic build with -DSE_TRACE).

  python -c "import paper_1803_04880_b200 as se; se.build(force=True, defines=('SE_TRACE',), out='variants/v_trace.so')"
  SE_LIB_PATH=variants/v_trace.so python tools/cta_trace.py

Runs C2 protect and recover (masked) a few times, then prints, for the last
call of each, the kernel span, the start-time spread of the first wave, the
per-SM busy fraction and the tail (time after the median SM finished).
"""
import ctypes

import numpy as np
import torch

import paper_1803_04880_b200 as se
import synth

x = torch.from_numpy(synth.config_input(2)).cuda()
W, L = synth.CONFIGS[2]["width"], synth.CONFIGS[2]["levels"]
key, iv = synth.KEY, synth.iv_for(2, 0)
lib = se.lib()
fn = lib.se_trace_read
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]


def trace(n):
    buf = np.zeros(3 * n, np.uint64)
    assert fn(buf.ctypes.data, n) == 0
    t = buf.reshape(n, 3).astype(np.int64)
    return t[:, 0], t[:, 1], t[:, 2]


def report(name, n):
    sm, t0, t1 = trace(n)
    base = t0.min()
    t0, t1 = t0 - base, t1 - base
    span = t1.max()
    dur = t1 - t0
    nsm = sm.max() + 1
    busy_end = np.array([t1[sm == s].max() if (sm == s).any() else 0 for s in range(nsm)])
    first = np.sort(t0)[: nsm * 5]
    print(f"{name}: {n} CTAs, span {span / 1e3:.1f} us, CTA duration median {np.median(dur) / 1e3:.1f} us "
          f"(min {dur.min() / 1e3:.1f}, max {dur.max() / 1e3:.1f}); first {len(first)} starts within "
          f"{first.max() / 1e3:.1f} us; SM finish median {np.median(busy_end) / 1e3:.1f} us, "
          f"min {busy_end.min() / 1e3:.1f}; CTAs per SM {np.bincount(sm).min()}..{np.bincount(sm).max()}")
    hist = np.histogram(t0 / 1e3, bins=12, range=(0, span / 1e3))[0]
    print("   start histogram (12 bins over span):", hist.tolist())


fks = lib.se_trace_ks_read
fks.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = torch.empty(63 << 20, dtype=torch.int32, device="cuda")     # 252 MB > L2, as bench.py


def timed(fn):
    # as bench.py's timed loop: L2 flushed, then CUDA events around the call
    ms = []
    for k in range(5):
        flush.fill_(k)
        flush.amax()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1) * 1e3)
    return out, ms


def ks_span(n_fused):
    buf = np.zeros(3 * 4096, np.uint64)
    assert fks(buf.ctypes.data, 4096) == 0
    t = buf.reshape(-1, 3).astype(np.int64)
    t = t[t[:, 1] > 0]
    _, f0, f1 = trace(n_fused)
    base = min(t[:, 1].min(), f0.min())
    print(f"   keystream CTAs (this call): {len(t)}, span {(t[:, 1].min() - base) / 1e3:.1f}..{(t[:, 2].max() - base) / 1e3:.1f} us; "
          f"fused CTAs {(f0.min() - base) / 1e3:.1f}..{(f1.max() - base) / 1e3:.1f} us (same time base)")


nb = x.numel() // 64
BPC = int(__import__("os").environ.get("BPC", "128"))
(a, b, c), ms = timed(lambda: se.fragment_protect(x, W, L, key, iv))
print(f"protect call (events, L2 flushed): {[round(v, 1) for v in ms]} us")
report("protect", (nb + BPC - 1) // BPC)
ks_span((nb + BPC - 1) // BPC)
(y, rep), ms = timed(lambda: se.fragment_recover(a, b, c, x.numel(), W, L, key, iv))
print(f"recover call (events, L2 flushed): {[round(v, 1) for v in ms]} us")
report("recover", (nb + BPC - 1) // BPC)
ks_span((nb + BPC - 1) // BPC)
