#!/usr/bin/env python3
"""C2 host-API breakdown: fragment_protect_host alone, fragment_recover_host
alone, the blocking pair and the asynchronous pair, per chunk size / stream
count, next to plain pinned copies of the same bytes in the same chunks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

torch.cuda.init()
x_np, W, L = synth.config_input(2), 6144, 2
key, iv = synth.KEY, synth.iv_for(2)
x = torch.from_numpy(x_np).pin_memory()
n = x.numel()
lay = se.fragment_layout(n, W, L)
frag = tuple(se._host_empty(lay[k]) for k in ("a_bytes", "b_bytes", "c_bytes"))
y = se._host_empty(n)
fb = sum(lay[k] for k in ("a_bytes", "b_bytes", "c_bytes"))


def wall(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e6


# plain copies: the pair's PCIe traffic alone (H2D n + fb, D2H fb + n), chunked the same way, 3 streams
d_in = torch.empty(n + fb, dtype=torch.uint8, device="cuda")
h_in = torch.empty(n + fb, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n + fb, dtype=torch.uint8).pin_memory()
d_out = torch.empty(n + fb, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(6)]
for chunk in ([] if os.environ.get("NOCOPIES") else (1 << 20, 2 << 20, 4 << 20)):
    def copies():
        for k, o in enumerate(range(0, n + fb, chunk)):
            e = min(n + fb, o + chunk)
            with torch.cuda.stream(streams[k % 3]):
                d_in[o:e].copy_(h_in[o:e], non_blocking=True)
                h_out[o:e].copy_(d_out[o:e], non_blocking=True)
    t = wall(copies)
    print(f"copies only, {chunk >> 10} KiB pieces on 3 streams, both directions: {t:.0f} us "
          f"({(n + fb) / t / 1e3:.1f} GB/s each way)", flush=True)

for chunk in [int(c) << 10 for c in os.environ.get("CHUNKS", "1024 2048 4096").split()]:
    for ns in [int(c) for c in os.environ.get("STREAMS", "3 4 8").split()]:
        kw = dict(chunk_bytes=chunk, n_streams=ns)
        tp = wall(lambda: se.fragment_protect_host(x, W, L, key, iv, out=frag, **kw))
        tr = wall(lambda: se.fragment_recover_host(*frag, n, W, L, key, iv, out=y, **kw))

        def pair():
            se.fragment_protect_host(x, W, L, key, iv, out=frag, **kw)
            se.fragment_recover_host(*frag, n, W, L, key, iv, out=y, **kw)

        def apair():
            _, t1 = se.fragment_protect_host_async(x, W, L, key, iv, out=frag, **kw)
            _, t2 = se.fragment_recover_host_async(*frag, n, W, L, key, iv, out=y, after=t1, **kw)
            t2.wait()
            t1.wait()

        tq, ta = wall(pair), wall(apair)
        print(f"chunk={chunk >> 10}KiB streams={ns}: protect {tp:.0f} us, recover {tr:.0f} us, pair {tq:.0f} us "
              f"({n / tq / 1e3:.2f} GB/s), async pair {ta:.0f} us ({n / ta / 1e3:.2f} GB/s)", flush=True)
assert torch.equal(x, y)
