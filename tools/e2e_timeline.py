#!/usr/bin/env python3
"""GPU timeline (CUPTI via torch.profiler) of the C2 host-API pair: every
memcpy and kernel of fragment_protect_host(_async) + fragment_recover_host(_async),
printed as start / end offsets per stream, to see where the pipeline idles."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

x_np, W, L = synth.config_input(2), 6144, 2
key, iv = synth.KEY, synth.iv_for(2)
x = torch.from_numpy(x_np).pin_memory()
n = x.numel()
lay = se.fragment_layout(n, W, L)
frag = tuple(se._host_empty(lay[k]) for k in ("a_bytes", "b_bytes", "c_bytes"))
y = se._host_empty(n)
out = os.environ.get("OUT", "gpurun_out")
for chunk in [int(c) << 10 for c in os.environ.get("CHUNKS", "4096 1024").split()]:
    for mode in ("sync", "async"):
        kw = dict(chunk_bytes=chunk, n_streams=3)

        def run():
            if mode == "sync":
                se.fragment_protect_host(x, W, L, key, iv, out=frag, **kw)
                se.fragment_recover_host(*frag, n, W, L, key, iv, out=y, **kw)
            else:
                _, t1 = se.fragment_protect_host_async(x, W, L, key, iv, out=frag, **kw)
                _, t2 = se.fragment_recover_host_async(*frag, n, W, L, key, iv, out=y, after=t1, **kw)
                t2.wait()
                t1.wait()

        for _ in range(5):
            run()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            run()
            torch.cuda.synchronize()
        path = f"{out}/tl_{mode}_{chunk >> 10}.json"
        prof.export_chrome_trace(path)
        ev = [e for e in json.load(open(path))["traceEvents"]
              if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
        ev.sort(key=lambda e: e["ts"])
        t0 = ev[0]["ts"]
        print(f"== {mode} chunk {chunk >> 10} KiB: span {max(e['ts'] + e['dur'] for e in ev) - t0:.0f} us, {len(ev)} ops")
        for e in ev:
            nm = e["name"][:60]
            print(f"  {e['ts'] - t0:8.1f} {e['ts'] - t0 + e['dur']:8.1f}  s{e['args'].get('stream', '?'):<4} {nm}")
