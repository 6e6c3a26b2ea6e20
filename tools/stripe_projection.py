#!/usr/bin/env python3
"""Strong-scaling projection for C4 (the 1 GiB file split into N row stripes)
from ONE GPU: for N = 1, 2, 4, 8, time every stripe's protect + recover
exactly as a rank of `bench.py --gpus N` runs it (same plan, same
block_offset, L2 flushed between steps, CUDA events), and report
N x bytes of the slowest stripe / its time — what N independent GPUs would
reach if nothing but the per-GPU work limited them (no collective is on the
path).  Not a multi-GPU measurement: the driver's SCALE run is.

  python tools/stripe_projection.py > gpurun_out/stripes.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402
from paper_1803_04880_b200 import shard  # noqa: E402

dev = torch.device("cuda:0")
c = synth.CONFIGS[4]
W, L, N_BYTES = c["width"], c["levels"], c["n_bytes"]
full = synth.config_input(4)
key, iv = synth.KEY, synth.iv_for(4)
flush = torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.int32, device=dev)
steps, warm = int(os.environ.get("STEPS", "10")), 3
out = {"what": __doc__.strip().splitlines()[0], "config": "C4-1GiB-file-L2", "runs": []}
for world in (1, 2, 4, 8):
    per = []
    for rank, p in enumerate(shard.plan_stripes(N_BYTES, W, L, world)):
        x = torch.from_numpy(full[p["byte_begin"]: p["byte_end"]].copy()).to(dev)
        n = x.numel()
        lay = se.fragment_layout(n, W, L, block_offset=p["block_offset"])
        a, b, cc = (se._empty(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
        y = se._empty(n, dev)
        rep = torch.empty(2, dtype=torch.int64, device=dev)
        ms = []
        for k in range(warm + steps):
            bench.l2_flush(flush, k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            se.fragment_protect(x, W, L, key, iv, block_offset=p["block_offset"], out=(a, b, cc))
            se.fragment_recover(a, b, cc, n, W, L, key, iv, block_offset=p["block_offset"], out=y, report=rep)
            e1.record()
            torch.cuda.synchronize()
            if k >= warm:
                ms.append(e0.elapsed_time(e1))
        assert torch.equal(y, x) and rep.cpu().tolist() == [-1, 0]
        per.append({"rank": rank, "bytes": n, "ms": sum(ms) / len(ms)})
        del x, a, b, cc, y
    slow = max(per, key=lambda r: r["ms"])
    value = N_BYTES / (slow["ms"] / 1e3) / 1e9          # all N stripes in the slowest stripe's time
    out["runs"].append({"n_gpus": world, "projected_gbs": round(value, 2),
                        "slowest_stripe_ms": round(slow["ms"], 4),
                        "per_stripe_ms": [round(r["ms"], 4) for r in per]})
base = out["runs"][0]["projected_gbs"]
for r in out["runs"]:
    r["speedup_vs_1"] = round(r["projected_gbs"] / base, 3)
print(json.dumps(out, indent=1))
