#!/usr/bin/env python3
"""PCIe reference numbers for the e2e path: pinned H2D, D2H and concurrent
(both directions) copy bandwidth, and fragment_protect_host /
fragment_recover_host throughput vs chunk size and stream count."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


out = {}
out["h2d_gbs"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_gbs"] = n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


out["duplex_gbs_each"] = n / timed(both) / 1e9
# zero-copy: a kernel (AES-CTR, ~0.6 TB/s on device) reading pinned host
# memory / writing pinned host memory directly over PCIe
m = 64 << 20
out["zero_copy_read_gbs"] = m / timed(lambda: se.cipher_encrypt(synth.KEY, bytes(16), h[:m], out=d[:m])) / 1e9
out["zero_copy_write_gbs"] = m / timed(lambda: se.cipher_encrypt(synth.KEY, bytes(16), d[:m], out=h[:m])) / 1e9
out["zero_copy_rw_gbs"] = m / timed(lambda: se.cipher_encrypt(synth.KEY, bytes(16), h2[:m], out=h[:m])) / 1e9
if len(sys.argv) > 1 and sys.argv[1] == "zc":
    print(json.dumps(out, indent=1))
    sys.exit(0)
x = synth.config_input(2)
hx = torch.from_numpy(x).pin_memory()
lay = se.fragment_layout(x.size, 6144, 2)
frag = (se._host_empty(lay["a_bytes"]), se._host_empty(lay["b_bytes"]), se._host_empty(lay["c_bytes"]))
ho = se._host_empty(x.size)
for chunk in (1, 2, 4, 8):
    for streams in (2, 4, 8):
        def step():
            se.fragment_protect_host(hx, 6144, 2, synth.KEY, synth.iv_for(2), out=frag, chunk_bytes=chunk << 20,
                                     n_streams=streams)
            se.fragment_recover_host(*frag, x.size, 6144, 2, synth.KEY, synth.iv_for(2), out=ho,
                                     chunk_bytes=chunk << 20, n_streams=streams)
        out[f"e2e_c2_chunk{chunk}MiB_s{streams}_gbs"] = x.size / timed(step, 10) / 1e9
print(json.dumps(out, indent=1))
