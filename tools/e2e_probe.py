#!/usr/bin/env python3
"""Wall time of fragment_protect_host and fragment_recover_host alone (pinned
buffers) on C2 and a 256 MiB slice of C4, per chunk size / stream count, next
to the PCIe model (input + fragments at the measured copy rates)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_04880_b200 as se  # noqa: E402
import synth  # noqa: E402

torch.cuda.init()
for name, x_np, W in (("C2", synth.config_input(2), 6144), ("C4/4", synth.random_bytes(1 << 28, 4), 1024)):
    x = torch.from_numpy(x_np).pin_memory()
    n = x.numel()
    lay = se.fragment_layout(n, W, 2)
    frag = tuple(se._host_empty(lay[k]) for k in ("a_bytes", "b_bytes", "c_bytes"))
    y = se._host_empty(n)
    for chunk in (4 << 20, 8 << 20, 16 << 20):
        for ns in (3, 4, 6):
            for _ in range(3):
                se.fragment_protect_host(x, W, 2, synth.KEY, synth.iv_for(2), out=frag, chunk_bytes=chunk, n_streams=ns)
                se.fragment_recover_host(*frag, n, W, 2, synth.KEY, synth.iv_for(2), out=y, chunk_bytes=chunk,
                                         n_streams=ns)
            reps = 10 if n < (1 << 26) else 3
            t0 = time.perf_counter()
            for _ in range(reps):
                se.fragment_protect_host(x, W, 2, synth.KEY, synth.iv_for(2), out=frag, chunk_bytes=chunk, n_streams=ns)
            t1 = time.perf_counter()
            for _ in range(reps):
                se.fragment_recover_host(*frag, n, W, 2, synth.KEY, synth.iv_for(2), out=y, chunk_bytes=chunk,
                                         n_streams=ns)
            t2 = time.perf_counter()
            tp, tr = (t1 - t0) / reps * 1e6, (t2 - t1) / reps * 1e6
            print(f"{name} chunk={chunk >> 20}MiB streams={ns}: protect {tp:.0f} us ({n / tp / 1e3:.1f} GB/s), "
                  f"recover {tr:.0f} us ({n / tr / 1e3:.1f} GB/s); D2H-bound model "
                  f"{1.258 * n / 47.5e3:.0f} us", flush=True)
    assert torch.equal(x, y)
