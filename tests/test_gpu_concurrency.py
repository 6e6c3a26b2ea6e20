"""Concurrent calls (SURVEY §5 race detection, on the path): the library keeps
no device-global scratch — keystreams live in the caller's buffers, FULL mode
in the caller's workspace — so any number of protect / recover calls may be
in flight at once on different streams.  Here 8 streams each enqueue a
different job (masked and PUBLIC_PLAIN, per-CTA and tile kernels, FULL mode,
cipher, every level) several times over without host synchronisation; every
result must equal the oracle's (a shared scratch buffer, a static device
counter or a cross-stream PDL hazard would corrupt some of them)."""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


JOBS = [   # (n, W, L, mode, flags)
    (6144 * 8 * 20 + 7, 6144, 2, 0, 0),
    (1024 * 8 * 40, 1024, 2, 0, 0),            # whole 1024-byte rows: recover keystream parked in the output
    (1024 * 8 * 33 + 100, 1024, 3, 0, 0),
    (512 * 64 * 5 + 999, 1024, 2, 0, 1),        # PUBLIC_PLAIN: tile kernels
    (256 * 8 * 40 + 3, 256, 1, 0, 1),
    (2048 * 8 * 12 + 11, 2048, 2, 1, 0),        # FULL mode, own workspace
    (777 * 8 + 5, 56, 2, 0, 0),
    (4096 * 8 * 9, 4096, 2, 0, 1),
]


def test_concurrent_streams_bit_exact(dev, orc):
    streams = [torch.cuda.Stream(device=dev) for _ in JOBS]
    inputs, expect = [], []
    for i, (n, W, L, mode, flags) in enumerate(JOBS):
        x = synth.random_bytes(n, 4242 + i)
        iv = synth.iv_for(6, i)
        inputs.append((torch.from_numpy(x).to(dev), iv))
        expect.append(orc.protect(x, W, L, KEY, iv, mode=mode, flags=flags))
    torch.cuda.synchronize()
    results = [None] * len(JOBS)
    for rnd in range(3):                        # several rounds in flight, no host sync in between
        for i, (n, W, L, mode, flags) in enumerate(JOBS):
            x, iv = inputs[i]
            s = streams[i]
            with torch.cuda.stream(s):
                ws = None
                if mode == se.MODE_FULL:
                    ws = torch.empty(se.fragment_workspace_size(n, W, L, mode), dtype=torch.uint8, device=dev)
                a, b, c = se.fragment_protect(x, W, L, KEY, iv, mode=mode, flags=flags, stream=s, workspace=ws)
                y, rep = se.fragment_recover(a, b, c, n, W, L, KEY, iv, mode=mode, flags=flags, stream=s,
                                             workspace=ws)
                e = se.cipher_encrypt(KEY, iv, x, ctr_block_offset=rnd, stream=s)
                d = se.cipher_decrypt(KEY, iv, e, ctr_block_offset=rnd, stream=s)
                results[i] = (a, b, c, y, rep, d)
    torch.cuda.synchronize()
    for i, (a, b, c, y, rep, d) in enumerate(results):
        oa, ob, oc = expect[i]
        assert np.array_equal(a.cpu().numpy(), oa), i
        assert np.array_equal(b.cpu().numpy(), ob), i
        assert np.array_equal(c.cpu().numpy(), oc), i
        assert torch.equal(y, inputs[i][0]) and rep.cpu().tolist() == [-1, 0], i
        assert torch.equal(d, inputs[i][0]), i
