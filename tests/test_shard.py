"""Multi-GPU partitioning (row e) on CPU: the stripe / file planners, and a
world_size-2 gloo run where each rank protects its stripe and the gathered
streams must equal the single-process streams byte for byte (the oracle
stands in for the GPU here; tests/test_gpu_parity.py checks the same
invariant through libse.so on one GPU)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import synth
from paper_1803_04880_b200 import shard

KEY = synth.KEY
IV = bytes.fromhex("00112233445566778899aabbccddeeff")


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_block_align(levels):
    g = shard.block_align(levels)
    a, b, c = shard.BITS[levels]
    assert (g * a) % 128 == 0 and (g * b) % 8 == 0 and (g * c) % 8 == 0
    assert all((h * a) % 128 or (h * b) % 8 or (h * c) % 8 for h in range(1, g))


@pytest.mark.parametrize("n,W,L,world", [(1 << 20, 1024, 2, 8), (6144 * 2048, 6144, 2, 3), ((1 << 20) + 77, 256, 3, 4),
                                         (5000, 64, 1, 8), (100, 8, 2, 4), (0, 8, 2, 2)])
def test_plan_stripes_cover_and_align(orc, n, W, L, world):
    lay = orc.layout(n, W, L)
    plan = shard.plan_stripes(n, W, L, world)
    assert len(plan) == world
    assert plan[0]["byte_begin"] == 0 and plan[-1]["byte_end"] == n
    total = 0
    for p, q in zip(plan, plan[1:]):
        assert p["byte_end"] == q["byte_begin"]
        for s in "abc":
            assert p[s][1] == q[s][0]
    for p in plan:
        assert p["block_offset"] % shard.block_align(L) == 0 or p["n_blocks"] == 0
        total += p["n_blocks"]
        sub = orc.layout(p["byte_end"] - p["byte_begin"], W, L)
        assert sub["n_blocks"] == p["n_blocks"]
    assert total == lay["n_blocks"]
    assert plan[-1]["a"][1] == lay["a_bytes"] and plan[-1]["c"][1] == lay["c_bytes"]


@pytest.mark.parametrize("n,W,L,world", [(64 * 1024 + 333, 128, 2, 3), (40000, 64, 3, 2), (30000, 32, 1, 4)])
def test_stripes_concatenate_to_whole_file(orc, n, W, L, world):
    x = synth.random_bytes(n, n)
    whole = orc.protect(x, W, L, KEY, IV)
    parts = [[], [], []]
    for p in shard.plan_stripes(n, W, L, world):
        part = x[p["byte_begin"]: p["byte_end"]]
        streams = orc.protect(part, W, L, KEY, IV, block_offset=p["block_offset"])
        for s in range(3):
            parts[s].append(streams[s])
            lo, hi = p["abc"[s]]
            assert len(streams[s]) == hi - lo
    for s in range(3):
        assert np.array_equal(np.concatenate(parts[s]), whole[s])


def test_plan_files_lpt_balance():
    sizes = synth.c5_file_sizes(10000, 5)
    for world in (1, 2, 4, 8):
        plan = shard.plan_files(sizes, world)
        assert sorted(i for r in plan for i in r) == list(range(len(sizes)))
        loads = [int(sizes[r].sum()) for r in map(np.array, plan)]
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(loads) / world + int(sizes.max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, n, W, L, result_path):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = synth.random_bytes(n, 123)                      # every rank holds the file (or its stripe)
    p = shard.plan_stripes(n, W, L, world)[rank]
    streams = oracle.protect(x[p["byte_begin"]: p["byte_end"]], W, L, KEY, IV, block_offset=p["block_offset"])
    gathered = []
    for s in range(3):
        t = torch.from_numpy(np.ascontiguousarray(streams[s]).copy())
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([t.numel()], dtype=torch.int64))
        mx = int(max(v.item() for v in sizes))
        buf = torch.zeros(mx, dtype=torch.uint8)
        buf[: t.numel()] = t
        bufs = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(bufs, buf)
        gathered.append(np.concatenate([b[: int(sz.item())].numpy() for b, sz in zip(bufs, sizes)]))
    if rank == 0:
        whole = oracle.protect(x, W, L, KEY, IV)
        ok = all(np.array_equal(g, w) for g, w in zip(gathered, whole))
        with open(result_path, "w") as f:
            f.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_stripes(tmp_path):
    import torch.multiprocessing as mp
    result = str(tmp_path / "result.txt")
    mp.spawn(_rank_main, args=(2, _free_port(), 8 * 1024 * 9 + 500, 1024, 2, result), nprocs=2, join=True)
    assert open(result).read() == "ok"


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("n,W,world", [(256 * 200 + 77, 256, 3), (32768 * 64, 32768, 8), (1024 * 96, 1024, 5),
                                       (64 * 1000 + 3, 64, 2)])
def test_plan_full_stripes_windows(orc, n, W, L, world):
    """FULL stripes: rows partition the matrix; protect windows add 2(2^L-1)
    halo rows per side (clipped); recover windows add whole halo block rows
    and start on CTR/byte-aligned block rows; output slices tile the whole
    FULL streams (oracle layout)."""
    lay = orc.layout(n, W, L, orc.MODE_FULL)
    plan = [s for s in shard.plan_full_stripes(n, W, L, world) if s is not None]
    halo = 2 * ((1 << L) - 1)
    assert plan[0]["row_begin"] == 0 and plan[-1]["row_end"] == lay["rows"]
    for s0, s1 in zip(plan, plan[1:]):
        assert s0["row_end"] == s1["row_begin"]
    bits = dict(zip("abc", shard.FULL_BITS[L]))
    for st in plan:
        assert st["src_row0"] == max(0, st["row_begin"] - halo)
        assert st["src_row0"] + st["src_rows"] == min(lay["rows"], st["row_end"] + halo)
        r0 = st["rec_row0"]
        assert r0 <= max(0, st["row_begin"] - 8 * -(-halo // 8)) and r0 % 8 == 0
        assert r0 + st["rec_rows"] >= min(lay["rows"], st["row_end"] + 8 * -(-halo // 8))
        blocks_before = r0 // 8 * (W // 8)
        assert (blocks_before * bits["a"]) % 128 == 0
        assert all((blocks_before * b) % 8 == 0 for b in bits.values())
    for k in "abc":
        assert plan[0]["out"][k][0] == 0 and plan[-1]["out"][k][1] == lay[f"{k}_bytes"]
        for s0, s1 in zip(plan, plan[1:]):
            assert s0["out"][k][1] == s1["out"][k][0]
