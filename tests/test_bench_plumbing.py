"""bench.py's multi-rank plumbing on CPU (row d/e, VERDICT r1 "missing" 1):
the max-over-ranks reduction on every backend branch, the --gpus / WORLD_SIZE
check, and the config dict both arms print (the driver pairs the repo arm
and the reference arm by it)."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_allreduce_max_nccl_branch_calls_all_reduce_once(monkeypatch):
    """The non-gloo branch must reduce (round 1 recursed into itself)."""
    import torch
    import torch.distributed as dist
    calls = []
    monkeypatch.setattr(dist, "get_backend", lambda *a, **k: "nccl")

    def fake_all_reduce(t, op=None):
        calls.append(op)
        t.fill_(7.0)
    monkeypatch.setattr(dist, "all_reduce", fake_all_reduce)
    t = torch.tensor([1.0, 2.0], dtype=torch.float64)
    assert bench.allreduce_max(t) is t
    assert calls == [dist.ReduceOp.MAX] and t.tolist() == [7.0, 7.0]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([float(rank + 1), 10.0 - rank], dtype=torch.float64)
    bench.allreduce_max(t)
    q.put((rank, t.tolist()))
    dist.destroy_process_group()


def test_allreduce_max_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: [2.0, 10.0], 1: [2.0, 10.0]}


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_default_config_is_the_1GiB_file():
    args = bench.argparse.Namespace(config=4, plain=False)
    d1 = bench.config_dict(args, 1)
    d8 = bench.config_dict(args, 8)
    assert d1["workload"].startswith("C4-1GiB") and d1["n_bytes"] == 1 << 30
    assert d8["n_bytes"] == 1 << 30                      # strong scaling: one file cut into stripes
    a2 = bench.argparse.Namespace(config=2, plain=True)
    assert bench.config_dict(a2, 4)["n_bytes"] == 4 * 6144 * 2048      # weak: one file per rank
    import inspect
    src = inspect.getsource(bench.main)
    assert "default=4" in src


def test_reference_arm_config_identical_to_repo_arm(monkeypatch):
    """Both arms build `config` from the same function (C1: small enough to run here)."""
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")
    args = bench.argparse.Namespace(config=1, plain=False, steps=1, warmup=1)
    line = bench.run_reference(args)
    assert line["config"] == bench.config_dict(args, 1)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
