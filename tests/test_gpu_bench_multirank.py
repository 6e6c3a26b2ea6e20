"""The multi-rank code paths of bench.py (row e) on the one-GPU box: launched
as the driver launches them (torch.distributed.run, one process per rank,
127.0.0.1 rendezvous) with the test-only SE_BENCH_TEST_GLOO=1 switch (gloo
for the barrier / max-over-ranks, ranks sharing the GPU; their kernels never
wait on one another).  Not a performance number: it checks that every rank
exits 0 and rank 0 alone prints one well-formed JSON line."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [["--steps", "1"], ["--config", "2"], ["--config", "1", "--impl", "reference"]])
def test_two_ranks_print_one_line(extra):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-comparator", "--e2e-steps", "0",
           "--soak", "0"] + extra
    env = dict(os.environ, SE_BENCH_TEST_GLOO="1")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] in (1, 2) and d["warmup"] == 3
    assert d["scaling"] in ("weak", "strong")


def _nccl_worker(port):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    t = torch.tensor([3.0, 5.0], dtype=torch.float64, device=dev)
    bench.allreduce_max(t)
    torch.cuda.synchronize()
    assert t.tolist() == [3.0, 5.0]
    dist.destroy_process_group()


def test_allreduce_max_inside_a_real_nccl_group():
    """bench.allreduce_max on a CUDA tensor in an NCCL process group (the
    branch round 1 never ran: it recursed)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = torch.multiprocessing.get_context("spawn")
    p = ctx.Process(target=_nccl_worker, args=(free_port(),))
    p.start()
    p.join(timeout=300)
    assert p.exitcode == 0
