#!/usr/bin/env python3
"""bench.py — protect+recover throughput of the agnostic SE hot path on B200.

Contract (see task / DESIGN.md §6):
  python bench.py [--gpus N --steps K --warmup W] [--config 2] [--impl se|reference]
One step = one pass of the whole hot path (fused
protect, then fused recover) over one synthetic input resident in HBM.  The
metric is BASELINE.json's: input GB/s through protect+recover, whole job, and
the dominant kernel's fraction of its roofline.  Under torchrun each rank
processes its own independent file (weak scaling, no data-path collective);
NCCL is used only for the barrier and the max-over-ranks of the timings.

--impl reference times the CPU oracle (oracle/, plain C) on the host cores on
a bounded sample of the same workload — the paper-defined computation, as it
stands; it is a reported baseline, not a target.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_BYTES = 126 * (1 << 20)


def l2_flush(buf, k: int):
    """Evict L2 between timed steps: write a buffer of 2x L2, then read it back,
    so the dirty lines of the write are written back here, outside the timed
    region, instead of inside the next timed kernel."""
    buf.fill_(k)
    buf.amax()

# ---------------------------------------------------------------- roofline model
# Algorithmic ALU-pipe operations per 8x8 block: the shift /
# rotate / logic operations (SHF, LOP3, PRMT class) the method needs in a
# minimal 32-bit mapping.  Adds are excluded (they may issue on the FMA pipe
# as IMAD), so these ops alone set a lower bound on ALU-pipe cycles.
#   SHA-256 rounds 8..63 (host midstate covers 0..7):  8*10 + 48*18 = 944
#   SHA-512 rounds 4..79 (host midstate covers 0..3): 12*20 + 64*36 = 2544,
#     less what the launch-constant schedule (sha2_spec.cuh) removes: 8 ops per
#     sigma not evaluated in W16..W31 (18 at L = 2, 17 at L = 1, 3) and the low
#     half of K_t + W_t for the block-independent W_t (12 / 11 / 11 rounds)
#   5/3 lifting shifts: L1 16 lifts*8 + L2 8 lifts*4 (+ L3 4 lifts*2) = 160 (168)
#   byte unpack 64; field pack/unpack ~2 per field + word splits = 140
#   mask XORs: B + C words = 19;  AES-CTR: 260 ops per AES block * a_bits/128
ALU_OPS = {
    1: {"sha256": 0, "sha512": 2544 - 8 * 17 - 11, "dwt": 128 + 64, "pack": 140, "xor": 15, "aes": 260 * 160 / 128},
    2: {"sha256": 944, "sha512": 2544 - 8 * 18 - 12, "dwt": 160 + 64, "pack": 140, "xor": 19, "aes": 260 * 40 / 128},
    3: {"sha256": 944, "sha512": 2544 - 8 * 17 - 11, "dwt": 168 + 64, "pack": 140, "xor": 20, "aes": 260 * 10 / 128},
}
ALU_LANES_PER_SM_CLK = 64      # guide fallback (B300_MICROARCH.md); measured value: alu_lanes_per_clk()
NUM_SMS = 148


def alu_ops_per_block(levels: int, masked: bool) -> float:
    d = ALU_OPS[levels]
    ops = d["dwt"] + d["pack"] + d["aes"]
    if masked:
        ops += d["sha256"] + d["sha512"] + d["xor"]
    return float(ops)


def _profile_entries():
    """Per-(kernel, workload) ncu summaries committed under profiles/
    (round*_traffic.json: {"entries": [{"kernel", "workload", "dram_bytes",
    "inst_per_block", "source"}]}), newest round first."""
    import glob
    out = []
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "round*_traffic.json")), reverse=True):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        for e in d.get("entries", []):
            out.append(dict(e, file=os.path.basename(f)))
    return out


def load_traffic(kernel_key: str, workload: str):
    """DRAM bytes per launch of `kernel_key` on `workload` from the newest
    committed ncu capture of exactly that pair, else (None, None)."""
    for e in _profile_entries():
        if e.get("kernel") == kernel_key and e.get("workload") == workload and e.get("dram_bytes"):
            return e["dram_bytes"], f"{e['file']}: {e.get('source', '')}"
    return None, None


def load_profile_stats(kernel_key: str, workload: str):
    for e in _profile_entries():
        if e.get("kernel") == kernel_key and e.get("workload") == workload:
            return e
    return None


def alu_lanes_per_clk():
    """ALU-pipe lane operations per SM clock: measured by tools/intbench.cu
    (profiles/round2_intpeak.json: SHF / LOP3 chains, SM cycles from clock64),
    else the microarchitecture guide's 64."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "round2_intpeak.json")))
        return float(d["alu_lanes_per_clk_per_sm"]), "measured: profiles/round2_intpeak.json"
    except (OSError, ValueError, KeyError):
        return float(ALU_LANES_PER_SM_CLK), "guide value (no measurement committed)"


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------- clocks sampler

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 10:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(s):
            try:
                return float(s)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[3]) or 0) > 0] or self.rows
        sm = [num(r[1]) for r in loaded if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in loaded:
            for name, v in zip(names, r[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(loaded[0][2]),
                "reasons": sorted(reasons), "samples": len(loaded),
                "power_w_max": max((num(r[4]) or 0) for r in loaded)}


# ---------------------------------------------------------------- distributed plumbing

def init_dist(local: int):
    """One process per GPU over NCCL (barrier + max-over-ranks timing only).
    SE_BENCH_TEST_GLOO=1 (test only): gloo, ranks sharing the visible GPUs
    round-robin - exercises the multi-rank code path on a one-GPU box; the
    ranks' kernels never wait on one another (independent inputs)."""
    import torch
    import torch.distributed as dist
    if os.environ.get("SE_BENCH_TEST_GLOO") == "1":
        dev = torch.device(f"cuda:{local % torch.cuda.device_count()}")
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")
        return dev
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    return dev


def allreduce_max(t):
    """In-place max over ranks of a small float64 tensor: NCCL reduces the
    device tensor directly; gloo (CPU tests) through a host copy."""
    import torch.distributed as dist
    if dist.get_backend() == "gloo" and t.device.type != "cpu":
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg: int):
    c = synth.CONFIGS[cfg]
    x = synth.config_input(cfg)
    return c, x


def config_dict(args, world: int) -> dict:
    """The `config` of the JSON line: identical for the repo arm and the
    reference arm (same workload, same keys), so the driver can pair them."""
    c = synth.CONFIGS[args.config]
    stripes = args.config == 4
    return {"workload": c["name"] + (" (PUBLIC_PLAIN)" if args.plain else ""),
            "n_bytes": c["n_bytes"] * (1 if stripes else world), "width": c["width"], "levels": c["levels"],
            "mode": "BLOCK8", "masks": "none (C26)" if args.plain else "SHA-256 on B, SHA-512 on C",
            "parallelism": (f"dp{world}: one row stripe of the file per rank" if stripes else
                            f"dp{world}: one independent file per rank"),
            "l2": ("input 1 GiB > L2; L2 flushed between steps anyway" if stripes else
                   "flushed between steps (2x L2 write + read-back)")}


def local_input(args, rank: int, world: int):
    """This rank's share of the workload: C4 = one row stripe of the 1 GiB
    file (shard.plan_stripes: block_offset = global index of its first block;
    strong scaling); C1-C3 = an independent file per rank (own IV; weak)."""
    from paper_1803_04880_b200 import shard
    c = synth.CONFIGS[args.config]
    W, L = c["width"], c["levels"]
    if args.config == 4:
        plan = shard.plan_stripes(c["n_bytes"], W, L, world)[rank]
        x_np = np.ascontiguousarray(synth.config_input(4)[plan["byte_begin"]: plan["byte_end"]])
        return x_np, W, L, synth.iv_for(4), plan["block_offset"], "strong"
    return synth.config_input(args.config), W, L, synth.iv_for(args.config, rank), 0, "weak"


# ---------------------------------------------------------------- our arm

def run_se(args):
    """Configs 1-4 (BLOCK8).  One step = fragment_protect + fragment_recover
    of this rank's input, device-resident."""
    import torch
    import torch.distributed as dist

    import paper_1803_04880_b200 as se

    rank, world, local = dist_env()
    dev = init_dist(local) if world > 1 else torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    se.lib()
    x_np, W, L, iv, boff, scaling = local_input(args, rank, world)
    n = x_np.size
    key = synth.KEY
    flags = se.FLAG_PUBLIC_PLAIN if args.plain else 0
    masked = not args.plain
    lay = se.fragment_layout(n, W, L, block_offset=boff)
    stream = torch.cuda.Stream(device=dev)
    x = torch.from_numpy(x_np).to(dev)
    a = se._empty(lay["a_bytes"], dev)
    b = se._empty(lay["b_bytes"], dev)
    cc = se._empty(lay["c_bytes"], dev)
    out = se._empty(n, dev)
    rep = torch.empty(2, dtype=torch.int64, device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)   # 252 MB > L2
    torch.cuda.synchronize()

    def protect():
        se.fragment_protect(x, W, L, key, iv, flags=flags, block_offset=boff, out=(a, b, cc), stream=stream)

    def recover():
        se.fragment_recover(a, b, cc, n, W, L, key, iv, flags=flags, block_offset=boff, out=out, report=rep,
                            stream=stream)

    # correctness of the timed configuration (cheap property at full size)
    with torch.cuda.stream(stream):
        protect()
        recover()
    stream.synchronize()
    assert torch.equal(out, x), "recover(protect(x)) != x in the timed configuration"
    assert rep.cpu().tolist() == [-1, 0]

    clocks = ClockSampler(dev.index if dev.index is not None else local)
    clocks.start()
    # warm-up: at least W steps and ~soak s of sustained load (clock sampling)
    t_end = time.time() + args.soak
    i = 0
    with torch.cuda.stream(stream):
        while i < args.warmup or time.time() < t_end:
            protect()
            recover()
            i += 1
    stream.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    se.launch_count(reset=True)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            l2_flush(flush, k)                                  # evict L2 between timed steps
            ev[k][0].record(stream)
            protect()
            ev[k][1].record(stream)
            recover()
            ev[k][2].record(stream)
    stream.synchronize()
    launches = se.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.stop()
    t_prot = [e[0].elapsed_time(e[1]) for e in ev]          # ms
    t_rec = [e[1].elapsed_time(e[2]) for e in ev]
    mp, mr = sum(t_prot) / args.steps, sum(t_rec) / args.steps
    t = torch.tensor([mp + mr, mp, mr], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce_max(t)                                    # max over ranks
    ms_step, mp_max, mr_max = (float(v) for v in t.tolist())

    # ---- the PUBLIC_PLAIN measurement mode (C26) on the same input in the same
    #      run: the HBM-bound sub-path (transform + split + AES), reported beside
    #      the masked headline with its own roofline
    variants = {}
    if masked and not args.no_variants:
        pflags = flags | se.FLAG_PUBLIC_PLAIN
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                se.fragment_protect(x, W, L, key, iv, flags=pflags, block_offset=boff, out=(a, b, cc), stream=stream)
                se.fragment_recover(a, b, cc, n, W, L, key, iv, flags=pflags, block_offset=boff, out=out,
                                    report=rep, stream=stream)
        stream.synchronize()
        assert torch.equal(out, x) and rep.cpu().tolist() == [-1, 0], "PUBLIC_PLAIN round trip"
        pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                l2_flush(flush, k)
                pev[k][0].record(stream)
                se.fragment_protect(x, W, L, key, iv, flags=pflags, block_offset=boff, out=(a, b, cc), stream=stream)
                pev[k][1].record(stream)
                se.fragment_recover(a, b, cc, n, W, L, key, iv, flags=pflags, block_offset=boff, out=out,
                                    report=rep, stream=stream)
                pev[k][2].record(stream)
        stream.synchronize()
        pp = sum(e[0].elapsed_time(e[1]) for e in pev) / args.steps
        pr = sum(e[1].elapsed_time(e[2]) for e in pev) / args.steps
        tv = torch.tensor([pp + pr, pp, pr], dtype=torch.float64, device=dev)
        if world > 1:
            allreduce_max(tv)
        pms, pp_max, pr_max = (float(v) for v in tv.tolist())
        pdom, pdom_ms = ("k_tile_protect", pp) if pp >= pr else ("k_tile_recover", pr)
        pkey = f"k_tile<{L}, 0, {0 if pdom == 'k_tile_protect' else 1}>"
        variants["public_plain"] = {
            "what": "PUBLIC_PLAIN (C26): B and C left unmasked, transform + split + AES-CTR on A only; "
                    "same input, same run, L2 flushed between steps",
            "value": None, "unit": "GB/s", "ms_per_step": round(pms, 5),
            "kernels_ms": {"protect": round(pp, 5), "recover": round(pr, 5)},
            "max_over_ranks_ms": {"protect": round(pp_max, 5), "recover": round(pr_max, 5)},
            "_dom": (pkey, pdom_ms)}

    # ---- e2e: same metric through the public host API (pinned host buffers,
    #      H2D of the inputs and D2H of the results inside the timed region)
    e2e = run_e2e(se, torch, x_np, W, L, key, iv, flags | (se.FLAG_HOST_MAPPED if args.e2e_mapped else 0), dev,
                  args.e2e_steps, chunk_bytes=args.e2e_chunk_kib << 10, n_streams=args.e2e_streams,
                  block_offset=boff, world=world) if args.e2e_steps > 0 else \
        {"value": None, "unit": "GB/s", "note": "skipped (--e2e-steps 0, profiling runs only)"}
    if args.e2e_steps > 0:      # the asynchronous pair, recover chunk-pipelined behind protect, for comparison
        e2e["pipelined_variant"] = run_e2e(se, torch, x_np, W, L, key, iv, flags, dev, args.e2e_steps,
                                           chunk_bytes=args.e2e_chunk_kib << 10, n_streams=args.e2e_streams,
                                           block_offset=boff, world=world, pipelined=True)

    # ---- comparator: AES-128-CTR over all input bytes on the same GPU (paper methodology)
    aes_gbs = None
    if not args.no_comparator:
        y = torch.empty_like(x)
        with torch.cuda.stream(stream):
            for _ in range(3):
                se.cipher_encrypt(key, iv, x, out=y, stream=stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record(stream)
            for _ in range(reps):
                se.cipher_encrypt(key, iv, x, out=y, stream=stream)
            e1.record(stream)
        stream.synchronize()
        aes_gbs = n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
        del y

    # ---- NEXT row f2: security battery on the protected public fragment C' vs the original
    battery = None
    if not args.no_comparator:
        m = min(cc.numel(), 64 << 20)
        xs, ys = x[:m], cc[:m]
        st, jt = se.stats_accumulate(ys, W, x=xs, stream=stream)
        stream.synchronize()
        metrics = se.stats_metrics(st, jt)
        battery = {"on": f"C' vs original (first {m} bytes)",
                   **{k_: (round(v, 6) if isinstance(v, float) else v) for k_, v in metrics.items()}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peaks, peak_src = load_peaks()
    clk = clocks.summary()
    total_bytes = synth.CONFIGS[args.config]["n_bytes"] * (1 if scaling == "strong" else world)
    gbs = total_bytes / (ms_step / 1e3) / 1e9
    # dominant kernel = the slower of the two fused calls (each call is one kernel launch)
    dom_name, dom_ms = ("k_protect_block8", mp) if mp >= mr else ("k_recover_block8", mr)
    if masked:      # per-CTA kernels (se_api.cu use_tile); protect = keystream kernel + fused kernel
        kkey = f"{dom_name}<{L}, 1>"
    else:           # the persistent tile kernels
        kkey = f"k_tile<{L}, 0, {0 if dom_name == 'k_protect_block8' else 1}>"
    roofline = make_roofline(kkey, config_dict(args, world)["workload"], L, masked, n, lay, dom_ms, peaks, peak_src)
    hbm_bytes = n + lay["a_bytes"] + lay["b_bytes"] + lay["c_bytes"]
    line = {
        "metric": "protect+recover GB/s per GPU and at 1/2/4/8 B200; % of HBM roofline",
        "value": round(gbs, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": config_dict(args, world),
        "roofline": roofline,
        "hbm": {"bytes_per_step": 2 * hbm_bytes, "achieved_gbs": round(2 * hbm_bytes / (ms_step / 1e3) / 1e9, 1),
                "peak_gbs": peaks.get("hbm_gbs"),
                "frac": round(2 * hbm_bytes / (ms_step / 1e3) / 1e9 / peaks.get("hbm_gbs", 6551.7), 4),
                "note": "rank 0's algorithmic bytes over the max-over-ranks step time"},
        "rank0": {"n_bytes": n, "block_offset": boff, "n_blocks": lay["n_blocks"],
                  "kernels_ms": {"protect": round(mp, 5), "recover": round(mr, 5)},
                  "protect_gbs": round(n / (mp / 1e3) / 1e9, 3), "recover_gbs": round(n / (mr / 1e3) / 1e9, 3),
                  "step_ms_stats": {"mean": round(mp + mr, 5),
                                    "median": round(statistics.median(p + r for p, r in zip(t_prot, t_rec)), 5),
                                    "best": round(min(p + r for p, r in zip(t_prot, t_rec)), 5)}},
        "max_over_ranks_ms": {"protect": round(mp_max, 5), "recover": round(mr_max, 5)},
        "variants": variants or None,
        "comparator_aes128_ctr_gbs": None if aes_gbs is None else round(aes_gbs, 2),
        "security_battery": battery,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if "public_plain" in variants:
        v = variants["public_plain"]
        pkey, pdom_ms = v.pop("_dom")
        v["value"] = round(total_bytes / (v["ms_per_step"] / 1e3) / 1e9, 3)
        v["roofline"] = make_roofline(pkey, config_dict(args, world)["workload"] + " (PUBLIC_PLAIN)", L, False, n,
                                      lay, pdom_ms, peaks, peak_src)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(x_np, W, L, key, iv, flags, args.cpu_seconds, block_offset=boff)
    if world > 1:
        dist.destroy_process_group()
    return line


def make_roofline(kkey, workload_name, L, masked, n_in, lay, dom_ms, peaks, peak_src):
    """roofline object of the dominant kernel: masked = ALU-pipe
    bound (algorithmic ALU ops / measured ALU-pipe peak, tools/intbench.cu ->
    profiles/round2_intpeak.json), PUBLIC_PLAIN = HBM bound (algorithmic bytes /
    measured copy bandwidth).  `traffic` = ncu DRAM bytes of this kernel on
    THIS workload (profiles/round*_traffic.json), else null."""
    alg_bytes = n_in + lay["a_bytes"] + lay["b_bytes"] + lay["c_bytes"]     # per launch
    traffic, tsrc = load_traffic(kkey, workload_name)
    prof = load_profile_stats(kkey, workload_name)
    if masked:
        ops = alu_ops_per_block(L, True) * lay["n_blocks"]
        achieved = ops / (dom_ms / 1e3) / 1e9                        # Gop/s
        lanes, lsrc = alu_lanes_per_clk()
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak_alu = NUM_SMS * lanes * mhz * 1e6 / 1e9
        r = {"bound": "alu", "kernel": kkey, "achieved": round(achieved, 1), "peak": round(peak_alu, 1),
             "unit": "Gop/s", "frac": round(achieved / peak_alu, 4), "traffic": traffic, "traffic_source": tsrc,
             "algorithmic_bytes": alg_bytes, "alu_ops_per_block": alu_ops_per_block(L, True),
             "peak_source": f"{NUM_SMS} SMs x {lanes} ALU-pipe lanes/clk/SM ({lsrc}) x {mhz} MHz (max clock)"}
    else:
        ach = alg_bytes / (dom_ms / 1e3) / 1e9
        r = {"bound": "hbm", "kernel": kkey, "achieved": round(ach, 1), "peak": peaks.get("hbm_gbs"),
             "unit": "GB/s", "frac": round(ach / peaks.get("hbm_gbs", 6551.7), 4), "traffic": traffic,
             "traffic_source": tsrc, "algorithmic_bytes": alg_bytes,
             "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    if traffic:
        r["traffic_over_algorithmic"] = round(traffic / alg_bytes, 3)
    if prof and prof.get("inst_per_block"):
        # issue view: executed SASS instructions (ncu, same kernel and workload) per issue slot
        mhz = peaks.get("sm_max_mhz", 1965.0)
        issue = prof["inst_per_block"] * lay["n_blocks"] / (dom_ms / 1e3) / (NUM_SMS * 128 * mhz * 1e6)
        r["issue_frac"] = round(issue, 4)
        r["inst_per_block"] = prof["inst_per_block"]
    return r


def run_multi(args):
    """BASELINE.json's multi-GPU configs: C4 (1 GiB file, row stripes, one per
    rank: strong scaling) and C5 (10,000 files 1 KiB-16 MiB, LPT by file bytes,
    one batched launch per rank per direction: strong scaling).  No data-path
    collective; NCCL only for the barrier and the max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_1803_04880_b200 as se
    from paper_1803_04880_b200 import shard

    rank, world, local = dist_env()
    dev = init_dist(local) if world > 1 else torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    se.lib()
    key, L = synth.KEY, 2
    flags = se.FLAG_PUBLIC_PLAIN if args.plain else 0
    if args.config == 4 and args.full:
        # C4-FULL (row a11 with row e): whole-matrix DWT, W = 32768, stripes of
        # block rows protected from their rows + 2(2^L-1) halo rows and recovered
        # from their fragments + one halo block row per side
        c = synth.CONFIGS[4]
        n, W = c["n_bytes"], 32768
        plan = shard.plan_full_stripes(n, W, L, world)[rank]
        full = synth.config_input(4)
        iv = synth.iv_for(4)
        src = torch.from_numpy(np.ascontiguousarray(full[plan["src_byte_begin"]: plan["src_byte_end"]])).to(dev)
        rec_src0 = max(0, plan["rec_row0"] - 2 * ((1 << L) - 1))
        rec_src1 = min(n, (plan["rec_row0"] + plan["rec_rows"] + 2 * ((1 << L) - 1)) * W)
        ext_in = torch.from_numpy(np.ascontiguousarray(full[rec_src0 * W: rec_src1])).to(dev)
        x = torch.from_numpy(np.ascontiguousarray(full[plan["byte_begin"]: plan["byte_end"]])).to(dev)
        del full
        # the fragments of the recover window (untimed setup: in a deployment they are read from storage)
        ext = se.fragment_protect_stripe(ext_in, n, W, L, key, iv, plan["rec_row0"],
                                         plan["rec_row0"] + plan["rec_rows"], rec_src0, flags=flags)
        del ext_in
        nb = plan["n_blocks"]
        lay = se.fragment_layout(n, W, L, se.MODE_FULL)
        frag = tuple(se._empty(-(-nb * lay[k] // 8), dev) for k in ("a_bits", "b_bits", "c_bits"))
        out = se._empty(x.numel(), dev)
        rep = torch.empty(2, dtype=torch.int64, device=dev)

        def protect():
            se.fragment_protect_stripe(src, n, W, L, key, iv, plan["row_begin"], plan["row_end"], plan["src_row0"],
                                       flags=flags, out=frag)

        def recover():
            se.fragment_recover_stripe(*ext, n, W, L, key, iv, plan["row_begin"], plan["row_end"], plan["rec_row0"],
                                       plan["rec_rows"], flags=flags, out=out, report=rep)

        def check():
            return torch.equal(out, x) and rep.cpu().tolist() == [-1, 0]
        total_bytes, n_blocks_local = n, nb
        workload = (f"C4-FULL 1 GiB W=32768 whole-matrix DWT L=2: {world} row stripes with "
                    f"{2 * ((1 << L) - 1)} halo rows per side (protect) / 1 halo block row (recover)")
        extra = {"stripe_rows": plan["row_end"] - plan["row_begin"], "mode_detail": "FULL"}
    else:
        sizes = synth.c5_file_sizes(10000, 5)
        mine = shard.plan_files(sizes, world)[rank]
        gen = torch.Generator(device=dev)
        files = []
        for i in mine:
            gen.manual_seed(5_000_000 + i)
            files.append(torch.randint(0, 256, (int(sizes[i]),), dtype=torch.uint8, device=dev, generator=gen))
        widths = [synth.width_rule(int(sizes[i])) for i in mine]
        ivs = [synth.iv_for(5, i) for i in mine]
        batch = se.Batch(files, widths, ivs, L, key, flags=flags)

        def protect():
            batch.protect()

        def recover():
            batch.recover()

        def check():
            outs, reps = batch.recover()
            return all(torch.equal(o, f) for o, f in zip(outs, files)) and bool((reps[:, 1] == 0).all())
        total_bytes = int(sizes.sum())
        n_blocks_local = sum(se.fragment_layout(f.numel(), w, L)["n_blocks"] for f, w in zip(files, widths))
        workload = "C5-10000-files-1KiB-16MiB-L2 (LPT by bytes; content uniform random bytes generated on device)"
        extra = {"files_total": len(sizes), "files_this_rank": len(files), "bytes_this_rank": int(sum(sizes[mine]))}
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    protect()
    recover()
    torch.cuda.synchronize()
    assert check(), "recover(protect(x)) != x"
    clocks = ClockSampler(dev.index if dev.index is not None else local)
    clocks.start()
    i, t_end = 0, time.time() + args.soak          # >= W steps and ~soak s of load for the clock samples
    while i < args.warmup or time.time() < t_end:
        protect()
        recover()
        torch.cuda.synchronize()
        i += 1
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    se.launch_count(reset=True)
    for k in range(args.steps):
        l2_flush(flush, k)
        ev[k][0].record()
        protect()
        ev[k][1].record()
        recover()
        ev[k][2].record()
    torch.cuda.synchronize()
    launches = se.launch_count()
    clocks.stop()
    t_p = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
    t_r = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
    t = torch.tensor([t_p + t_r, t_p, t_r], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce_max(t)
        dist.destroy_process_group()
    if rank != 0:
        return None
    ms, mp, mr = (float(v) for v in t.tolist())
    peaks, peak_src = load_peaks()
    lanes, lsrc = alu_lanes_per_clk()
    peak_alu = NUM_SMS * lanes * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
    achieved = alu_ops_per_block(L, not args.plain) * n_blocks_local / (max(mp, mr) / 1e3) / 1e9
    return {
        "metric": "protect+recover GB/s per GPU and at 1/2/4/8 B200; % of HBM roofline",
        "value": round(total_bytes / (ms / 1e3) / 1e9, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": dict({"workload": workload + (" (PUBLIC_PLAIN)" if args.plain else ""),
                        "n_bytes_total": total_bytes, "levels": L,
                        "mode": "FULL" if getattr(args, "full", False) else "BLOCK8",
                        "parallelism": f"dp{world} ({'row stripes' if args.config == 4 else 'by file'})",
                        "l2": "flushed between steps (2x L2 write + read-back)"}, **extra),
        "roofline": {"bound": "alu", "kernel": "k_protect/k_recover (rank 0 slowest)", "achieved": round(achieved, 1),
                     "peak": round(peak_alu, 1), "unit": "Gop/s", "frac": round(achieved / peak_alu, 4),
                     "traffic": None, "peak_source": f"{NUM_SMS} SMs x {lanes} ALU lanes/clk ({lsrc}) x "
                                                     f"{peaks.get('sm_max_mhz')} MHz ({peak_src})"},
        "protect_gbs": round(total_bytes / (mp / 1e3) / 1e9, 3), "recover_gbs": round(total_bytes / (mr / 1e3) / 1e9, 3),
        "e2e": {"value": None, "unit": "GB/s", "note": "multi-file / stripe modes are device-resident; e2e is measured "
                                                       "on the default config"},
        "gpu_launches": int(launches), "clocks": clocks.summary(),
    }


def run_e2e(se, torch, x_np, W, L, key, iv, flags, dev, steps, chunk_bytes=0, n_streams=3, block_offset=0,
            world=1, pipelined=False):
    """The same metric end to end through the public host API: one step =
    fragment_protect_host (pinned input -> H2D -> fused kernel -> D2H of the three
    fragments) + fragment_recover_host (H2D fragments -> kernel -> D2H bytes);
    the library pipelines chunks over several streams.  Both calls block, so
    the step is timed host-side (perf_counter) around them; with several
    ranks, between barriers and as the max over ranks."""
    import torch.distributed as dist
    n = x_np.size
    lay = se.fragment_layout(n, W, L, block_offset=block_offset)
    hx = torch.from_numpy(x_np).pin_memory()
    frag = (se._host_empty(lay["a_bytes"]), se._host_empty(lay["b_bytes"]), se._host_empty(lay["c_bytes"]))
    hout = se._host_empty(n)

    def one():
        if pipelined:       # recover chunk k starts as soon as protect chunk k's fragments are in host memory
            _, tp = se.fragment_protect_host_async(hx, W, L, key, iv, flags=flags, block_offset=block_offset,
                                                   out=frag, chunk_bytes=chunk_bytes, n_streams=n_streams)
            _, tr = se.fragment_recover_host_async(*frag, n, W, L, key, iv, flags=flags, block_offset=block_offset,
                                                   out=hout, chunk_bytes=chunk_bytes, n_streams=n_streams, after=tp)
            rep = tr.wait()
            tp.wait()
            return rep
        se.fragment_protect_host(hx, W, L, key, iv, flags=flags, block_offset=block_offset, out=frag,
                                 chunk_bytes=chunk_bytes, n_streams=n_streams)
        _, rep = se.fragment_recover_host(*frag, n, W, L, key, iv, flags=flags, block_offset=block_offset,
                                          out=hout, chunk_bytes=chunk_bytes, n_streams=n_streams)
        return rep

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        rep = one()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    assert torch.equal(hout, hx) and rep == (-1, 0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        allreduce_max(t)
        ms = float(t.item())
    frag_bytes = lay["a_bytes"] + lay["b_bytes"] + lay["c_bytes"]
    mapped = bool(flags & se.FLAG_HOST_MAPPED)
    how = ("SE_FLAG_HOST_MAPPED: the kernels read / write the pinned host buffers over PCIe, no staging"
           if mapped else (f"{chunk_bytes >> 10} KiB chunks" if chunk_bytes else
                           f"library-default chunks ({min(16 << 20, max(4 << 20, n // 4)) >> 10} KiB)")
           + f" on {n_streams} streams")
    calls = ("fragment_protect_host_async + fragment_recover_host_async(after=protect ticket) + se_host_wait"
             if pipelined else "fragment_protect_host + fragment_recover_host")
    return {"value": round(n * world / (ms / 1e3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": n + frag_bytes,
            "d2h_bytes_per_step": frag_bytes + n, "ms_per_step": round(ms, 4),
            "path": f"{calls} (C ABI, pinned host buffers, {how}), "
                    f"host wall clock" + (", max over ranks; bytes are per rank" if world > 1 else "")}


# ---------------------------------------------------------------- NEXT row f3: Chapter 4 DCT SE

# Table 4.1 / 4.9 image sizes (grey scale)
DCT_SIZES = [(1024, 768), (1600, 1200), (3240, 2592), (4800, 4800)]
# ALU-pipe ops per 8x8 block at level 2 (DESIGN.md §5 f3): SHA-512 of one
# message block (unkeyed: from round 0, 16 message rounds x 20 + 64 schedule
# rounds x 36; keyed: from the round-4 midstate, 12 x 20 + 64 x 36), less what
# the launch-constant schedule removes (sha2_spec.cuh: 8 per sigma of
# W16..W31 not evaluated - 16 unkeyed, 18 keyed - and the low half of K + W
# for the 14 / 12 block-independent words), pixel byte PRMTs (64 in, 48
# pack), mask XOR 16, record pack ~30, AES-CTR share 260 * 66/128.  The fp32
# DCT work issues on the FMA pipe.
DCT_ALU_OPS = {"bytes": 64 + 48, "xor": 16, "record": 30, "aes": 260 * 66 / 128}
DCT_SHA512_OPS = {False: 16 * 20 + 64 * 36 - 8 * 16 - 14, True: 12 * 20 + 64 * 36 - 8 * 18 - 12}


def run_dct(args):
    import torch

    import paper_1803_04880_b200 as se
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    se.lib()
    level, flags = args.dct, (se.DCT_KEYED if args.dct_keyed else 0)
    key, iv = synth.KEY, synth.iv_for(6)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    per_size = []
    clocks = ClockSampler(0)
    clocks.start()
    for (W, H) in DCT_SIZES:
        x_np = synth.bitmap(H, W, 1, W + H).reshape(-1)
        n = x_np.size
        lay = se.dct_layout(W, H, 1, level, flags)
        x = torch.from_numpy(x_np).to(dev)
        a = torch.empty(lay["a_bytes"], dtype=torch.uint8, device=dev)
        p = torch.empty(n, dtype=torch.uint8, device=dev)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        with torch.cuda.stream(stream):
            se.dct_protect(x, W, H, 1, level, key, iv, flags=flags, out=(a, p), stream=stream)
            se.dct_recover(a, p, W, H, 1, level, key, iv, flags=flags, out=out, stream=stream)
        stream.synchronize()
        d = (out.to(torch.int16) - x.to(torch.int16)).abs()
        mse = float((d.float() ** 2).mean())
        assert int(d.max()) <= 1, "DCT round trip off by more than 1"
        t_end = time.time() + args.soak / len(DCT_SIZES)
        i = 0
        while i < args.warmup or time.time() < t_end:
            se.dct_protect(x, W, H, 1, level, key, iv, flags=flags, out=(a, p), stream=stream)
            se.dct_recover(a, p, W, H, 1, level, key, iv, flags=flags, out=out, stream=stream)
            i += 1
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        se.launch_count(reset=True)
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                l2_flush(flush, k)                                  # evict L2 (images are < L2)
                ev[k][0].record(stream)
                se.dct_protect(x, W, H, 1, level, key, iv, flags=flags, out=(a, p), stream=stream)
                ev[k][1].record(stream)
                se.dct_recover(a, p, W, H, 1, level, key, iv, flags=flags, out=out, stream=stream)
                ev[k][2].record(stream)
        stream.synchronize()
        launches = se.launch_count()
        tp = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
        tr = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
        # AES-128-CTR of the whole image on the same GPU: the paper's comparator (Table 4.9)
        y = torch.empty_like(x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for _ in range(3):
                se.cipher_encrypt(key, iv, x, out=y, stream=stream)
            e0.record(stream)
            for k in range(args.steps):
                se.cipher_encrypt(key, iv, x, out=y, stream=stream)
            e1.record(stream)
        stream.synchronize()
        t_aes = e0.elapsed_time(e1) / args.steps
        # the DCT 8x8 alone, forward and inverse (Table 4.1's operation), L2 flushed
        coef = torch.empty(n, dtype=torch.float32, device=dev)
        ef = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            se.dct8_forward(x, W, H, 1, out=coef, stream=stream)
            se.dct8_inverse(coef, W, H, 1, out=out, stream=stream)
            for k in range(args.steps):
                l2_flush(flush, k)
                ef[k][0].record(stream)
                se.dct8_forward(x, W, H, 1, out=coef, stream=stream)
                ef[k][1].record(stream)
                se.dct8_inverse(coef, W, H, 1, out=out, stream=stream)
                ef[k][2].record(stream)
        stream.synchronize()
        assert torch.equal(out, x), "dct8_inverse(dct8_forward(x)) != x"
        t_f = sum(e[0].elapsed_time(e[1]) for e in ef) / args.steps
        t_i = sum(e[1].elapsed_time(e[2]) for e in ef) / args.steps
        del coef
        per_size.append({"image": f"{W}x{H}", "n_bytes": n, "a_bytes": lay["a_bytes"],
                         "dct8_forward_ms": round(t_f, 5), "dct8_inverse_ms": round(t_i, 5),
                         "dct8_hbm_gbs": round(5 * n / ((t_f + t_i) / 2) / 1e6, 1),
                         "protect_ms": round(tp, 5), "recover_ms": round(tr, 5),
                         "protect_gbs": round(n / tp / 1e6, 2), "recover_gbs": round(n / tr / 1e6, 2),
                         "aes128_ctr_ms": round(t_aes, 5),
                         "psnr_db": round(10 * np.log10(255.0 ** 2 / mse), 3) if mse else None,
                         "launches_per_step": launches / args.steps})
        big = (x, a, p, out, W, H, n, lay, tp, tr, launches, x_np)
    clocks.stop()
    x, a, p, out, W, H, n, lay, tp, tr, launches, x_np = big
    peaks, peak_src = load_peaks()
    ms_step = tp + tr
    dom_name, dom_ms = ("k_dct_protect", tp) if tp >= tr else ("k_dct_recover", tr)
    aesf = 1 if (dom_name == "k_dct_recover" or level == 1) else 0   # AES inside the kernel (k_dct.cu)
    kkey = f"{dom_name}<1, {level}, {1 if flags else 0}, {aesf}>"
    traffic, traffic_src = load_traffic(kkey, f"Table 4.1 image {W}x{H} grey, level {level}")
    alg_bytes = 2 * n + lay["a_bytes"]
    if level == 2:
        ops_blk = sum(DCT_ALU_OPS.values()) + DCT_SHA512_OPS[bool(flags)]
        ach = ops_blk * lay["records"] / (dom_ms / 1e3) / 1e9
        lanes, lsrc = alu_lanes_per_clk()
        peak_alu = NUM_SMS * lanes * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
        roofline = {"bound": "alu", "kernel": kkey, "achieved": round(ach, 1), "peak": round(peak_alu, 1),
                    "unit": "Gop/s", "frac": round(ach / peak_alu, 4), "traffic": traffic,
                    "traffic_source": traffic_src, "algorithmic_bytes": alg_bytes, "alu_ops_per_block": ops_blk,
                    "peak_source": f"{NUM_SMS} SMs x {lanes} ALU lanes/clk ({lsrc}) x "
                                   f"{peaks.get('sm_max_mhz', 1965.0)} MHz ({peak_src} max clock)"}
    else:
        ach = alg_bytes / (dom_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": kkey, "achieved": round(ach, 1), "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": round(ach / peaks.get("hbm_gbs", 6551.7), 4), "traffic": traffic,
                    "traffic_source": traffic_src, "algorithmic_bytes": alg_bytes,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    # e2e: pinned host image -> device -> protect -> fragments to host -> back -> recover -> image to host
    hx = torch.from_numpy(x_np).pin_memory()
    ha = torch.empty(lay["a_bytes"], dtype=torch.uint8).pin_memory()
    hp, ho = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, args.steps // 4)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            x.copy_(hx, non_blocking=True)
            se.dct_protect(x, W, H, 1, level, key, iv, flags=flags, out=(a, p), stream=stream)
            ha.copy_(a, non_blocking=True)
            hp.copy_(p, non_blocking=True)
            a.copy_(ha, non_blocking=True)
            p.copy_(hp, non_blocking=True)
            se.dct_recover(a, p, W, H, 1, level, key, iv, flags=flags, out=out, stream=stream)
            ho.copy_(out, non_blocking=True)
        e1.record(stream)
    stream.synchronize()
    e2e_ms = e0.elapsed_time(e1) / reps
    line = {
        "metric": "DCT 8x8 SE (Ch. 4) protect+recover GB/s per GPU",
        "value": round(n / (ms_step / 1e3) / 1e9, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"Table 4.1 image {W}x{H} grey, level {level}" + (" keyed" if flags else ""),
                   "row": "f3", "l2": "flushed between steps (2x L2 write + read-back)"},
        "roofline": roofline,
        "per_image": per_size,
        "paper_context": "Table 4.9 (GTX 780): SE level 2 5.41 ms, AES-128 5.46 ms for 4800x4800; "
                         "Table 4.1: DCT 8x8 on GPU 1.12 ms (desktop) / 9.98 ms (laptop) for 4800x4800",
        "e2e": {"value": round(n / (e2e_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                "h2d_bytes_per_step": n + lay["a_bytes"] + n, "d2h_bytes_per_step": lay["a_bytes"] + n + n,
                "path": "pinned host image, H2D, dct_protect, D2H fragments, H2D fragments, dct_recover, D2H"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if not args.no_cpu_baseline:
        import oracle
        rows = 64
        xs = x_np[: rows * W]
        t0 = time.perf_counter()
        reps_c = 0
        while True:
            a_o, p_o = oracle.dct_protect(xs, W, rows, 1, level, key, iv, flags=flags)
            oracle.dct_recover(a_o, p_o, W, rows, 1, level, key, iv, flags=flags)
            reps_c += 1
            if time.perf_counter() - t0 > args.cpu_seconds / 3:
                break
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": round(xs.size * reps_c / dt / 1e9, 6), "unit": "GB/s", "cores": 1,
                                "kind": "oracle",
                                "sample": f"{reps_c} pass(es) over the first {rows} rows ({xs.size} bytes) of the "
                                          f"{W}x{H} image (protect+recover), 1 host thread, {dt:.1f} s",
                                "host_cpu": cpu_model()}
    return line


# ---------------------------------------------------------------- CPU oracle baseline

def oracle_time(x_np, W, L, key, iv, flags, n_blocks_sample, threads, reps=1, block_offset=0):
    """Oracle protect + recover over the first n_blocks_sample blocks, split
    across `threads` host threads (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    lay = oracle.layout(x_np.size, W, L)
    nb = min(n_blocks_sample, lay["n_blocks"])
    bufs = [np.zeros(max(lay[k], 1), np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes")]
    out = np.zeros(max(x_np.size, 1), np.uint8)
    groups = -(-nb // 128)
    per = -(-groups // threads)
    ranges = [(g0 * 128, min(nb, (g0 + per) * 128)) for g0 in range(0, groups, per)]

    def prot(r):
        oracle.protect(x_np, W, L, key, iv, flags=flags, block_offset=block_offset, block_range=r, out=bufs)

    def rec(r):
        oracle.recover(bufs[0], bufs[1], bufs[2], x_np.size, W, L, key, iv, flags=flags, block_offset=block_offset,
                       block_range=r, out=out)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        t0 = time.perf_counter()
        for _ in range(reps):
            list(ex.map(prot, ranges))
            list(ex.map(rec, ranges))
        dt = time.perf_counter() - t0
    return nb * reps, dt


def oracle_rate(x_np, W, L, key, iv, flags, threads, block_offset=0, min_seconds=0.5):
    """Blocks per second of the oracle on `threads` threads, from a probe grown
    until it runs >= min_seconds (a tiny probe is dominated by thread start-up)."""
    total_nb = -(-x_np.size // (W * 8)) * (W // 8)
    nb = min(total_nb, 256 * threads)
    while True:
        done, dt = oracle_time(x_np, W, L, key, iv, flags, nb, threads, block_offset=block_offset)
        if dt >= min_seconds or nb >= total_nb:
            return done / max(dt, 1e-6)
        nb = min(total_nb, int(nb * max(2.0, 1.5 * min_seconds / max(dt, 1e-3))))


def cpu_baseline(x_np, W, L, key, iv, flags, seconds, block_offset=0):
    threads = os.cpu_count() or 1
    rate = oracle_rate(x_np, W, L, key, iv, flags, threads, block_offset)
    total_nb = -(-x_np.size // (W * 8)) * (W // 8)
    want = max(128, rate * seconds)
    nb = int(min(total_nb, want))
    reps = max(1, min(50, int(want // nb)))
    done, dt = oracle_time(x_np, W, L, key, iv, flags, nb, threads, reps, block_offset=block_offset)
    gbs = done * 64 / dt / 1e9
    # the same on one core (SURVEY.md §8.1 row d: 1 core and all host cores), a ~3 s sample
    nb1 = int(min(total_nb, max(128, rate / threads * 3.0)))
    done1, dt1 = oracle_time(x_np, W, L, key, iv, flags, nb1, 1, block_offset=block_offset)
    return {"value": round(gbs, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{reps} pass(es) over the first {nb} of {total_nb} 8x8 blocks of the same input "
                      f"(protect+recover), {threads} host threads, {dt:.1f} s",
            "one_core": {"value": round(done1 * 64 / dt1 / 1e9, 6), "unit": "GB/s", "cores": 1,
                         "sample": f"first {nb1} blocks, {dt1:.1f} s"},
            "host_cpu": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """The reference arm: the CPU oracle (oracle/, plain C) as it stands, on
    all host cores, over the SAME workload as the repo arm's line (same
    `config`): every timed step is protect + recover of the whole input (C4:
    the whole 1 GiB file; C1-C3: one file per rank of the repo arm).  Warm-up
    steps run on a bounded prefix (they only warm caches and threads).  Under
    torchrun, rank 0 alone runs; the other ranks exit without work."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    c = synth.CONFIGS[args.config]
    W, L = c["width"], c["levels"]
    key = synth.KEY
    flags = 1 if args.plain else 0
    threads = os.cpu_count() or 1
    if args.config == 4:
        inputs = [(synth.config_input(4), synth.iv_for(4))]
        scaling = "strong"
    else:
        x_np = synth.config_input(args.config)
        inputs = [(x_np, synth.iv_for(args.config, r)) for r in range(world)]
        scaling = "weak"
    total_bytes = sum(x.size for x, _ in inputs)
    nb_of = [-(-x.size // (W * 8)) * (W // 8) for x, _ in inputs]
    x0, iv0 = inputs[0]
    rate = oracle_rate(x0, W, L, key, iv0, flags, threads, min_seconds=0.3)   # blocks/s, all threads
    nb_warm = int(min(nb_of[0], max(128, rate * 1.0)))
    for _ in range(args.warmup):
        oracle_time(x0, W, L, key, iv0, flags, nb_warm, threads)
    times = []
    for _ in range(args.steps):
        dt = 0.0
        for (x, iv), nb in zip(inputs, nb_of):
            _, d = oracle_time(x, W, L, key, iv, flags, nb, threads)
            dt += d
        times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    gbs = total_bytes / (ms / 1e3) / 1e9
    sample = (f"every timed step = protect + recover of the whole workload ({sum(nb_of)} 8x8 blocks, "
              f"{total_bytes} bytes), {threads} host threads; warm-up steps on the first {nb_warm} blocks")
    return {
        "metric": "protect+recover GB/s per GPU and at 1/2/4/8 B200; % of HBM roofline",
        "impl": "reference", "value": round(gbs, 6), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": round(gbs, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "host_cpu": cpu_model()},
        "e2e": {"value": round(gbs, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def relaunch_distributed(n: int):
    """`python bench.py --gpus N` outside torchrun: re-run this command as N
    ranks, one process per GPU (the driver's own launch line)."""
    port = os.environ.get("MASTER_PORT", "29533")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", port, os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default 4: the 1 GiB file, one row stripe per rank)")
    ap.add_argument("--stripes", action="store_true", help="(kept for old command lines: C4 always runs as stripes)")
    ap.add_argument("--full", action="store_true", help="C4 stripes in FULL mode (whole-matrix DWT, halo rows)")
    ap.add_argument("--impl", default="se", choices=["se", "reference"])
    ap.add_argument("--plain", action="store_true", help="PUBLIC_PLAIN measurement mode (C26)")
    ap.add_argument("--soak", type=float, default=1.5, help="seconds of sustained warm-up load")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunk-kib", type=int, default=0, help="host-API chunk size (input KiB; 0 = library default)")
    ap.add_argument("--e2e-streams", type=int, default=3, help="host-API CUDA streams")
    ap.add_argument("--e2e-mapped", type=int, default=0, help="1: zero-copy host API (SE_FLAG_HOST_MAPPED)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparator", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the PUBLIC_PLAIN line inside the masked run")
    ap.add_argument("--dct", type=int, default=0, choices=[0, 1, 2],
                    help="NEXT row f3: bench the Chapter 4 DCT SE at this protection level instead")
    ap.add_argument("--dct-keyed", action="store_true", help="level 2 with the keyed hash framing (D9)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_distributed(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    if args.impl == "reference":
        line = run_reference(args)
    elif args.dct:
        line = run_dct(args)
    elif args.config == 5 or (args.config == 4 and args.full):
        line = run_multi(args)
    else:
        line = run_se(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
