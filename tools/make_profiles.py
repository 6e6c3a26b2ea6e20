#!/usr/bin/env python3
"""Turn a gpurun evidence directory (tools/gpu_evidence.sh) into the committed
profiles/ summaries: ncu launch list with per-kernel share, per-kernel
`--set full` summaries (pipes, stalls, DRAM traffic, SASS opcode mix) and a
traffic JSON that bench.py reports as roofline.traffic.

usage: python tools/make_profiles.py gpurun_out/ev profiles round1
"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def launch_list(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = defaultdict(list)
    order = []
    for r in rows[1:]:
        name = r[ik]
        short = re.sub(r"\(.*", "", name).replace("void ", "")
        per[short].append(float(r[iv]))
        order.append((short, float(r[iv])))
    total = sum(v for _, v in order)
    out = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
           f"# {len(order)} launches, total {total/1e3:.1f} us", "",
           f"{'kernel':60s} {'launches':>8s} {'avg_us':>9s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:60s} {len(v):8d} {sum(v)/len(v)/1e3:9.2f} {sum(v)/total:7.1%}")
    out += ["", "# launch sequence (first 40)"]
    out += [f"{k:60s} {v/1e3:9.2f} us" for k, v in order[:40]]
    return "\n".join(out) + "\n"


def raw_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2]


KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__waves_per_multiprocessor", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def kernel_summary(rep):
    import sass_mix  # noqa: F401  (same directory)
    hdr, units, v = raw_metrics(rep)
    name = v[hdr.index("Kernel Name")]
    lines = [f"# ncu --set full summary: {name}", f"# report: {os.path.basename(rep)}", ""]
    vals = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k:72s} {v[i]} {units[i]}")
            vals[k] = (v[i], units[i])
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x >= 0.03:
                stalls.append((x, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    lines += ["", "# warp stall reasons (cycles per issued instruction)"]
    lines += [f"  {n:28s} {x:.2f}" for x, n in sorted(stalls, reverse=True)]
    # dynamic opcode mix from the source page
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        h = rows[1]
        isrc, iexe = h.index("Source"), h.index("Instructions Executed")
        mix = Counter()
        for r in rows[2:]:
            if len(r) <= iexe:
                continue
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[isrc])
            try:
                n = float(r[iexe])
            except ValueError:
                continue
            if m:
                mix[m.group(2) + (m.group(3) or "")] += n
        warps = float(vals.get("launch__grid_size", ("1", ""))[0].replace(",", "")) * \
            float(vals.get("launch__block_size", ("32", ""))[0].replace(",", "")) / 32
        lines += ["", f"# dynamic SASS opcode mix, executed warp-instructions per warp (= per thread)"]
        for k, n in mix.most_common(25):
            lines.append(f"  {k:28s} {n / warps:9.1f}")
    rd = float(vals.get("dram__bytes_read.sum", ("0", "byte"))[0].replace(",", ""))
    wr = float(vals.get("dram__bytes_write.sum", ("0", "byte"))[0].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(vals.get("dram__bytes_read.sum", ("", "byte"))[1], 1)
    wr *= scale.get(vals.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
    return "\n".join(lines) + "\n", name, rd + wr


def main(src, dst, tag):
    os.makedirs(dst, exist_ok=True)
    traffic = {}
    if os.path.exists(os.path.join(src, "launches.csv")):
        open(os.path.join(dst, f"{tag}_launches.txt"), "w").write(launch_list(os.path.join(src, "launches.csv")))
    for f in sorted(os.listdir(src)):
        if f.endswith(".ncu-rep"):
            text, name, tb = kernel_summary(os.path.join(src, f))
            open(os.path.join(dst, f"{tag}_{f[:-8]}_ncu.txt"), "w").write(text)
            short = re.sub(r"\(.*", "", name).replace("void ", "").replace("se::", "")
            short = re.sub(r"^(unnamed>::|\(anonymous namespace\)::)", "", short)
            traffic[short] = tb
    for f in sorted(os.listdir(src)):
        if f.endswith(".json") or f.endswith(".txt"):
            data = open(os.path.join(src, f)).read()
            open(os.path.join(dst, f"{tag}_{f}"), "w").write(data)
    json.dump({"note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full "
                       "capture of the bench workload (writes that stay in the 126 MB L2 show as 0)",
               "bytes": traffic}, open(os.path.join(dst, f"{tag}_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
