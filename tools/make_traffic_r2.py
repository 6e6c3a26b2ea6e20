#!/usr/bin/env python3
"""profiles/round2_traffic.json from ncu `--set full` captures of the bench
workloads: per (kernel, workload) the DRAM bytes per launch (read + write),
executed SASS instructions per 8x8 block and the kernel time.  bench.py
reports these as roofline.traffic / issue_frac for the same kernel on the
same workload only.

usage: make_traffic_r2.py out.json n_blocks "<workload>" rep.ncu-rep [n_blocks "<workload>" rep ...]"""
import csv
import io
import json
import os
import re
import subprocess
import sys


def rows_of(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
            "nsecond": 1e-3, "ns": 1e-3}.get(u, 1)


def main(out, triples):
    entries = []
    for nb, workload, rep in triples:
        hdr, units, rows = rows_of(rep)
        seen = set()
        for r in rows:
            name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("void ", "").replace("se::", "")
            name = re.sub(r"\(int\)|\(bool\)", "", name).replace("true", "1").replace("false", "0")
            if name in seen:
                continue
            seen.add(name)
            get = lambda k: float(r[hdr.index(k)]) * unit_scale(units[hdr.index(k)])   # noqa: E731
            rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
            inst = get("smsp__inst_executed.sum")
            entries.append({"kernel": name, "workload": workload, "dram_bytes": rd + wr, "dram_read": rd,
                            "dram_write": wr, "inst_per_block": round(inst * 32 / int(nb), 1),
                            "gpu_time_us": round(get("gpu__time_duration.sum"), 2),
                            "source": os.path.basename(rep)})
    json.dump({"note": "per launch, from one ncu --set full --clock-control none capture per kernel on the named "
                       "bench workload; inst_per_block = smsp__inst_executed x 32 / 8x8 blocks of the launch",
               "entries": entries}, open(out, "w"), indent=1)
    for e in entries:
        print(e)


if __name__ == "__main__":
    a = sys.argv[2:]
    main(sys.argv[1], [(a[i], a[i + 1], a[i + 2]) for i in range(0, len(a), 3)])
