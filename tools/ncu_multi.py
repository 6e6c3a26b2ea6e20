#!/usr/bin/env python3
"""Summarise every kernel of an ncu report (key metrics, stalls, SASS mix).
usage: python tools/ncu_multi.py report.ncu-rep [kernel-regex ...]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from make_profiles import KEYS  # noqa: E402

rep = sys.argv[1]
pats = sys.argv[2:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for v in rows[2:]:
    name = v[hdr.index("Kernel Name")]
    if pats and not any(re.search(p, name) for p in pats):
        continue
    print(name)
    for k in KEYS + ["dram__throughput.avg.pct_of_peak_sustained_elapsed"]:
        if k in hdr:
            print(f"  {k:70s} {v[hdr.index(k)]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), h[34:-23]))
            except ValueError:
                pass
    print("  stalls", [(round(x, 2), n) for x, n in sorted(st, reverse=True)[:8]])
    short = re.sub(r"\(.*", "", name).replace("void ", "")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          "regex:" + re.escape(short.split("<")[0])], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2 and "Source" in srows[1]:
        h = srows[1]
        isrc, iexe = h.index("Source"), h.index("Instructions Executed")
        mix, tot = Counter(), 0.0
        for r in srows[2:]:
            if len(r) <= iexe:
                continue
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[isrc])
            try:
                n = float(r[iexe])
            except ValueError:
                continue
            tot += n
            if m:
                mix[m.group(2) + (m.group(3) or "")] += n
        print("  sass total", tot, " top:", ", ".join(f"{k} {n / tot * 100:.1f}%" for k, n in mix.most_common(14)))
