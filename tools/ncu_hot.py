#!/usr/bin/env python3
"""Hot SASS lines of one kernel from `ncu --page source --csv --print-source sass`:
stall-sample share and executed instructions per thread-block unit.
usage: ncu_hot.py src.csv <kernel substring> <units (warps) for per-unit counts> [top]"""
import csv
import re
import sys
from collections import Counter


def sections(path):
    rows = list(csv.reader(open(path)))
    cur = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            yield cur
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None:
            cur[2].append(r)


def main(path, kname, units, top=40):
    for name, hdr, rows in list(sections(path)):
        if kname not in name:
            continue
        isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
        ist = hdr.index("Warp Stall Sampling (All Samples)")
        tot = sum(float(r[ist] or 0) for r in rows)
        ex = sum(float(r[iex] or 0) for r in rows)
        print(name, f"samples {tot:.0f}  inst/unit {ex / units:.1f}")
        mix = Counter()
        for r in rows:
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc])
            if m:
                mix[m.group(2)] += float(r[iex] or 0) / units
        print("  mix:", ", ".join(f"{k} {v:.0f}" for k, v in mix.most_common(16)))
        for i, r in sorted(enumerate(rows), key=lambda x: -float(x[1][ist] or 0))[:top]:
            print(f"  {float(r[ist]) / tot * 100:5.1f}%  ex={float(r[iex] or 0) / units:6.2f}  #{i:5d}  {r[isrc][:100]}")
        return


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
