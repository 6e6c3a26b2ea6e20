#!/usr/bin/env python3
"""Dynamic SASS opcode mix from `ncu --page source --csv --print-source sass`:
executed warp-instructions per opcode (optionally per 'region' of lines)."""
import csv
import re
import sys
from collections import Counter

ALU = ("SHF", "LOP3", "IADD3", "PRMT", "ISETP", "LEA", "SEL", "VIADD", "IABS", "FLO", "POPC", "BMSK", "SGXT", "PLOP3", "BREV", "IMNMX", "VIMNMX", "I2IP")
FMA = ("IMAD",)


def main(path, per=1.0):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    isrc = hdr.index("Source")
    iexe = hdr.index("Instructions Executed")
    mix = Counter()
    for r in rows[2:]:
        if len(r) <= iexe:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[isrc])
        if not m:
            continue
        try:
            n = float(r[iexe])
        except ValueError:
            continue
        mix[m.group(2) + (m.group(3) or "")] += n
    total = sum(mix.values())
    alu = sum(v for k, v in mix.items() if k.startswith(ALU))
    fma = sum(v for k, v in mix.items() if k.startswith(FMA))
    print(f"total {total/per:.0f}  alu-class {alu/per:.0f}  imad-class {fma/per:.0f}  (per {per:g} warps)")
    for k, v in mix.most_common(30):
        print(f"  {k:28s} {v/per:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
