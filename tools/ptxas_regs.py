#!/usr/bin/env python3
"""Compile one .cu with -Xptxas -v and print (kernel, regs, spill bytes) per entry."""
import re
import subprocess
import sys

src = sys.argv[1]
extra = sys.argv[2:]
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
       "-diag-suppress", "177", "-Xptxas=-v", "-c", "-o", "/tmp/ptxas_regs.o", src] + extra
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(anonymous namespace\)::|se::|\(se::\w+\)", "", cur)
        spill = None
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        spill = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs={m.group(1):>4s} spill={spill}")
        cur = None
