# round-2 call 2: intbench (per-SM clock64 windows), the new default bench line (C4), C4 PUBLIC_PLAIN + ncu
mkdir -p gpurun_out
./tools/intbench > gpurun_out/intbench2.json 2>&1; cat gpurun_out/intbench2.json
timeout 900 python bench.py > gpurun_out/c4_default.json 2> gpurun_out/c4_default.err; echo "default rc=$?"; tail -c 4000 gpurun_out/c4_default.json; tail -5 gpurun_out/c4_default.err
CMD="python bench.py --plain --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CMD > gpurun_out/c4_plain2.log 2>&1 && echo plain ok && tail -c 3000 gpurun_out/c4_plain2.log && \
ncu --set full --clock-control none --import-source on -k regex:"k_(protect|recover)_block8" -s 6 -c 2 -o gpurun_out/r2_c4_plain_kernels $CMD > gpurun_out/ncu_c4_plain2.log 2>&1 && echo ncu ok
tail -3 gpurun_out/ncu_c4_plain2.log
