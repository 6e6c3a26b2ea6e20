# round-2 call 1: measured INT/issue peaks, C4 PUBLIC_PLAIN line, ncu of the plain kernels on C4
mkdir -p gpurun_out
./tools/intbench > gpurun_out/intbench.json 2>&1; cat gpurun_out/intbench.json
CMD="python bench.py --config 4 --stripes --plain --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CMD > gpurun_out/c4_plain.log 2>&1 && echo plain ok && tail -c 3000 gpurun_out/c4_plain.log && \
ncu --set full --clock-control none --import-source on -k regex:"k_(protect|recover)_block8" -s 6 -c 2 -o gpurun_out/r2_c4_plain $CMD > gpurun_out/ncu_c4_plain.log 2>&1 && echo ncu ok
tail -3 gpurun_out/ncu_c4_plain.log
