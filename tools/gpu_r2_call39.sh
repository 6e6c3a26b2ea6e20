mkdir -p gpurun_out/c39
CP="python bench.py --plain --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CP > gpurun_out/c39/p.log 2>&1 && echo p ok && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 8 -c 2 -o gpurun_out/c39/c4_plain $CP > gpurun_out/c39/ncu_p.log 2>&1 && echo ncu-p ok
