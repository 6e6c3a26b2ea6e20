mkdir -p gpurun_out/c64
CF="python bench.py --config 4 --full --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
timeout 1200 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:"k_dwt_full_(fwd|inv)" -s 6 -c 2 -o gpurun_out/c64/full_tr $CF > gpurun_out/c64/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/c64/ncu.log
