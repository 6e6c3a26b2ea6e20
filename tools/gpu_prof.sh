# one-GPU profiling pass: plain run, then the ncu launch list and full captures
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CMD="python bench.py --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 2"
$CMD > gpurun_out/plain.log 2>&1 && echo plain ok && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && echo ncu1 ok && \
ncu --set full --clock-control none --import-source on -k regex:k_protect_block8 -s 3 -c 1 -o gpurun_out/prof_protect $CMD > gpurun_out/ncu2.log 2>&1 && echo ncu2 ok && \
ncu --set full --clock-control none --import-source on -k regex:k_recover_block8 -s 3 -c 1 -o gpurun_out/prof_recover $CMD > gpurun_out/ncu3.log 2>&1 && echo ncu3 ok
tail -3 gpurun_out/ncu3.log
