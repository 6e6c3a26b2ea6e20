mkdir -p gpurun_out
CMD="python bench.py --plain --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 1"
$CMD > gpurun_out/plain_pl.log 2>&1 && echo plain ok && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_pl.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_protect_block8 -s 2 -c 1 -o gpurun_out/p_pl $CMD > gpurun_out/ncu_pl.log 2>&1 && echo ncu ok
