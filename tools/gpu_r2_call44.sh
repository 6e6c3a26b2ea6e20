mkdir -p gpurun_out/c44
CM5="python bench.py --config 5 --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
timeout 900 $CM5 > gpurun_out/c44/m5.log 2>&1 && echo m5 ok && tail -c 400 gpurun_out/c44/m5.log && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_batch" -s 6 -c 3 -o gpurun_out/c44/c5_batch $CM5 > gpurun_out/c44/ncu5.log 2>&1 && echo ncu5 ok
tail -5 gpurun_out/c44/ncu5.log
