# round-2 call 6: ALU/FMA rebalanced lean kernels; parity + C4 plain/masked + C2/C3
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for c in 4 2 3; do for f in "" "--plain"; do
  echo "== C$c $f"; timeout 300 $B --config $c $f 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'], d['hbm']['frac'])"
done; done
CMD="python bench.py --plain --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CMD > gpurun_out/c4_p.log 2>&1 && echo plain-run ok && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 8 -c 2 -o gpurun_out/r2_tile_plain3 $CMD > gpurun_out/ncu_tp3.log 2>&1 && echo ncu ok
tail -n 2 gpurun_out/ncu_tp3.log
