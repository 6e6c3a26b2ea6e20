# round-2 call 4: tile vs per-CTA kernels (masked, plain) on C4 + ncu of the tile kernels
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for k in tile cta; do for f in "" "--plain"; do
  echo "== $k $f"; SE_KERNEL=$k timeout 300 $B $f 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'])"
done; done
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CMD > gpurun_out/c4_m.log 2>&1 && $CMD --plain > gpurun_out/c4_p.log 2>&1 && echo plain-runs ok && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 8 -c 2 -o gpurun_out/r2_tile_masked $CMD > gpurun_out/ncu_tm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 8 -c 2 -o gpurun_out/r2_tile_plain $CMD --plain > gpurun_out/ncu_tp.log 2>&1 && echo ncu ok
tail -2 gpurun_out/ncu_tm.log gpurun_out/ncu_tp.log
