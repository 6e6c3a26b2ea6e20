# round-2 call 7: per-CTA (keystream kernel for masked protect) vs tile, by config
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for c in 2 3 4; do for k in tile cta; do for f in "" "--plain"; do
  echo "== C$c $k $f"; SE_KERNEL=$k timeout 300 $B --config $c $f 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'], d['hbm']['frac'])"
done; done; done
