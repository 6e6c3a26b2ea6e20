# round-2 call 8: kernel policy (masked: per-CTA, plain: tile); tests; repeated C4 plain timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for c in 2 4; do for f in "" "--plain" "--plain"; do
  echo "== C$c $f"; timeout 300 $B --config $c $f 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'], d['hbm']['frac'], d['clocks']['sm_mhz'])"
done; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
