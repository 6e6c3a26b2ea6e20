# round-2 call 12: keystream kernel table for masked protect (5 KB tables vs 64 KB lane LUT)
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
for c in 2 3 4; do for l in 0 1 0 1; do
  echo "== C$c lut=$l"; SE_KS_LUT=$l timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'])"
done; done
