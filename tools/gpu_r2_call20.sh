# round-2 call 20: keystream kernel shape for the masked calls: full-SM lane table (1) vs one 256-thread CTA per SM (2)
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
for r in 1 2; do for c in 4 2; do for l in 1 2; do
  echo "C$c lut=$l $(SE_KS_LUT=$l timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'])" 2>&1 | tail -1)"
done; done; done
