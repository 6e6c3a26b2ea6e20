# round-2 call 15: masked per-CTA tuning variants on C4 and C2 (variants/*.so, SE_LIB_PATH)
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
for r in 1 2; do for v in variants/*.so; do for c in 4 2; do
  echo "$v C$c $(SE_LIB_PATH=$v timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'])" 2>&1 | tail -1)"
done; done; done
