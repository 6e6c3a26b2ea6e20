# round-2 call 22: A/B variants of the PUBLIC_PLAIN kernels (variants/*.so)
B="python bench.py --plain --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for r in 1 2; do for v in variants/*.so; do
  echo "$v $(SE_LIB_PATH=$v timeout 300 $B 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'])" 2>&1 | tail -1)"
done; done
SE_LIB_PATH=variants/ex1.so timeout 300 python -m pytest tests/test_gpu_tile.py -x -q 2>&1 | tail -1
