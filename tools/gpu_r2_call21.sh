# round-2 call 21: PUBLIC_PLAIN tile kernels with PRMT unpack and mbarrier suspend hints
timeout 600 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
B="python bench.py --plain --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for r in 1 2; do for c in 4 2 3; do
  echo "C$c $(timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done; done
