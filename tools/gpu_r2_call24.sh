# round-2 call 24: full GPU suite; e2e chunk sizes on C2 and C4
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 2 4; do for k in 0 1024 2048 8192; do
  echo "C$c chunk=$k $(timeout 600 python bench.py --config $c --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 10 --e2e-chunk-kib $k 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], d['e2e']['ms_per_step'])" 2>&1 | tail -1)"
done; done
