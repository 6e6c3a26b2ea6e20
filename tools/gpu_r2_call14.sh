# round-2 call 14: warp-unit masked kernels (L = 1, 2) vs per-CTA; tests
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
for c in 2 4 1; do for k in 1 0; do
  echo "== C$c warp=$k"; SE_WARP=$k timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'])"
done; done
