# round-2 call 13: recover keystream parked in the output region; tests + C2/C3/C4 masked
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
for c in 2 3 4; do for k in 0 1; do
  echo "== C$c ks_out=$k"; SE_KS_OUT=$k timeout 300 $B --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['rank0']['kernels_ms'])"
done; done
