# round-2 call 17: tests; C4-FULL stripes, C5 batch, C3 lines (masked and plain)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B="python bench.py --steps 5 --warmup 3 --soak 0.5 --no-cpu-baseline --no-comparator --e2e-steps 0"
for a in "--config 4 --full" "--config 4 --full --plain" "--config 5" "--config 5 --plain" "--config 3" "--config 2"; do
  echo "== $a"; timeout 600 $B $a > gpurun_out/r2_$(echo $a | tr -d ' -').json 2>&1; tail -c 1200 gpurun_out/r2_$(echo $a | tr -d ' -').json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d.get('protect_gbs') or d['rank0']['protect_gbs'], d.get('recover_gbs') or d['rank0']['recover_gbs'], d['roofline']['frac'], (d.get('variants') or {}).get('public_plain',{}).get('value'))" 2>&1 | tail -1
done
