mkdir -p gpurun_out/c36
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_no_alloc.py -x -q -m gpu 2>&1 | tail -3
for cfg in 2 3 4; do for v in 1 0 1 0; do
  SE_KS_LANE_NARROW=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/c36/b.json 2>/dev/null
  echo "C$cfg narrow=$v $(python -c "import json;d=json.load(open('gpurun_out/c36/b.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done; done
