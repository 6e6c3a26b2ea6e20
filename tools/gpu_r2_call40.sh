mkdir -p gpurun_out/c40
SE_LIB_PATH=variants/v_mm7.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py -x -q -m gpu 2>&1 | tail -2
for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/*.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --steps 10 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/c40/b.json 2>gpurun_out/c40/b.err
  echo "$v $(python -c "import json;d=json.load(open('gpurun_out/c40/b.json'));print(d['value'], d['rank0']['kernels_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done; done
