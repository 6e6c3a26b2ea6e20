mkdir -p gpurun_out/c49
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py -x -q -m gpu -k "batch or Batch" 2>&1 | tail -1
for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/v_bs32.so; do
  SE_LIB_PATH=$v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 > gpurun_out/c49/b.json 2>gpurun_out/c49/b.err
  echo "$v $(python -c "import json;t=open('gpurun_out/c49/b.json').read();d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]);print(d['value'], d['protect_gbs'], d['recover_gbs'], d['roofline']['frac'])" 2>&1 | tail -1)"
done; done
