timeout 900 python -m pytest tests/test_gpu_full.py -x -q -m gpu 2>&1 | tail -1
for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/v_fl0.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --config 4 --full --steps 10 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 > gpurun_out/b65.json 2>/dev/null
  echo "C4FULL $v $(python -c "import json;t=open('gpurun_out/b65.json').read();d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]);print(d['value'], d['protect_gbs'], d['recover_gbs'])")"
done; done
