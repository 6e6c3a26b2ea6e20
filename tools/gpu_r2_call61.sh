for v in variants/v_setilenawplain2.so variants/v_setilenawplain3.so; do SE_LIB_PATH=$v timeout 600 python -m pytest tests/test_gpu_tile.py -x -q -m gpu 2>&1 | tail -1; done
for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/*.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --plain --steps 20 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 > gpurun_out/b61.json 2>/dev/null
  echo "plain $v $(python -c "import json;d=json.load(open('gpurun_out/b61.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done; done
