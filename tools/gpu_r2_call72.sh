for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/*.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --steps 10 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b72.json 2>/dev/null
  echo "C4 $v $(python -c "import json;d=json.load(open('gpurun_out/b72.json'));print(d['value'], d['rank0']['kernels_ms'])")"
  SE_LIB_PATH=$v timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b72.json 2>/dev/null
  echo "C2 $v $(python -c "import json;d=json.load(open('gpurun_out/b72.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done; done
