SE_LIB_PATH=variants/v_mpi.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "protect_recover" 2>&1 | tail -1
for rep in 1 2 3; do for v in paper_1803_04880_b200/libse.so variants/v_mpi.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --steps 10 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b62.json 2>/dev/null
  echo "masked $v $(python -c "import json;d=json.load(open('gpurun_out/b62.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done; done
