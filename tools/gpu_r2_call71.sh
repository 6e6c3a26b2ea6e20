for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/*.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --steps 10 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b71.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.load(open('gpurun_out/b71.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done
SE_KS_LANE_NARROW=1 timeout 300 python bench.py --steps 10 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b71.json 2>/dev/null
echo "narrow-ks $(python -c "import json;d=json.load(open('gpurun_out/b71.json'));print(d['value'], d['rank0']['kernels_ms'])")"
done
