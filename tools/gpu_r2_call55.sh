for cfg in 2 3 4; do for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/v_co.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/b55.json 2>/dev/null
  echo "C$cfg $v $(python -c "import json;t=open('gpurun_out/b55.json').read();d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]);print(d['value'], d['rank0']['kernels_ms'])")"
done; done; done
