SE_LIB_PATH=variants/v_lba.so timeout 600 python -m pytest tests/test_gpu_tile.py -x -q -m gpu 2>&1 | tail -1
for cfg in 2 3 4; do for rep in 1 2; do for v in paper_1803_04880_b200/libse.so variants/v_lba.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --config $cfg --plain --steps 20 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 > gpurun_out/b58.json 2>/dev/null
  echo "C$cfg plain $v $(python -c "import json;t=open('gpurun_out/b58.json').read();d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]);print(d['value'], d['rank0']['kernels_ms'])")"
done; done; done
