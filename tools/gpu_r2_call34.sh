mkdir -p gpurun_out/c34
for cfg in 2 3; do for v in "SE_PROT_KS=1 SE_KS_OUT=1" "SE_PROT_KS=0 SE_KS_OUT=1" "SE_PROT_KS=1 SE_KS_OUT=0" "SE_PROT_KS=0 SE_KS_OUT=0"; do
  for rep in 1 2; do
  env $v timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 0 > gpurun_out/c34/b.json 2>/dev/null
  echo "C$cfg $v $(python -c "import json;d=json.load(open('gpurun_out/c34/b.json'));print(d['value'], d['rank0']['kernels_ms'])")"
  done
done; done
