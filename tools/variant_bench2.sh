# bench every variants/*.so, masked and PUBLIC_PLAIN (C2), protect/recover GB/s
mkdir -p gpurun_out
for v in variants/*.so; do
  for m in "" "--plain"; do
    SE_LIB_PATH=$v timeout 300 python bench.py $m --steps 200 --warmup 5 --no-cpu-baseline --no-comparator --e2e-steps 0 --soak 0.5 > gpurun_out/vb.json 2>gpurun_out/vb.err
    echo "$v $m rc=$? $(python -c "import json;d=json.load(open('gpurun_out/vb.json'));print(d['protect_gbs'], d['recover_gbs'], d['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
