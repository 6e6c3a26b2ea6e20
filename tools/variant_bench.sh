# bench every variants/*.so (tuning builds of libse.so); parity of each vs oracle on C2 via smoke-like check
mkdir -p gpurun_out
for v in variants/*.so; do
  SE_LIB_PATH=$v timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-comparator --e2e-steps 2 --soak 0.5 > gpurun_out/vb.json 2>gpurun_out/vb.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/vb.json'));print(d['protect_gbs'], d['recover_gbs'], d['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  SE_LIB_PATH=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "protect_recover_parity and random" 2>&1 | tail -1
done
