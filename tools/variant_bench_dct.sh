# bench every variants/*.so on the row-f3 DCT path (levels 1 and 2), 4800x4800 protect/recover us
mkdir -p gpurun_out
for v in variants/*.so; do
  for l in 1 2; do
    SE_LIB_PATH=$v timeout 300 python bench.py --dct $l --steps 50 --warmup 5 --no-cpu-baseline --soak 0.5 > gpurun_out/vd.json 2>gpurun_out/vd.err
    echo "$v L$l rc=$? $(python -c "import json;d=json.load(open('gpurun_out/vd.json'));print([(r['image'], r['protect_ms'], r['recover_ms']) for r in d['per_image']])" 2>&1 | tail -1)"
  done
done
