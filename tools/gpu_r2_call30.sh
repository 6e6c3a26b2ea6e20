# C2 diagnostics: CTA timeline of the masked kernels (trace build) and the
# e2e host-API chunk / stream sweep, sync pair and async pipelined pair
mkdir -p gpurun_out/c30
python -c "import paper_1803_04880_b200 as se; se.build(force=True, defines=('SE_TRACE',), out='variants/v_trace.so')" > gpurun_out/c30/build.log 2>&1
SE_LIB_PATH=variants/v_trace.so timeout 300 python tools/cta_trace.py > gpurun_out/c30/trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/c30/trace.txt
for c in 512 1024 2048 4096; do for s in 3 4 6; do
  timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --no-variants --e2e-steps 30 --e2e-chunk-kib $c --e2e-streams $s > gpurun_out/c30/e2e.json 2>/dev/null
  echo "chunk=${c}KiB streams=$s $(python -c "import json;d=json.load(open('gpurun_out/c30/e2e.json'))['e2e'];print(d['value'], d['ms_per_step'], d['pipelined_variant']['value'], d['pipelined_variant']['ms_per_step'])")"
done; done
