mkdir -p gpurun_out/c48
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py tests/test_gpu_no_alloc.py -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 > gpurun_out/c48/b.json 2>gpurun_out/c48/b.err
python -c "import json;t=open('gpurun_out/c48/b.json').read();d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]);print(d['value'], d['protect_gbs'], d['recover_gbs'], d['roofline']['frac'])"
