# quick GPU check: parity tests, smoke, bench (no profiler)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
