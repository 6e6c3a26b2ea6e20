set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 8 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
nproc
