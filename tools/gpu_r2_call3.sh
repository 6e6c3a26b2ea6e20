# round-2 call 3: first run of the persistent tile kernels
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tile.py -x -q 2>&1 | tail -25 > gpurun_out/tile_tests.log; cat gpurun_out/tile_tests.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 2>&1 | tail -c 1500
timeout 300 python bench.py --plain --steps 10 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 2>&1 | tail -c 1500
