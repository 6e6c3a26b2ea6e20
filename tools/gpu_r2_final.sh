# final round-2 check: pytest -m gpu, smoke(), and the C4-FULL line after the last FULL change
mkdir -p gpurun_out/final
bash tools/gpu_r2_call41.sh
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config 4 --full > gpurun_out/final/bench_config4full.json 2>&1; echo "c4full rc=$?"
