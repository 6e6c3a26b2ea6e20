# All bench lines of the round evidence (no profiler): gpurun_out/evb/bench*.json
mkdir -p gpurun_out/evb
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python bench.py > gpurun_out/evb/bench.json 2> gpurun_out/evb/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --plain --no-cpu-baseline > gpurun_out/evb/bench_plain.json 2>> gpurun_out/evb/bench.err
timeout 900 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/evb/bench_c4.json 2>> gpurun_out/evb/bench.err
timeout 900 python bench.py --config 4 --stripes --full --steps 5 > gpurun_out/evb/bench_c4_full_stripes.json 2>> gpurun_out/evb/bench.err
timeout 900 python bench.py --config 5 --steps 5 > gpurun_out/evb/bench_c5.json 2>> gpurun_out/evb/bench.err
timeout 900 python bench.py --config 3 --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/evb/bench_c3.json 2>> gpurun_out/evb/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/evb/bench_ref.json 2>> gpurun_out/evb/bench.err
timeout 600 python bench.py --dct 1 --steps 100 > gpurun_out/evb/bench_dct_level1.json 2>> gpurun_out/evb/bench.err
timeout 600 python bench.py --dct 2 --steps 100 --no-cpu-baseline > gpurun_out/evb/bench_dct_level2.json 2>> gpurun_out/evb/bench.err
timeout 300 python tools/time_full.py > gpurun_out/evb/time_full.txt 2>&1
echo benches done
