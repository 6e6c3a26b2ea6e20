# Round evidence on one B200: tests, smoke, bench lines, ncu launch list + full captures.
mkdir -p gpurun_out/ev
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/ev/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/ev/host.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/ev/pytest_gpu.txt
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1 | tee gpurun_out/ev/smoke.txt
timeout 600 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --plain --no-cpu-baseline > gpurun_out/ev/bench_plain.json 2>> gpurun_out/ev/bench.err
timeout 900 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/ev/bench_c4.json 2>> gpurun_out/ev/bench.err
timeout 900 python bench.py --config 4 --stripes --full --steps 5 > gpurun_out/ev/bench_c4_full_stripes.json 2>> gpurun_out/ev/bench.err
timeout 900 python bench.py --config 5 --steps 5 > gpurun_out/ev/bench_c5.json 2>> gpurun_out/ev/bench.err
timeout 900 python bench.py --config 3 --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev/bench_c3.json 2>> gpurun_out/ev/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ev/bench_ref.json 2>> gpurun_out/ev/bench.err
timeout 600 python bench.py --dct 1 --steps 100 > gpurun_out/ev/bench_dct_level1.json 2>> gpurun_out/ev/bench.err
timeout 600 python bench.py --dct 2 --steps 100 --no-cpu-baseline > gpurun_out/ev/bench_dct_level2.json 2>> gpurun_out/ev/bench.err
CMD="python bench.py --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CMD > gpurun_out/ev/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/ev/launches.csv $CMD > gpurun_out/ev/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_protect_block8 -s 2 -c 1 -o gpurun_out/ev/protect $CMD > gpurun_out/ev/ncu_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_recover_block8 -s 2 -c 1 -o gpurun_out/ev/recover $CMD > gpurun_out/ev/ncu_r.log 2>&1
CMD2="python tools/prof_cipher.py"
$CMD2 > gpurun_out/ev/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cipher_ctr -s 2 -c 1 -o gpurun_out/ev/cipher $CMD2 > gpurun_out/ev/ncu_c.log 2>&1
CMD3="python tools/prof_dct.py 1"
$CMD3 > gpurun_out/ev/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dct_protect -s 1 -c 1 -o gpurun_out/ev/dct1_protect $CMD3 > gpurun_out/ev/ncu_d1p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dct_recover -s 1 -c 1 -o gpurun_out/ev/dct1_recover $CMD3 > gpurun_out/ev/ncu_d1r.log 2>&1
CMD5="python tools/prof_full.py"
$CMD5 > gpurun_out/ev/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dwt_full_fwd -s 1 -c 1 -o gpurun_out/ev/full_fwd $CMD5 > gpurun_out/ev/ncu_ff.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dwt_full_inv -s 1 -c 1 -o gpurun_out/ev/full_inv $CMD5 > gpurun_out/ev/ncu_fi.log 2>&1
CMD4="python tools/prof_dct.py 2"
$CMD4 > gpurun_out/ev/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dct_protect -s 1 -c 1 -o gpurun_out/ev/dct2_protect $CMD4 > gpurun_out/ev/ncu_d2p.log 2>&1
# summarise here (ncu -i) and drop the large reports: gpurun returns <= 64 MiB
python tools/make_profiles.py gpurun_out/ev gpurun_out/evp round1 > gpurun_out/ev/make_profiles.log 2>&1
du -sh gpurun_out/ev/*.ncu-rep 2>/dev/null | tail -20 > gpurun_out/ev/rep_sizes.txt
rm -f gpurun_out/ev/*.ncu-rep
echo evidence done
ls gpurun_out/ev gpurun_out/evp
