# round-2 evidence: the default bench line, the reference arm, the ncu launch list of
# the bench command, and --set full captures of the masked and PUBLIC_PLAIN kernels on C4
mkdir -p gpurun_out/ev12
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/ev12/bench_default.json 2> gpurun_out/ev12/bench_default.err; echo "default rc=$?"
tail -c 600 gpurun_out/ev12/bench_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev12/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/ev12/bench_ref.json
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 1"
$CMD > gpurun_out/ev12/short.log 2>&1 && echo short ok && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/ev12/launches.csv $CMD > gpurun_out/ev12/ncu_ll.log 2>&1 && echo ll ok
CM="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0 --no-variants"
$CM > gpurun_out/ev12/m.log 2>&1 && echo m ok && \
ncu --set full --clock-control none --import-source on -k regex:"k_(protect|recover)_block8|k_cipher_ctr" -s 16 -c 4 -o gpurun_out/ev12/c4_masked $CM > gpurun_out/ev12/ncu_m.log 2>&1 && echo ncu-m ok
CP="python bench.py --plain --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CP > gpurun_out/ev12/p.log 2>&1 && echo p ok && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 8 -c 2 -o gpurun_out/ev12/c4_plain $CP > gpurun_out/ev12/ncu_p.log 2>&1 && echo ncu-p ok
# C2 / C3 / C5 / C4-FULL lines (device-resident, masked with the PUBLIC_PLAIN variant where available)
for a in "--config 2" "--config 3" "--config 5" "--config 4 --full"; do
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $a > "gpurun_out/ev12/bench_$(echo $a | tr -d ' -').json" 2>&1; echo "$a rc=$?"
done
for l in 1 2; do
  timeout 600 python bench.py --dct $l --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ev12/bench_dct$l.json 2>&1; echo "dct$l rc=$?"
done
