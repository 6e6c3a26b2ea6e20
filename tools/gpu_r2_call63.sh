mkdir -p gpurun_out/c63
CF="python bench.py --config 4 --full --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 0"
$CF > gpurun_out/c63/f.log 2>&1 && echo f ok && \
timeout 1200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(protect|recover)_full|k_dwt_full" --csv $CF > gpurun_out/c63/ncu_full.csv 2>&1; echo "ncu rc=$?"
grep -v "^==" gpurun_out/c63/ncu_full.csv | python3 -c "
import csv,sys,collections
rows=list(csv.reader(sys.stdin))
h=rows[0]; d=collections.defaultdict(dict)
for r in rows[1:]:
    if len(r)<len(h): continue
    d[(r[h.index('ID')], r[h.index('Kernel Name')][:40])][r[h.index('Metric Name')]]=r[h.index('Metric Value')]
for k,v in list(d.items())[-8:]: print(k, v)
"
