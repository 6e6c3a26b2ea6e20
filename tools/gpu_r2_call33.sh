mkdir -p gpurun_out/c33
for h in 1 0; do
  echo "== SE_HOST_HYBRID=$h"
  SE_HOST_HYBRID=$h NOCOPIES=1 CHUNKS="2048 3072 4096 6144" STREAMS="3 4" timeout 600 python tools/e2e_c2_probe.py 2>&1
done | tee gpurun_out/c33/probe.txt
SE_HOST_HYBRID=0 OUT=gpurun_out/c33 CHUNKS="4096 2048" timeout 600 python tools/e2e_timeline.py > gpurun_out/c33/timeline_h0.txt 2>&1
OUT=gpurun_out/c33 CHUNKS="4096" timeout 600 python tools/e2e_timeline.py > gpurun_out/c33/timeline_h1.txt 2>&1
grep "==" gpurun_out/c33/timeline_h*.txt
