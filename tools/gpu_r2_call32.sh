mkdir -p gpurun_out/c32
OUT=gpurun_out/c32 timeout 600 python tools/e2e_timeline.py > gpurun_out/c32/timeline.txt 2>&1; echo "rc=$?"
head -c 3000 gpurun_out/c32/timeline.txt
