# profile the protect kernel of the given lib ($SE_LIB_PATH or default) — plain run first
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 2"
TAG=${TAG:-prof}
$CMD > gpurun_out/plain_$TAG.log 2>&1 && echo plain ok && \
ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_protect_block8} -s 3 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1 && echo ncu ok
tail -2 gpurun_out/ncu_$TAG.log
