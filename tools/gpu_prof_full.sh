# ncu capture of the FULL transform kernels (64 MiB, W = 8192, L = 2): plain
# run first, then one --set full capture of k_dwt_full_fwd and k_dwt_full_inv
mkdir -p gpurun_out
TAG=${TAG:-fullstream}
python tools/prof_full.py > gpurun_out/plain_$TAG.log 2>&1 && echo plain ok && \
ncu --set full --clock-control none --import-source on -k regex:k_dwt_full -s 2 -c 2 -o gpurun_out/$TAG \
    python tools/prof_full.py > gpurun_out/ncu_$TAG.log 2>&1 && echo ncu ok
tail -2 gpurun_out/ncu_$TAG.log
