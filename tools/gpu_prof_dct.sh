# ncu captures of the row-f3 DCT kernels (4800x4800 grey): plain run first,
# then one --set full capture of protect and recover at level $LEVEL
mkdir -p gpurun_out
LEVEL=${LEVEL:-1}
TAG=${TAG:-dct$LEVEL}
python tools/prof_dct.py $LEVEL > gpurun_out/plain_$TAG.log 2>&1 && echo plain ok && \
ncu --set full --clock-control none --import-source on -k regex:k_dct_ -s 2 -c 2 -o gpurun_out/$TAG \
    python tools/prof_dct.py $LEVEL > gpurun_out/ncu_$TAG.log 2>&1 && echo ncu ok
tail -2 gpurun_out/ncu_$TAG.log
