mkdir -p gpurun_out/c35
SE_LIB_PATH=variants/v_trace.so PYTHONPATH=. timeout 300 python tools/cta_trace.py > gpurun_out/c35/trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/c35/trace.txt
