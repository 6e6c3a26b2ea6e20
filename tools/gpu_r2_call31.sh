mkdir -p gpurun_out/c31
python -c "import paper_1803_04880_b200 as se; se.build(force=True, defines=('SE_TRACE',), out='variants/v_trace.so')" > gpurun_out/c31/build.log 2>&1
SE_LIB_PATH=variants/v_trace.so PYTHONPATH=. timeout 300 python tools/cta_trace.py > gpurun_out/c31/trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/c31/trace.txt
timeout 600 python tools/e2e_c2_probe.py 2>&1 | tee gpurun_out/c31/probe.txt
