mkdir -p gpurun_out/c41
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/c41/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c41/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c41/smoke.txt 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/c41/smoke.txt
