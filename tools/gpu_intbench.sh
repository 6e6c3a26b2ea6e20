mkdir -p gpurun_out
./tools/intbench > gpurun_out/intbench.json 2>&1; cat gpurun_out/intbench.json
