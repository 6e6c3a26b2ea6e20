# NVTX ranges: ncu selects the kernels of one library call by its range name
mkdir -p gpurun_out/c54
python tools/nvtx_probe.py && \
for call in fragment_recover cipher_encrypt fragment_protect; do
  timeout 600 ncu --nvtx --nvtx-include "$call/" --metrics gpu__time_duration.sum --csv python tools/nvtx_probe.py > gpurun_out/c54/ncu_$call.csv 2>&1; echo "$call rc=$?"
  grep -o 'se::k_[a-z_0-9]*<[^>]*>' gpurun_out/c54/ncu_$call.csv | sort | uniq -c
done
