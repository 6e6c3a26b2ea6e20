for rep in 1 2; do
bash tools/variant_bench_dct.sh 2>&1
done
