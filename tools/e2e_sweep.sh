# e2e (host API) chunk-size / stream-count sweep on C2
for c in ${CHUNKS:-512 1024 2048 4096 8192}; do for s in ${STREAMS:-4}; do
  python bench.py --steps 5 --warmup 3 --soak 0 --no-cpu-baseline --no-comparator --e2e-steps 30 --e2e-chunk-kib $c --e2e-streams $s > gpurun_out/e2e.json 2>/dev/null
  echo "chunk=${c}KiB streams=$s $(python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print(d['e2e']['value'], d['e2e']['ms_per_step'])")"
done; done
