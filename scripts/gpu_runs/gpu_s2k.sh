# round 2: ring19 fused (default) vs partitioned dedup, and ring18 at 2 shards
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra"
timeout 900 python bench.py $Q --dedup > gpurun_out/s2k_ring19_dedup.json 2> gpurun_out/s2k_ring19_dedup.err
timeout 900 python bench.py $Q --workload ring18 --shards 2 --dedup > gpurun_out/s2k_ring18_dedup.json 2> gpurun_out/s2k_ring18_dedup.err
timeout 900 python bench.py $Q --workload ring18 --shards 2 > gpurun_out/s2k_ring18_fused.json 2> gpurun_out/s2k_ring18_fused.err
for f in gpurun_out/s2k_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.3g'%d['value'], d['ms_per_step'], d['probes_per_step'])"; done
tail -3 gpurun_out/s2k_ring19_dedup.err
