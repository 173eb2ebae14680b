# round 2: shard count at the final operating point (refill probe, load 0.8 / 0.85)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 900 python bench.py $Q --shards 3 > gpurun_out/s2zh_ring19_s3_l08.json 2>&1
timeout 900 python bench.py $Q --shards 4 > gpurun_out/s2zh_ring19_s4_l08.json 2>&1
timeout 900 python bench.py $Q --workload ring18 > gpurun_out/s2zh_ring18_auto_l08.json 2>&1
for f in gpurun_out/s2zh_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['config']['parallelism'][:30], round(d['config']['table_bytes']/2**30,1))" || tail -3 $f; done
