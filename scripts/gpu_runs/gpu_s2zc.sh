# round 2: refill probe: load factor 0.8 / 0.85 / 0.9 on ring19 (2 shards)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for l in 0.85 0.9; do timeout 900 python bench.py $Q --load $l > gpurun_out/s2zc_ring19_l$l.json 2>&1; done
timeout 900 python bench.py $Q --load 0.85 --shards 3 > gpurun_out/s2zc_ring19_l0.85_s3.json 2>&1
for f in gpurun_out/s2zc_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), round(d['config']['table_bytes']/2**30,1), d['probes_per_step'])" || tail -3 $f; done
