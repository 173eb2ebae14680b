# round 2: refill probe: shard count / load recheck on ring19, then the full GPU suite
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 900 python bench.py $Q --shards 3 > gpurun_out/s2zb_ring19_s3.json 2>&1
timeout 900 python bench.py $Q --load 0.8 > gpurun_out/s2zb_ring19_l08.json 2>&1
timeout 900 python bench.py $Q --load 0.7 > gpurun_out/s2zb_ring19_l07.json 2>&1
for f in gpurun_out/s2zb_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1))" || tail -3 $f; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -3
