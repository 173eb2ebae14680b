# round 2: cost of the worst-case chunk bound: ring19 with chunks sized for 16 / 24 successors per state instead of 38
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for c in 24 16; do
  GX_CHUNK_SUCC=$c timeout 900 python bench.py $Q > gpurun_out/s2x_ring19_chunk$c.json 2>&1
done
for f in gpurun_out/s2x_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['gpu_launches'])" || tail -3 $f; done
