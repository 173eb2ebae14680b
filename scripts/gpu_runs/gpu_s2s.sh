# round 2: group-bits and cache sweep with the grouped expansion (ring19 2 shards, ring16 one table)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in g8 g10 g12; do
  if [ $v != g10 ]; then export GX_LIB=$PWD/build_variants/libgx_$v.so; fi
  timeout 900 python bench.py $Q > gpurun_out/s2s_ring19_$v.json 2>&1
  timeout 600 python bench.py $Q --workload ring16 > gpurun_out/s2s_ring16_$v.json 2>&1
  unset GX_LIB
done
timeout 900 python bench.py $Q --cache-slots 1 > gpurun_out/s2s_ring19_nocache.json 2>&1
timeout 900 python bench.py $Q --cache-slots 16384 > gpurun_out/s2s_ring19_cache16k.json 2>&1
for f in gpurun_out/s2s_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'])" || tail -3 $f; done
