# round 2: successor queue 768 / 1280 words (the cache takes the rest of the shared-memory budget)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in q768 q1280; do
  export GX_LIB=$PWD/build_variants/libgx_$v.so
  timeout 900 python bench.py $Q > gpurun_out/s2zm_ring19_$v.json 2>&1
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zm_ring16_$v.json 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zm_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'])" || tail -3 $f; done
