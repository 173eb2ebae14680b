# round 2: absorb kernel without the block-local cache vs with (ring19 default)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 900 python bench.py $Q > gpurun_out/s2ze_ring19_abscache.json 2>&1
GX_LIB=$PWD/build_variants/libgx_noabscache.so timeout 900 python bench.py $Q > gpurun_out/s2ze_ring19_noabscache.json 2>&1
for f in gpurun_out/s2ze_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'])" || tail -3 $f; done
