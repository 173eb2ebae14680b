# round 2: per-lane bucket staging vs cooperative (ring19 2 shards, ring16)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 900 python bench.py $Q > gpurun_out/s2v_ring19_coop.json 2>&1
timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2v_ring16_coop.json 2>&1
export GX_LIB=$PWD/build_variants/libgx_perlane.so
timeout 900 python bench.py $Q > gpurun_out/s2v_ring19_perlane.json 2>&1
timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2v_ring16_perlane.json 2>&1
unset GX_LIB
for f in gpurun_out/s2v_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1))" || tail -3 $f; done
