# round 2: 4 resident blocks per SM (64 registers, 512-word queues) vs the default 3 (grouped expansion)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
export GX_LIB=$PWD/build_variants/libgx_m4q512.so
timeout 900 python bench.py $Q > gpurun_out/s2t_ring19_m4q512.json 2>&1
timeout 600 python bench.py $Q --workload ring16 > gpurun_out/s2t_ring16_m4q512.json 2>&1
timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2t_ring16l5_m4q512.json 2>&1
unset GX_LIB
timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2t_ring16l5_default.json 2>&1
for f in gpurun_out/s2t_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1))" || tail -3 $f; done
