# round 2: probe_refill judging the claim CAS one round later (GX_DEFER_CAS=1, default) vs at once; then the GPU suite
mkdir -p gpurun_out
Q="--steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in defer nodefer; do
  if [ $v = nodefer ]; then export GX_LIB=$PWD/build_variants/libgx_nodefer.so; fi
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zu_ring16_$v.json 2>&1
  timeout 900 python bench.py $Q > gpurun_out/s2zu_ring19_$v.json 2>&1
  timeout 600 python scripts/prof_peterson.py > gpurun_out/s2zu_pet_$v.txt 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zu_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'], d.get('digest',{}).get('equal'))" || tail -n 3 $f; done
for f in gpurun_out/s2zu_pet_*.txt; do echo $f; tail -n 1 $f; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2zu_tests.log 2>&1; tail -n 3 gpurun_out/s2zu_tests.log
