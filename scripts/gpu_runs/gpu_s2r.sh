# round 2: grouped expansion: parity (expand KATs, explore goldens, shards, digests) + A/B vs per-process expansion
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_digest.py -m gpu -q -p no:cacheprovider --timeout 900 -x 2>&1 | tail -3 > gpurun_out/s2r_tests.log
cat gpurun_out/s2r_tests.log
Q="--steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --crosscheck 0"
for v in group nogroup; do
  if [ $v = nogroup ]; then export GX_LIB=$PWD/build_variants/libgx_nogroup.so; fi
  timeout 600 python bench.py $Q --workload ring16 > gpurun_out/s2r_ring16_$v.json 2>&1
  timeout 900 python bench.py $Q --no-extra > gpurun_out/s2r_ring19_$v.json 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2r_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); x=d.get('extra_workloads') or []
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), [(e['workload'], round(e['ms_per_exploration'],1)) for e in x])" || tail -3 $f; done
