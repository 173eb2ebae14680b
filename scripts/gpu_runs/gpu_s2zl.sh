# round 2: cross-process barrier waits for the shard stream (IPC test x4); cache of any slot count (~1000 vs 512)
mkdir -p gpurun_out
for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "two_processes" 2>&1 | tail -1; done > gpurun_out/s2zl_ipc.log
cat gpurun_out/s2zl_ipc.log
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in any pow2; do
  if [ $v = pow2 ]; then export GX_LIB=$PWD/build_variants/libgx_pow2cache.so; fi
  timeout 900 python bench.py $Q > gpurun_out/s2zl_ring19_$v.json 2>&1
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zl_ring16_$v.json 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zl_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'])" || tail -3 $f; done
