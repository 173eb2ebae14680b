# round 2: slot walk with whole-slot compares vs the per-word walk; parity subset
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 900 -x 2>&1 | tail -2 > gpurun_out/s2zg_tests.log
cat gpurun_out/s2zg_tests.log
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in new old; do
  if [ $v = old ]; then export GX_LIB=$PWD/build_variants/libgx_oldwalk.so; fi
  timeout 900 python bench.py $Q > gpurun_out/s2zg_ring19_$v.json 2>&1
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zg_ring16_$v.json 2>&1
  timeout 600 python scripts/fill_check.py 32 32 > gpurun_out/s2zg_fill32_$v.txt 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zg_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1))" || tail -3 $f; done
for f in gpurun_out/s2zg_fill*.txt; do echo $f; cat $f | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print(d['fill'], '%.3g'%d['insert_ops_per_sec'], '%.3g'%d['lookup_ops_per_sec'])"; done
