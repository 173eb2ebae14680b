# round 2: TMA bucket staging + merged filter/route: parity subset, then A/B (TMA vs cp.async) on ring16 (1 table) and ring19 (2 shards)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3 > gpurun_out/s2o_tests.log
cat gpurun_out/s2o_tests.log
Q="--steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in tma notma; do
  if [ $v = notma ]; then export GX_LIB=$PWD/build_variants/libgx_notma.so; fi
  timeout 600 python bench.py $Q --workload ring16 > gpurun_out/s2o_ring16_$v.json 2>&1
  timeout 900 python bench.py $Q > gpurun_out/s2o_ring19_$v.json 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2o_ring*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.4g'%d['value'], round(d['ms_per_step'],1), round(d['roofline']['frac'],3))" || tail -3 $f; done
