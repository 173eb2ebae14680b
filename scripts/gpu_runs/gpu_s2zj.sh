# round 2: rule targets without division for combination 0 (peterson6, ring19); parity subset
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 900 -x 2>&1 | tail -2 > gpurun_out/s2zj_tests.log
cat gpurun_out/s2zj_tests.log
for v in new base; do
  if [ $v = base ]; then export GX_LIB=$PWD/build_variants/libgx_base.so; fi
  for i in 1 2 3; do timeout 300 python scripts/prof_peterson.py; done > gpurun_out/s2zj_pet_$v.txt 2>&1
  timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0 > gpurun_out/s2zj_ring19_$v.json 2>&1
  unset GX_LIB
done
for v in new base; do echo $v; grep -v Warn gpurun_out/s2zj_pet_$v.txt | grep -v build_network; python -c "
import json; d=json.loads(open('gpurun_out/s2zj_ring19_$v.json').read().strip().splitlines()[-1]); print('ring19', '%.4g'%d['value'])"; done
