# round 2: overlapped level body (expansion during the probe rounds) vs the previous body (GX_OVERLAP=0)
mkdir -p gpurun_out
Q="--steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in ov noov; do
  if [ $v = noov ]; then export GX_LIB=$PWD/build_variants/libgx_noov.so; fi
  timeout 900 python bench.py $Q > gpurun_out/s2zp_ring19_$v.json 2>&1
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zp_ring16_$v.json 2>&1
  timeout 600 python scripts/prof_peterson.py > gpurun_out/s2zp_pet_$v.txt 2>&1
  timeout 600 python scripts/prof_peterson.py >> gpurun_out/s2zp_pet_$v.txt 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zp_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'], d.get('digest',{}).get('equal'))" || tail -3 $f; done
tail -2 gpurun_out/s2zp_pet_*.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2zp_tests.log 2>&1; tail -3 gpurun_out/s2zp_tests.log
