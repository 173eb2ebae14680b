# round 2: L2 prefetch of the next round's first buckets in probe_refill (default) vs none (GX_PREFETCH=0)
mkdir -p gpurun_out
Q="--steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for v in pf nopf; do
  if [ $v = nopf ]; then export GX_LIB=$PWD/build_variants/libgx_nopf.so; fi
  timeout 600 python bench.py $Q --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/s2zr_ring16_$v.json 2>&1
  timeout 900 python bench.py $Q > gpurun_out/s2zr_ring19_$v.json 2>&1
  timeout 600 python scripts/prof_peterson.py > gpurun_out/s2zr_pet_$v.txt 2>&1
  unset GX_LIB
done
for f in gpurun_out/s2zr_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'], d.get('digest',{}).get('equal'))" || tail -n 3 $f; done
for f in gpurun_out/s2zr_pet_*.txt; do echo $f; tail -n 1 $f; done
