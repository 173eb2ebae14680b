# round 2: overlapped level body, successors per probe round 64 / 256 (default build 128, previous body = noov)
mkdir -p gpurun_out
Q="--steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0 --workload ring16 --load 0.5 --hash-functions 8"
for v in ov64 ov256 noov; do
  GX_LIB=$PWD/build_variants/libgx_$v.so timeout 600 python bench.py $Q > gpurun_out/s2zq_ring16_$v.json 2>&1
done
for f in gpurun_out/s2zq_ring*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d.get('digest',{}).get('equal'))" || tail -3 $f; done
