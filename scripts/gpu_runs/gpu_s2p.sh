# round 2: ring19 load factor x shard count sweep (cp.async staging, merged filter/route)
mkdir -p gpurun_out
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
for cfg in "0.75 2" "0.8 2" "0.85 2" "0.8 3" "0.85 3"; do
  set -- $cfg
  timeout 900 python bench.py $Q --load $1 --shards $2 > gpurun_out/s2p_ring19_l$1_s$2.json 2>&1
done
for f in gpurun_out/s2p_ring19*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['probes_per_step'], round(d['config']['table_bytes']/2**30,1), d['roofline']['random_access_table_size'])" || tail -3 $f; done
