set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for f in 0 20 22 24; do timeout 300 $B --filter-log2 $f > gpurun_out/r1t_ring16_f$f.json 2>&1; done
for f in 0 23; do timeout 1200 python bench.py --workload ring19 --load 0.75 --hash-functions 32 --steps 1 --warmup 1 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --filter-log2 $f > gpurun_out/r1t_ring19_f$f.json 2>&1; done
timeout 600 python scripts/shard_time.py 16 1,3 > gpurun_out/r1t_shard16.log 2>&1
