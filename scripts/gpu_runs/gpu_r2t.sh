set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 2 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra --workload ring18 --load 0.5"
timeout 900 $B > gpurun_out/r2t_ring18.json 2>&1
timeout 900 $B --shards 2 > gpurun_out/r2t_ring18_w2.json 2>&1
