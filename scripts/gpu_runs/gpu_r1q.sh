set -x
mkdir -p gpurun_out
timeout 600 python scripts/ra_alloc.py > gpurun_out/r1q_alloc.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
timeout 300 $B > gpurun_out/r1q_bw32.json 2>&1
