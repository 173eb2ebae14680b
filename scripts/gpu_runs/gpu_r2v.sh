set -x
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --no-extra --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/r2v_ring16.json 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2v_default_ring19.json 2>&1
