set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
timeout 300 $B --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/r2b_ring16.json 2>&1
timeout 300 $B --workload ring16 --load 0.4 --bucket-words 8 > gpurun_out/r2b_ring16_bw8.json 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2b_default.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -2 > gpurun_out/r2b_tests.log
