set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -30 > gpurun_out/r1g_shard_tests.log
timeout 600 python scripts/shard_time.py 14 1,2,4,8 > gpurun_out/r1g_shard_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4 > gpurun_out/r1g_tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 > gpurun_out/r1g_ring16.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1g_ring16_bw8.json 2>&1
