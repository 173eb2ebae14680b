set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3 > gpurun_out/r2o_tests.log
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline"
timeout 900 $B > gpurun_out/r2o_default.json 2>&1
