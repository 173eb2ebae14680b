set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload ring14 --load 0.5 --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2j_extra.json 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3 > gpurun_out/r2j_tests.log
