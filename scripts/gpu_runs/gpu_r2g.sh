set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x -k peterson6 2>&1 | tail -3 > gpurun_out/r2g_tests.log
timeout 600 python bench.py --workload ring14 --load 0.5 --steps 2 --warmup 2 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
