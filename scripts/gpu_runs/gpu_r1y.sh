set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline"
timeout 900 $B > gpurun_out/r1y_w4.json 2>&1
timeout 900 $B --shards 5 > gpurun_out/r1y_w5.json 2>&1
GX_LIB=$PWD/build_variants/routeall.so timeout 900 $B > gpurun_out/r1y_routeall_w4.json 2>&1
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -2 > gpurun_out/r1y_tests.log
