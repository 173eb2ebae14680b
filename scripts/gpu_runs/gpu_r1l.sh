# single-pass emission: parity (default + tiny-queue stress build), A/B, profile
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4 > gpurun_out/r1l_tests.log
GX_LIB=$PWD/build_variants/q64.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 300 -x -k "explore or contention or closed or bucket or sharded or generated or deadlock" 2>&1 | tail -4 > gpurun_out/r1l_tests_q64.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
timeout 300 $B > gpurun_out/r1l_bw32.json 2>&1
timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1l_bw8.json 2>&1
GX_LIB=$PWD/build_variants/q2048.so timeout 300 $B > gpurun_out/r1l_q2048_bw32.json 2>&1
GX_LIB=$PWD/build_variants/q2048.so timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1l_q2048_bw8.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level -s 60 -c 1 -o gpurun_out/r1l_prof_ring16 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
