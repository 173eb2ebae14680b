# staged rehash rounds: parity (default + tiny-queue build), ring16 A/B, ring19 at 150 GB
set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
timeout 300 $B > gpurun_out/r1m_bw32.json 2>&1
timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1m_bw8.json 2>&1
GX_LIB=$PWD/build_variants/kb32.so timeout 300 $B > gpurun_out/r1m_kb32_bw32.json 2>&1
GX_LIB=$PWD/build_variants/kb32.so timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1m_kb32_bw8.json 2>&1
timeout 300 $B --load 0.75 --hash-functions 32 > gpurun_out/r1m_bw32_l75.json 2>&1
timeout 1200 python bench.py --workload ring19 --load 0.75 --hash-functions 32 --steps 2 --warmup 2 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1m_ring19.json 2> gpurun_out/r1m_ring19.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4 > gpurun_out/r1m_tests.log
GX_LIB=$PWD/build_variants/q64.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 300 -x -k "explore or contention or closed or bucket or sharded or generated or deadlock" 2>&1 | tail -4 > gpurun_out/r1m_tests_q64.log
