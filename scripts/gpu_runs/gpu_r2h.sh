set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -4 > gpurun_out/r2h_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --no-extra"
timeout 300 $B --workload ring16 --load 0.5 --hash-functions 8 > gpurun_out/r2h_ring16.json 2>&1
timeout 300 $B --workload ring16 --load 0.4 --bucket-words 8 > gpurun_out/r2h_ring16_bw8.json 2>&1
timeout 600 python bench.py --workload ring14 --load 0.5 --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2h_extra.json 2>&1
