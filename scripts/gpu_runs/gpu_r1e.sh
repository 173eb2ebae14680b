set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -k "contention or closed_forms or bucket_sizes" 2>&1 | tail -8 > gpurun_out/r1e_tests.log
for c in 1 2048; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --cache-slots $c > gpurun_out/r1e_ring16_c$c.json 2>&1; done
for bw in 4 8 16; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --bucket-words $bw --hash-functions 32 --load 0.4 > gpurun_out/r1e_ring16_bw$bw.json 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r1e_full.json 2> gpurun_out/r1e_full.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level -s 60 -c 1 -o gpurun_out/r1e_prof_ring16 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
