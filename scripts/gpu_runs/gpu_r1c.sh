# A/B: block-local cache and concurrent CAS; parity subset first
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -5 > gpurun_out/r1c_tests.log
for c in 1 1024 4096 8192; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --cache-slots $c > gpurun_out/r1c_ring16_c$c.json 2>&1; done
for g in 1 4; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --probe-group $g > gpurun_out/r1c_ring16_g$g.json 2>&1; done
for bw in 4 8 16; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --bucket-words $bw --hash-functions 32 --load 0.4 > gpurun_out/r1c_ring16_bw$bw.json 2>&1; done
timeout 600 python bench.py --workload ring17 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r1c_ring17.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level -s 60 -c 1 -o gpurun_out/r1c_prof_ring16 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
