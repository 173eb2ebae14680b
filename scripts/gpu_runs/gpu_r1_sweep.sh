set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -5 > gpurun_out/gpu_tests5.log
for g in 0 1 2 4; do timeout 200 python bench.py --workload ring14 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --probe-group $g > gpurun_out/b5_ring14_g$g.json 2>&1; done
for bw in 4 8 16; do timeout 200 python bench.py --workload ring14 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --bucket-words $bw --hash-functions 32 --load 0.4 > gpurun_out/b5_ring14_bw$bw.json 2>&1; done
timeout 300 python bench.py --workload ring16 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b5_ring16.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_level -s 45 -c 1 -o gpurun_out/prof5_ring14_lvl python bench.py --workload ring14 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
