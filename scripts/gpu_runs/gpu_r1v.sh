set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r1v_default.json 2> gpurun_out/r1v_default.err
timeout 600 python bench.py --workload ring16 --load 0.5 --hash-functions 8 --no-hash-bench --no-cpu-baseline > gpurun_out/r1v_ring16.json 2> gpurun_out/r1v_ring16.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1v_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
