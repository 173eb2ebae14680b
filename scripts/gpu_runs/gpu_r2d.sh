# the round's headline evidence: full default bench, reference arm, launch list, ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r2d_smi.txt 2>&1
timeout 1800 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2d_ref.json 2> gpurun_out/r2d_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 800 -c 2 -o gpurun_out/r2d_prof_default python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
