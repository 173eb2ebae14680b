set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/r2n_prof_default python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra > /dev/null 2>&1
