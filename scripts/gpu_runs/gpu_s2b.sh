# round 2: full ncu capture of one k_level_routed and one k_absorb launch of the 2-shard ring19 default (source-level)
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/s2b_prof_default python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra > gpurun_out/s2b_ncu.log 2>&1
tail -5 gpurun_out/s2b_ncu.log
