# round 2: full capture of K1 (k_level_part) on ring16, partitioned engine
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_level_part" -s 50 -c 1 -o gpurun_out/s2f_k1_ring16 python scripts/prof_dedup.py 16 1 > gpurun_out/s2f_ncu.log 2>&1
tail -2 gpurun_out/s2f_ncu.log
