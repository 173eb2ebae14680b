# round 2: K1 with the process-parallel expansion, one mid-run launch (ring14)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_level_part" -s 40 -c 1 -o gpurun_out/s2h_k1pp_ring14 python scripts/prof_dedup.py 14 1 > gpurun_out/s2h_ncu.log 2>&1
