# round 2: one mid-run K2 (k_absorb_dedup) launch, ring14, full capture
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_absorb_dedup" -s 60 -c 1 -o gpurun_out/s2j_k2_ring14 python scripts/prof_dedup.py 14 1 > gpurun_out/s2j_ncu.log 2>&1
