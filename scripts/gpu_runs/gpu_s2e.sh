# round 2: where the partitioned dedup engine spends its time (ring14 launch list, ring16 full capture of K1/K2)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2e_launches_ring14.csv python scripts/prof_dedup.py 14 1 > gpurun_out/s2e_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_level_part|k_absorb_dedup" -s 300 -c 2 -o gpurun_out/s2e_prof_ring16 python scripts/prof_dedup.py 16 1 > gpurun_out/s2e_ncu.log 2>&1
tail -3 gpurun_out/s2e_ncu.log
