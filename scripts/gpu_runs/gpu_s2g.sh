# round 2: launch list of ring14 on the partitioned engine (K1 vs K2 time)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/s2g_launches_ring14.csv python scripts/prof_dedup.py 14 1 > gpurun_out/s2g_l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/s2g_launches_ring14_fused.csv python scripts/prof_dedup.py 14 1 fused > gpurun_out/s2g_lf.log 2>&1
