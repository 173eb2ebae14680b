# round 2: partitioned engine after the K2 batch rewrite: launch list + timings
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/s2i_launches_ring14.csv python scripts/prof_dedup.py 14 1 > gpurun_out/s2i_l.log 2>&1
timeout 900 python scripts/dedup_check.py ring14 ring16 > gpurun_out/s2i_dedup.txt 2>&1
grep -v "UserWarn\|return build" gpurun_out/s2i_dedup.txt | tail -9
