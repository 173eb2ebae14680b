set -x
mkdir -p gpurun_out
timeout 600 python scripts/shard_time.py 16 1,2,3,4 > gpurun_out/r1s_shard16.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s_shard_launches.csv python scripts/shard_time.py 16 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 300 -c 2 -o gpurun_out/r1s_prof_shard python scripts/shard_time.py 16 3 > /dev/null 2>&1
