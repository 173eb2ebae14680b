# round 2: evidence for the headline (2-shard ring19 default): launch list with DRAM bytes of one exploration,
# and --set full captures of one k_level_routed and one k_absorb launch mid-run
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2q_launches_ring19.csv $B > gpurun_out/s2q_l.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/s2q_prof_ring19 $B > gpurun_out/s2q_ncu.log 2>&1
ls -la gpurun_out/ | grep s2q
