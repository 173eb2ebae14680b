# round 2: ncu evidence at the final code (block cache of any slot count): launch list with DRAM bytes of
# one default ring19 run, full captures of k_level_routed + k_absorb, per-line source page of k_level_routed
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2zt_launches_ring19.csv $B > gpurun_out/s2zt_l.log 2>&1
python scripts/launch_table.py gpurun_out/s2zt_launches_ring19.csv | head -8
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/s2zt_prof_ring19 $B > gpurun_out/s2zt_ncu.log 2>&1
tail -n 3 gpurun_out/s2zt_ncu.log; ls -la gpurun_out | grep s2zt
