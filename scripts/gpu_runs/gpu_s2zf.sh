# round 2 final evidence at the final default (refill probe, load 0.8): bench line, reference arm,
# ncu launch list with DRAM bytes, full captures of k_level_routed + k_absorb
mkdir -p gpurun_out
timeout 2400 python bench.py > gpurun_out/s2zf_bench.json 2> gpurun_out/s2zf_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/s2zf_ref.json 2> gpurun_out/s2zf_ref.err
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2zf_launches_ring19.csv $B > gpurun_out/s2zf_l.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/s2zf_prof_ring19 $B > gpurun_out/s2zf_ncu.log 2>&1
tail -c 300 gpurun_out/s2zf_ref.json; ls gpurun_out | grep s2zf
