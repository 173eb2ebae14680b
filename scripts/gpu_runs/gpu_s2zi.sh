# round 2: configs[2] peterson6: where the level kernel's time goes
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_level_staged" -s 50 -c 1 -o gpurun_out/s2zi_prof_peterson6 python scripts/prof_peterson.py > gpurun_out/s2zi_ncu.log 2>&1
timeout 300 python scripts/prof_peterson.py
