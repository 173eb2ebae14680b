# round 2: full GPU suite + smoke at the grouped-expansion state, and a --set full capture of the routed/absorb kernels
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -6 > gpurun_out/s2u_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2u_smoke.log 2>&1
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 600 -c 2 -o gpurun_out/s2u_prof_ring19 $B > gpurun_out/s2u_ncu.log 2>&1
cat gpurun_out/s2u_tests.log gpurun_out/s2u_smoke.log
