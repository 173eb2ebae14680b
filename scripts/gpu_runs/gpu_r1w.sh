set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -4 > gpurun_out/r1w_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1w_smoke.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-hash-bench --no-cpu-baseline > gpurun_out/r1w_default.json 2> gpurun_out/r1w_default.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_level_routed|k_absorb" -s 200 -c 2 -o gpurun_out/r1w_prof_ring19 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
