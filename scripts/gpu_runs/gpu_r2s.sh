# last full pass of the round: GPU tests, smoke, default bench (with the vlen-2 duplication sweep)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4 > gpurun_out/r2s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
