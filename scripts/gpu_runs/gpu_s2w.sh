# round 2: full default bench line (configs[3] + hash bench + extras + CPU baselines), reference arm, GPU suite, smoke
mkdir -p gpurun_out
timeout 2400 python bench.py > gpurun_out/s2w_bench.json 2> gpurun_out/s2w_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/s2w_ref.json 2> gpurun_out/s2w_ref.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -4 > gpurun_out/s2w_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2w_smoke.log 2>&1
cat gpurun_out/s2w_tests.log gpurun_out/s2w_smoke.log; tail -c 400 gpurun_out/s2w_ref.json; tail -3 gpurun_out/s2w_bench.err
