# round 2, first call: GPU tests, smoke, default bench (baseline of this round)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2a_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -15 > gpurun_out/s2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1
timeout 1800 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err
