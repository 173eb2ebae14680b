# final round evidence (after the shard-count sweep): GPU tests, smoke, full default bench, reference arm
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4 > gpurun_out/r2q_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q_smoke.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2q_ref.json 2> gpurun_out/r2q_ref.err
