# last full default bench of the round (hash bench at the survey's sizes)
set -x
mkdir -p gpurun_out
timeout 2400 python bench.py > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1
