set -x
mkdir -p gpurun_out
timeout 2400 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
