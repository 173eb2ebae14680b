set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.free --format=csv > gpurun_out/r1i_mem.txt
timeout 900 python bench.py --workload ring18 --steps 2 --warmup 2 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1i_ring18.json 2> gpurun_out/r1i_ring18.err
timeout 1200 python bench.py --workload ring19 --load 0.75 --hash-functions 32 --steps 2 --warmup 2 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1i_ring19.json 2> gpurun_out/r1i_ring19.err
