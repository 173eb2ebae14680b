set -x
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload ring14 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r1h_2rank.json 2> gpurun_out/r1h_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --workload ring14 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r1h_4rank.json 2> gpurun_out/r1h_4rank.err
timeout 300 python bench.py --workload ring14 --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1h_1rank.json 2>&1
