set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -2 > gpurun_out/r2c_tests.log
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline"
timeout 900 $B > gpurun_out/r2c_default.json 2>&1
timeout 900 $B --inbox-frac 0.18 > gpurun_out/r2c_inbox18.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload ring14 --steps 2 --warmup 2 --e2e-steps 1 > gpurun_out/r2c_2rank.json 2> gpurun_out/r2c_2rank.err
