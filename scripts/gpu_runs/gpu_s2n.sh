# round 2: oversubscribed N=2 bench line (both ranks on one GPU: CUDA IPC inboxes, gloo counters), all fields
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload ring16 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/s2n_bench_2ranks.json 2> gpurun_out/s2n_bench_2ranks.err
tail -3 gpurun_out/s2n_bench_2ranks.err
tail -c 3000 gpurun_out/s2n_bench_2ranks.json
