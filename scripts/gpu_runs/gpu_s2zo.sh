# round 2: e2e phase breakdown (ring19, 2 shards) and the oversubscribed N=2 bench line at the final code
mkdir -p gpurun_out
timeout 600 python scripts/e2e_phases.py --workload ring19 --reps 2 > gpurun_out/s2zo_e2e_phases.json 2> gpurun_out/s2zo_e2e_phases.err
tail -3 gpurun_out/s2zo_e2e_phases.err; cat gpurun_out/s2zo_e2e_phases.json
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload ring16 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/s2zo_bench_2ranks.json 2> gpurun_out/s2zo_bench_2ranks.err
tail -3 gpurun_out/s2zo_bench_2ranks.err
tail -c 1500 gpurun_out/s2zo_bench_2ranks.json
