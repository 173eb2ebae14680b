set -x
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload ring14 --shards 2 --steps 2 --warmup 2 --e2e-steps 1 > gpurun_out/r2e_2rank_2local.json 2> gpurun_out/r2e_2rank_2local.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_level --csv --log-file gpurun_out/r2e_traffic_ring16.csv python bench.py --workload ring16 --load 0.5 --hash-functions 8 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level_staged -s 60 -c 1 -o gpurun_out/r2e_prof_ring16 python bench.py --workload ring16 --load 0.5 --hash-functions 8 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-hash-bench > /dev/null 2>&1
