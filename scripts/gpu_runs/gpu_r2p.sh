set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra"
timeout 900 $B --shards 2 --inbox-frac 0.3 > gpurun_out/r2p_w2.json 2>&1
timeout 900 $B > gpurun_out/r2p_w3.json 2>&1
timeout 900 $B --shards 4 > gpurun_out/r2p_w4.json 2>&1
