set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra"
timeout 900 $B --inbox-frac 0.24 > gpurun_out/r2k_inbox24.json 2>&1
timeout 900 $B --shards 3 --inbox-frac 0.2 > gpurun_out/r2k_w3.json 2>&1
timeout 900 $B --bucket-words 16 > gpurun_out/r2k_bw16.json 2>&1
