set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra"
timeout 900 $B > gpurun_out/r2l_default.json 2>&1
timeout 900 $B --inbox-frac 0.3 > gpurun_out/r2l_inbox30.json 2>&1
timeout 900 $B --shards 2 --inbox-frac 0.3 > gpurun_out/r2l_w2.json 2>&1
