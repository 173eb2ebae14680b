set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline"
timeout 900 $B --shards 5 --inbox-frac 0.18 > gpurun_out/r1z_w5.json 2>&1
GX_LIB=$PWD/build_variants/routeall.so timeout 900 $B --inbox-frac 0.22 > gpurun_out/r1z_routeall_w4.json 2>&1
