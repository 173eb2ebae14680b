set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3 > gpurun_out/r2u_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --workload ring16 --load 0.5 --hash-functions 8"
for v in default noqsm default noqsm; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r2u_${v}_$RANDOM.json 2>&1
done
unset GX_LIB
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2u_default_ring19.json 2>&1
GX_LIB=$PWD/build_variants/noqsm.so timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra > gpurun_out/r2u_noqsm_ring19.json 2>&1
