set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for v in default q1536 q2048; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r1k_${v}_bw32.json 2>&1
  timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1k_${v}_bw8.json 2>&1
done
unset GX_LIB
for c in 1 512; do timeout 300 $B --cache-slots $c > gpurun_out/r1k_c${c}_bw32.json 2>&1; done
timeout 900 python bench.py --workload ring18 --steps 2 --warmup 2 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1k_ring18.json 2> gpurun_out/r1k_ring18.err
timeout 1200 python bench.py --workload ring19 --load 0.75 --hash-functions 32 --steps 2 --warmup 2 --no-cpu-baseline --no-hash-bench --e2e-steps 1 > gpurun_out/r1k_ring19.json 2> gpurun_out/r1k_ring19.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4 > gpurun_out/r1k_tests.log
