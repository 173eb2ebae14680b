# staging-shape sweep: KB_MAX 64/128(default)/256, 4 KB stage; bw 4/8/32
set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for v in default kb64 kb256 st4k; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r1f_${v}_bw32.json 2>&1
  for bw in 4 8; do timeout 300 $B --bucket-words $bw --hash-functions 32 --load 0.4 > gpurun_out/r1f_${v}_bw$bw.json 2>&1; done
done
unset GX_LIB
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4 > gpurun_out/r1f_tests.log
