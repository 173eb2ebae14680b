set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0 --workload ring16 --load 0.5 --hash-functions 8"
for v in default prefetch default prefetch; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r2f_${v}_$RANDOM.json 2>&1
done
