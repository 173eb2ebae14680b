set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline --no-extra"
for v in default m2kb64 q768; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 900 $B > gpurun_out/r2r_$v.json 2>&1
done
