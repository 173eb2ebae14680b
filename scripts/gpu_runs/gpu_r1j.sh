set -x
mkdir -p gpurun_out
python scripts/memdiag.py 18 0.5 > gpurun_out/r1j_memdiag.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for v in default q768 q1024; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r1j_${v}_bw32.json 2>&1
  timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1j_${v}_bw8.json 2>&1
done
