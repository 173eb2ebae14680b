set -x
mkdir -p gpurun_out
timeout 600 python scripts/ra_sweep.py > gpurun_out/r1n_ra_sweep.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for v in default m3kb32 m3q512; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r1n_${v}_bw32.json 2>&1
  timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1n_${v}_bw8.json 2>&1
done
unset GX_LIB
timeout 300 $B > gpurun_out/r1n_default2_bw32.json 2>&1
