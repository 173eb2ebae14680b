set -x
mkdir -p gpurun_out
timeout 900 python scripts/tlb_shards.py 18 0.3 1 2 3 > gpurun_out/r1o_tlb18.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hash-bench --e2e-steps 0"
for v in default m4q768 m3kb64q768; do
  if [ $v = default ]; then unset GX_LIB; else export GX_LIB=$PWD/build_variants/$v.so; fi
  timeout 300 $B > gpurun_out/r1o_${v}_bw32.json 2>&1
  timeout 300 $B --bucket-words 8 --hash-functions 32 --load 0.4 > gpurun_out/r1o_${v}_bw8.json 2>&1
done
