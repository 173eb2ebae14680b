set -x
mkdir -p gpurun_out
timeout 1500 python scripts/tlb_shards.py 19 0.75 1 3 > gpurun_out/r1r_tlb19.log 2>&1
