set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -x -k "shard or cli or closed" 2>&1 | tail -3 > gpurun_out/r1u_tests.log
timeout 1500 python scripts/tlb_shards.py 19 0.75 0 3 4 > gpurun_out/r1u_tlb19_f0.log 2>&1
timeout 1500 python scripts/tlb_shards.py 19 0.75 23 3 > gpurun_out/r1u_tlb19_f23.log 2>&1
