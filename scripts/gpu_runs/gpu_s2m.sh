# round 2: multi-shard / multi-process GPU tests (dedup mode, sharded hash bench, CUDA IPC, NCCL driver)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -25 > gpurun_out/s2m_tests.log
cat gpurun_out/s2m_tests.log
