# round 2: new GPU tests (digests, deadlock overflow, bench pins) + quick default bench with the digest check
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_digest.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 900 -x -k "digest or deadlock or pins or large" 2>&1 | tail -15 > gpurun_out/s2l_tests.log
timeout 1200 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench > gpurun_out/s2l_bench.json 2> gpurun_out/s2l_bench.err
cat gpurun_out/s2l_tests.log; tail -2 gpurun_out/s2l_bench.err
