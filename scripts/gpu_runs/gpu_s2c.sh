# round 2: L2 atomic / load throughput microbenchmark (dedup-set design study)
mkdir -p gpurun_out
timeout 300 ./scripts/micro/l2_atomics > gpurun_out/s2c_l2_atomics.txt 2>&1
cat gpurun_out/s2c_l2_atomics.txt
