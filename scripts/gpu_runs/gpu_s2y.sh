# round 2: pipelined fused levels (absorb of chunk c-1 inside chunk c's launch): parity + ring19/ring18 timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider --timeout 900 -k pipelined 2>&1 | tail -3 > gpurun_out/s2y_tests.log
cat gpurun_out/s2y_tests.log
Q="--steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-hash-bench --no-extra --crosscheck 0"
timeout 900 python bench.py $Q --pipeline 1 > gpurun_out/s2y_ring19_pipe.json 2>&1
timeout 900 python bench.py $Q --pipeline 1 --shards 3 > gpurun_out/s2y_ring19_pipe_s3.json 2>&1
timeout 900 python bench.py $Q --pipeline 1 --workload ring18 --shards 2 > gpurun_out/s2y_ring18_pipe.json 2>&1
for f in gpurun_out/s2y_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4g'%d['value'], round(d['step_breakdown_ms']['level_kernels'],1), d['gpu_launches'], d['digest']['equal'])" || tail -3 $f; done
