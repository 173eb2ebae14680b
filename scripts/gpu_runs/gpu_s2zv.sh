# round 2, final validation at the final tree (GX_OVERLAP, GX_PREFETCH, GX_DEFER_CAS all off): GPU suite, smoke, default bench line, reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -3 > gpurun_out/s2zv_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2zv_smoke.log 2>&1
timeout 2400 python bench.py > gpurun_out/s2zv_bench.json 2> gpurun_out/s2zv_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/s2zv_ref.json 2> gpurun_out/s2zv_ref.err
cat gpurun_out/s2zv_tests.log gpurun_out/s2zv_smoke.log
python -c "import json; d=json.loads(open('gpurun_out/s2zv_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic'], d['digest']['equal'], [(e['workload'], round(e['states_per_sec']/1e9,3)) for e in d['extra_workloads']])"
