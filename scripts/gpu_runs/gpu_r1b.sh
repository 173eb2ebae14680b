# round-1 re-entry GPU pass: tests, smoke, default bench, launch list, ncu capture of k_level
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1b_smi.txt 2>&1
nproc > gpurun_out/r1b_nproc.txt; lscpu | head -20 >> gpurun_out/r1b_nproc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -30 > gpurun_out/r1b_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1b_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r1b_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level -s 60 -c 1 -o gpurun_out/r1b_prof_ring16 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
