# round 2: first GPU run of the partitioned dedup engine (correctness + ring14/16 timing)
mkdir -p gpurun_out
timeout 900 python scripts/dedup_check.py ring14 ring16 > gpurun_out/s2d_dedup.txt 2>&1
tail -30 gpurun_out/s2d_dedup.txt
