set -x
mkdir -p gpurun_out
timeout 600 python scripts/ra_ballast.py > gpurun_out/r1p_ballast.log 2>&1
nvidia-smi -q | grep -i -A3 "bar1\|page\|mig" | head -40 > gpurun_out/r1p_smi.txt
