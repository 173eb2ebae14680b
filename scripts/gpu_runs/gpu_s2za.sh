# round 2: refill probe in the isolated bench with 512-key batches (fill and duplication cells)
mkdir -p gpurun_out
timeout 600 python scripts/fill_check.py 32 32 > gpurun_out/s2za_fill32.txt 2>&1
timeout 600 python scripts/fill_check.py 8 32 > gpurun_out/s2za_fill8.txt 2>&1
timeout 900 python scripts/dup_check.py > gpurun_out/s2za_dup.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pins or bench" 2>&1 | tail -2
for f in gpurun_out/s2za_*.txt; do echo $f; cat $f | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print({k:(round(v,3) if isinstance(v,float) and v<100 else ('%.3g'%v if isinstance(v,float) else v)) for k,v in d.items()})"; done
