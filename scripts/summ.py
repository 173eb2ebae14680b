"""Summarise bench JSON lines in gpurun_out (dev helper)."""
import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d.get("roofline", {})
        print(f"{f:45s} {d['value']/1e6:9.1f} Mst/s  frac={r.get('frac', 0):.3f}  kernel_ms={r.get('kernel_ms_per_step', 0):8.1f}")
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", open(f).read().strip().splitlines()[-1][:150])
