"""DRAM traffic of the level kernels per exploration, from an ncu launch list
taken with --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
(python scripts/traffic.py LAUNCHES.csv KEY [OUT.json] [EXPLORATIONS]): sums
the bytes of every k_level* / k_absorb launch of the captured command,
divides by the number of explorations it ran (bench.py --steps 1 --warmup 0
--e2e-steps 0 runs two: the timed one and the e2e warm-up) and writes
profiles/traffic.json[KEY] = {"bytes_per_step": ..., "launches": ...}."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
head = next(r for r in csv.reader(open(sys.argv[1])) if r and r[0] == "ID")
i_name, i_metric, i_unit, i_val = (head.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit",
                                                            "Metric Value"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
tot = defaultdict(float)
launches = set()
for r in rows:
    if not any(k in r[i_name] for k in ("k_level", "k_absorb")):
        continue
    launches.add(r[0])
    tot[r[i_metric]] += float(r[i_val].replace(",", "")) * scale.get(r[i_unit], 1)
ne = int(sys.argv[4]) if len(sys.argv) > 4 else 1
out = {"bytes_per_step": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / ne,
       "read_bytes": tot["dram__bytes_read.sum"] / ne, "write_bytes": tot["dram__bytes_write.sum"] / ne,
       "kernel_seconds_serialised": tot["gpu__time_duration.sum"] / ne, "launches": len(launches) / ne,
       "source": Path(sys.argv[1]).name}
if ne > 1:
    out["note"] = f"the captured command ran {ne} explorations; every total is divided by {ne}"
path = Path(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else \
    Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
data = json.loads(path.read_text()) if path.exists() else {}
data[sys.argv[2]] = out
path.write_text(json.dumps(data, indent=1) + "\n")
print(json.dumps(out))
