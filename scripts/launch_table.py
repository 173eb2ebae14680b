"""Per-kernel totals of an ncu --csv launch list (python scripts/launch_table.py CSV)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
rows = rows[1:]
iN, iM, iV, iU = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
sc = {"ns": 1e-6, "us": 1e-3, "ms": 1, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1, "inst": 1}
agg = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(set)
for r in rows:
    k = r[iN].split("(")[0].replace("void ", "")
    agg[k][r[iM]] += float(r[iV].replace(",", "")) * sc.get(r[iU], 1)
    cnt[k].add(r[0])
tot = sum(v["gpu__time_duration.sum"] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    print(f"{k[:40]:40s} n={len(cnt[k]):5d} ms={v['gpu__time_duration.sum']:8.2f} ({100*v['gpu__time_duration.sum']/tot:4.1f}%) "
          f"rdGB={v.get('dram__bytes_read.sum', 0):6.2f} wrGB={v.get('dram__bytes_write.sum', 0):6.2f} "
          f"Minst={v.get('smsp__inst_executed.sum', 0)/1e6:8.1f}")
