"""Stall samples and executed instructions per CUDA source line from
`ncu -i REP --page source --csv --print-source cuda,sass -k KERNEL` output
(python scripts/ncu_lines.py CSV [TOP]); the per-line view DESIGN.md and
profiles/README.md cite."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, header, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r and r[0] == "Line No":
        header = r
    elif header and r and r[0] not in ("", "Line No") and len(r) == len(header):
        d = dict(zip(header, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
            ni = int(d["Warp Stall Sampling (Not-issued Samples)"])
            inst = int(d["Instructions Executed"])
        except ValueError:
            continue
        out.append((s, ni, inst, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(o[0] for o in out) or 1
toti = sum(o[2] for o in out) or 1
print(f"total samples {tot}, instructions {toti}")
for s, ni, inst, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {100*inst/toti:5.1f}%i  {loc:22s} {src}")
