"""R(g) vs buffer size (TLB reach check): python scripts/ra_sweep.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1801_05857_b200.bench import random_access_roofline  # noqa: E402

for gb in (8, 32, 64, 96, 128, 160):
    for g in (32, 128):
        r = random_access_roofline(g, buffer_bytes=gb << 30, reads=1 << 28)
        print(json.dumps({"buffer_gib": gb, "g": g, "gbs": round(r["gbs"], 1),
                          "accesses_per_s": r["segments_per_sec"]}), flush=True)
