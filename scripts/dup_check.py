"""Developer check: a few cells of the Fig. 4 duplication sweep (bench.py
duplication_sweep protocol).  python scripts/dup_check.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1801_05857_b200.bench import DuplicationSpec, device_insert_bench, insert_bench_table_config  # noqa
from paper_1801_05857_b200.hashtable import StateTable  # noqa: E402

total = 1 << 30
for vlen in (1, 2):
    for bw in (4, 32):
        for d in (1, 10, 100):
            spec = DuplicationSpec(total=total, duplication=d, vector_length=vlen)
            t = StateTable(insert_bench_table_config(spec, bw), vlen, mark=(vlen - 1, 31))
            r = device_insert_bench(t, total, d, seed=11)
            t.close()
            print(json.dumps({"vlen": vlen, "bw": bw, "d": d, "ops_per_sec": r["ops_per_sec"], "full": r["full"],
                              "buckets_per_op": r["buckets_per_op"]}), flush=True)
