"""Developer check: the fill sweep of bench.py for one (bw, K) -- timed
inserts of 2% of the slots and 2^28 lookups per fill level, buckets per op.
python scripts/fill_check.py BW K"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1801_05857_b200.bench import device_insert_bench  # noqa: E402
from paper_1801_05857_b200.hashtable import StateTable, TableConfig  # noqa: E402

bw, k = int(sys.argv[1]), int(sys.argv[2])
t = StateTable(TableConfig(bucket_words=bw, num_hash_functions=k, capacity_words=1 << 33), 2, mark=(1, 31))
slots = t.total_slots
rows = 0
for fill in (0.5, 0.7, 0.8, 0.9):
    target, batch = int(fill * slots), int(0.02 * slots)
    occ = t.occupancy()[0]
    if target - batch > occ:
        n = target - batch - occ
        device_insert_bench(t, n, 1, seed=7, row_base=rows)
        rows += n
    r = device_insert_bench(t, batch, 1, seed=7, row_base=rows)
    rows += batch
    look = device_insert_bench(t, 1 << 28, 1, seed=7, row_base=rows - (1 << 28))
    print(json.dumps({"bw": bw, "k": k, "fill": fill, "insert_ops_per_sec": r["ops_per_sec"],
                      "lookup_ops_per_sec": look["ops_per_sec"], "lookup_buckets_per_op": look["buckets_per_op"],
                      "full": r["full"]}), flush=True)
t.close()
