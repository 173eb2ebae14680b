"""Single-GPU TLB-reach experiment: one big table vs W local hash shards
(each below the TLB cliff), same model.  python scripts/tlb_shards.py N LOAD W..."""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200 import distributed as D  # noqa: E402
from paper_1801_05857_b200.bench import gen_token_ring  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig, Explorer  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402

n, load = int(sys.argv[1]), float(sys.argv[2])
flt = int(sys.argv[3])
worlds = [int(x) for x in sys.argv[4:]] or [1, 2, 3]
_, p = gen_token_ring(n, Path(tempfile.mkdtemp()) / "ring")
net = gx.load_network(p)
states = 2 * n * 3 ** (n - 1)
for w in worlds:
    per = states // w + (states >> 8)
    cap = (int(per / load / 16) + 4096) * 32
    cfg = ExploreConfig(table=TableConfig(capacity_words=cap, num_hash_functions=32), detect_deadlocks=True,
                        filter_log2=flt)
    t0 = time.perf_counter()
    if w == 1:
        ex = Explorer(net, cfg, status=False)
        ex.run()
        t1 = time.perf_counter()
        rep = ex.run()
        dt = time.perf_counter() - t1
        ex.close()
    else:
        front = int(states * 0.035 / w) + (1 << 20)
        inbox = int(states * 0.12 / w) + (1 << 20)
        t1 = time.perf_counter()
        rep = D.explore_local_shards(net, cfg, w, inbox_capacity=inbox, frontier_capacity=front,
                                     status=False)
        dt = time.perf_counter() - t1
    assert rep.states == states, (rep.states, states)
    print(json.dumps({"ring": n, "load": load, "filter_log2": flt, "shards": w, "table_gb_total": cap * 4 * w / 1e9,
                      "seconds": dt, "states_per_s": states / dt}), flush=True)
