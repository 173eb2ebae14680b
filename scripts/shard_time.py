"""Time the fused sharded engine with W shards on one GPU (dev helper)."""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200 import distributed as D  # noqa: E402
from paper_1801_05857_b200.bench import gen_token_ring  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
worlds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4]
_, p = gen_token_ring(n, Path(tempfile.mkdtemp()) / "ring")
net = gx.load_network(p)
states = 2 * n * 3 ** (n - 1)
for w in worlds:
    cap = (int(states / w / 0.5 / 16) + 4096) * 32
    cfg = ExploreConfig(table=TableConfig(capacity_words=cap), detect_deadlocks=True)
    D.explore_local_shards(net, cfg, w)
    t0 = time.perf_counter()
    rep = D.explore_local_shards(net, cfg, w)
    dt = time.perf_counter() - t0
    assert rep.states == states, (rep.states, states)
    print(json.dumps({"ring": n, "shards": w, "states": rep.states, "wall_s": dt,
                      "states_per_s": rep.states / dt, "iterations": rep.iterations}))
