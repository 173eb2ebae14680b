"""One ringN exploration on the partitioned dedup engine (for ncu):
python scripts/prof_dedup.py N WORLD [fused]"""
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200.bench import gen_token_ring  # noqa: E402
from paper_1801_05857_b200.distributed import LocalShardExplorer  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig, slots_per_bucket  # noqa: E402

n, world = int(sys.argv[1]), int(sys.argv[2])
dedup = len(sys.argv) < 4
net = gx.load_network(gen_token_ring(n, Path(tempfile.mkdtemp()) / "r")[1])
states = 2 * n * 3 ** (n - 1)
per = states // world + (states >> 8) + 4096
cap = (int(per / 0.5 / slots_per_bucket(32, 2, "half")) + 64) * 32
cfg = ExploreConfig(table=TableConfig(capacity_words=cap, num_hash_functions=16), detect_deadlocks=True,
                    dedup=dedup, state_digest=False)
ex = LocalShardExplorer(net, cfg, world)
r = ex.run()
print(r.states, r.transitions, r.probes, r.level_ms)
ex.close()
