"""One peterson6 exploration on one table (for ncu): python scripts/prof_peterson.py"""
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200.bench import gen_peterson  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig, Explorer  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402

net = gx.load_network(gen_peterson(6, Path(tempfile.mkdtemp()) / "p6")[1])
ex = Explorer(net, ExploreConfig(table=TableConfig(capacity_words=1 << 31, num_hash_functions=16),
                                 state_digest=False))
r = ex.run()
print(r.states, r.transitions, r.level_ms, r.probes)
ex.close()
