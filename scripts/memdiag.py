import sys, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1801_05857_b200 as gx
from paper_1801_05857_b200 import distributed as D, statevec
from paper_1801_05857_b200.bench import gen_token_ring
from paper_1801_05857_b200.explore import ExploreConfig, Explorer
from paper_1801_05857_b200.hashtable import TableConfig
import bench as B
n = int(sys.argv[1])
_, p = gen_token_ring(n, Path(tempfile.mkdtemp()) / "ring")
net = gx.load_network(p)
print("free before", D.device_info())
cap = B.table_capacity(2 * n * 3 ** (n - 1), 2, 32, float(sys.argv[2]))
print("cap words", cap, "data GB", cap * 4 / 1e9)
ex = Explorer(net, ExploreConfig(table=TableConfig(capacity_words=cap, num_hash_functions=32)))
print("free after table", D.device_info(), "slots", ex.table.total_slots)
