"""Developer check of the partitioned dedup engine on the GPU: golden
models (digest vs tests/golden/ref_digests.json) through
explore_local_shards at 1-3 shards, then ringN timings dedup vs fused.
python scripts/dedup_check.py [ringN ...]"""
import json
import sys
import tempfile
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200.bench import gen_token_ring  # noqa: E402
from paper_1801_05857_b200.distributed import LocalShardExplorer, explore_local_shards  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig, slots_per_bucket  # noqa: E402

G = ROOT / "tests" / "golden"
REF = json.loads((G / "ref_digests.json").read_text())
MODELS = json.loads((G / "models.json").read_text())
bad = 0
for world in (1, 2, 3):
    for name in sorted(REF):
        net = gx.load_network(G / MODELS[name]["path"])
        sc = gx.statevec.make_scheme(net)
        if gx.statevec.device_vlen(sc) not in (1, 2, 4) or gx.statevec.mark_bit(sc, gx.statevec.device_vlen(sc)) is None:
            continue
        cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 20), detect_deadlocks=True)
        rep = explore_local_shards(net, cfg, world)
        b = MODELS[name]["bfs"]
        ok = (list(rep.digest) == REF[name] and (rep.states, rep.transitions, rep.deadlocks_total) ==
              (b["states"], b["transitions"], b["deadlocks_total"]) and
              [list(x) for x in rep.deadlocks] == b["deadlocks"][:100])
        if not ok:
            bad += 1
            print("MISMATCH", world, name, rep.states, b["states"], rep.transitions, b["transitions"], flush=True)
print("golden models checked, mismatches:", bad, flush=True)

for arg in sys.argv[1:] or ["ring14", "ring16"]:
    n = int(arg[4:])
    tmp = Path(tempfile.mkdtemp())
    net = gx.load_network(gen_token_ring(n, tmp / arg)[1])
    states, trans = 2 * n * 3 ** (n - 1), 4 * n * n * 3 ** (n - 2)
    for world in (1, 2):
        for dedup in (False, True):
            per = states // world + (states >> 8) + 4096
            spb = slots_per_bucket(32, 2, "half")
            cap = (int(per / 0.5 / spb) + 64) * 32
            cfg = ExploreConfig(table=TableConfig(capacity_words=cap, num_hash_functions=16),
                                detect_deadlocks=True, dedup=dedup, state_digest=False)
            ex = LocalShardExplorer(net, cfg, world)
            ex.run()
            t0 = time.perf_counter()
            r = ex.run()
            dt = time.perf_counter() - t0
            d = ex.digest()
            ex.close()
            print(f"{arg} world={world} dedup={dedup}: {dt*1e3:.1f} ms  {r.states/dt:.3g} st/s  "
                  f"probes={r.probes} ({r.probes/trans:.3f}/transition) ok={(r.states, r.transitions) == (states, trans)} "
                  f"digest_count={d[0]} level_ms={r.level_ms:.1f}", flush=True)
