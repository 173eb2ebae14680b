"""Golden reachable-set results for models too large for the Python
reference, generated with the C oracle (oracle/gx_oracle.c, itself pinned
to the reference by tests/golden/ref_digests.json and models.json):

    python tests/golden/make_digests.py            # writes tests/golden/digests.json

Per model: states, transitions, iterations (= BFS levels + 1), deadlocks
(total and the 100 smallest) and the set digest (include/gx.h
gx_table_digest) from a full oracle exploration (explore.py:300-395
restated, all host threads).  Token rings N = 11..20 additionally get the
digest of their reachable set enumerated in closed form
(gx_oracle.c or_ring_digest), with states 2 N 3^(N-1) and transitions
4 N^2 3^(N-2); for N <= 14 both routes are recorded and must agree.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_1801_05857_b200.bench import (gen_gas_station, gen_peterson,  # noqa: E402
                                         gen_philosophers, gen_token_ring)

GENS = {"ring": gen_token_ring, "gas": gen_gas_station, "peterson": gen_peterson,
        "phil": gen_philosophers}
EXPLORED = ["ring11", "ring12", "ring13", "ring14", "gas9", "gas10", "gas11", "peterson2", "peterson3",
            "peterson4", "peterson5", "peterson6", "phil8", "phil12", "phil14"]


def explore_entry(name: str, tmp: Path) -> dict:
    kind = name.rstrip("0123456789")
    n = int(name[len(kind):])
    path = GENS[kind](n, tmp / name)[1]
    net = O.Net.from_file(path)
    t0 = time.time()
    # size the table from a first BFS count (the oracle's sequential_bfs)
    states = net.bfs()["states"]
    slots_per_bucket = O.slots_per_bucket(32, net.vlen, O.HALF)
    cap = (int(states / 0.5 / slots_per_bucket) + 64) * 32
    r = O.explore(net, capacity_words=cap, workers=os.cpu_count() or 1, detect_deadlocks=True,
                  num_hash_functions=16)
    assert r.outcome == "COMPLETE", (name, r.outcome)
    d = r.table.digest()
    ent = {"states": r.states, "transitions": r.transitions, "iterations": r.iterations,
           "deadlocks_total": r.deadlocks_total, "deadlocks": [list(s) for s in r.deadlocks],
           "digest": list(d), "vlen": net.vlen, "source": "oracle explore"}
    print(name, r.states, r.transitions, f"{time.time() - t0:.1f}s", flush=True)
    return ent


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        tmp = Path(td)
        for name in EXPLORED:
            out[name] = explore_entry(name, tmp)
    for n in range(11, 21):
        d = O.ring_digest(n)
        name = f"ring{n}"
        states, trans = 2 * n * 3 ** (n - 1), 4 * n * n * 3 ** (n - 2)
        assert d[0] == states
        ent = out.setdefault(name, {"states": states, "transitions": trans, "deadlocks_total": 0,
                                    "deadlocks": [], "vlen": 1 if n <= 10 else 2,
                                    "source": "closed form"})
        if "digest" in ent:
            assert ent["digest"] == list(d) and ent["transitions"] == trans, name
        ent["digest"] = list(d)
        ent["digest_closed_form"] = True
        print(name, d, flush=True)
    (HERE / "digests.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
