"""Pin the reachable-set digest (include/gx.h gx_table_digest) to the real
reference: for every golden model, the reference's own sequential oracle
(ltsmc.oracle.sequential_bfs, oracle.py:32-88) enumerates the state set,
the reference's packer (statevec.pack) packs it, and the digest of those
packed vectors is written to tests/golden/ref_digests.json.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reference_digests.py

The digest function itself is the product's `statevec.state_digest`
(restated independently in oracle/gx_oracle.c `or_state_hash`); the state
sets are the reference's.
"""

from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

from ltsmc import statevec as ref_statevec
from ltsmc.network import load_network
from ltsmc.oracle import sequential_bfs

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent.parent))
from paper_1801_05857_b200.statevec import state_digest  # noqa: E402


def main():
    warnings.simplefilter("ignore")
    models = json.loads((OUT / "models.json").read_text())
    out = {}
    for name, entry in models.items():
        if "error" in entry:
            continue
        net = load_network(OUT / entry["path"])
        scheme = ref_statevec.make_scheme(net)
        orc = sequential_bfs(net, keep_states=True)
        packed = np.array([ref_statevec.pack(scheme, s) for s in orc.state_set], np.uint32)
        packed = packed.reshape(len(orc.state_set), scheme.vector_length)
        out[name] = list(state_digest(packed))
        print(name, out[name][0], flush=True)
    (OUT / "ref_digests.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
