"""Where the e2e step's time goes beyond the level kernels (bench.py's
default ring19 line on one GPU: 2 hash-owner shards): shard construction
(CSR upload, table + buffer allocation and zeroing), the exploration, the
digest, and the release.  Sizes as bench.py's defaults.  One JSON line.

    python scripts/e2e_phases.py [--workload ring19] [--reps 2]
"""
import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench as B  # noqa: E402
import paper_1801_05857_b200 as gx  # noqa: E402
from paper_1801_05857_b200 import statevec  # noqa: E402
from paper_1801_05857_b200.distributed import LocalShardExplorer  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="ring19")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--load", type=float, default=0.8)
    a = ap.parse_args()
    tmp = Path(tempfile.mkdtemp())
    net = gx.load_network(B.model_path(a.workload, tmp))
    vlen = statevec.make_scheme(net).vector_length
    states = B.closed_form(a.workload)[0]
    est = B.table_capacity(states, vlen, 32, a.load) * 4
    shards = 1 if est <= B.TLB_REACH else -(-est // B.SHARD_BYTES)
    per = states // shards + (states >> 8 if shards > 1 else 0)
    cap = B.table_capacity(per, vlen, 32, a.load)
    cfg = ExploreConfig(table=TableConfig(bucket_words=32, num_hash_functions=32, capacity_words=cap),
                        detect_deadlocks=True, state_digest=False)
    front = int(states * 0.035 / shards) + (1 << 20)
    left = torch.cuda.mem_get_info()[0] - cap * 4 * shards - front * 4 * vlen * shards
    inbox = max(1 << 20, min(int(states * 0.3 / shards) + (1 << 20), int(0.85 * left) // (4 * vlen * shards)))
    rows = []

    def sync_t():
        torch.cuda.synchronize()
        return time.perf_counter()

    for i in range(a.reps + 1):
        t0 = sync_t()
        ex = LocalShardExplorer(net, cfg, shards, inbox_capacity=inbox, frontier_capacity=front, status=False)
        t1 = sync_t()
        rep = ex.run()
        t2 = sync_t()
        ex.digest()
        t3 = sync_t()
        ex.close()
        t4 = sync_t()
        rows.append({"construct_s": t1 - t0, "run_s": t2 - t1, "level_s": rep.level_ms / 1e3,
                     "digest_s": t3 - t2, "close_s": t4 - t3, "total_s": t4 - t0, "warm": i > 0})
    print(json.dumps({"workload": a.workload, "shards": shards, "table_words_per_shard": cap,
                      "inbox_vectors": inbox, "frontier_vectors": front, "phases": rows}))


if __name__ == "__main__":
    main()
