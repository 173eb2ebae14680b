"""Generate the golden vectors that pin the oracle (and through it the B200
engine) to the real reference.

Run in the build container, where the read-only reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything is produced by calling the reference package `ltsmc` itself
(hashtable.py, network.py, statevec.py, explore.py, oracle.py, bench.py);
nothing here re-implements its algorithms.  Outputs (committed):

  tests/golden/hash_kats.json     hash constants / fold / probe sequences /
                                  slots_per_bucket (hashtable.py:89-217)
  tests/golden/table_runs.npz     serial find_or_insert codes + handles,
                                  claim/scan/occupancy (hashtable.py:224-331)
  tests/golden/models/<name>/     model files (generated + random networks)
  tests/golden/models.json        per model: explore reports for several
                                  table configs (explore.py:300-395),
                                  sha256 of --dump-states / --dump-table,
                                  sequential_bfs counts (oracle.py:32-88)
  tests/golden/expand_kats.json   expand() successor lists + counts for
                                  every reachable state of small models
                                  (network.py:184-238)
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import tempfile
import warnings
from pathlib import Path

import numpy as np

from ltsmc import statevec
from ltsmc.aut import parse_aut, parse_network
from ltsmc.bench import gen_gas_station, gen_token_ring
from ltsmc.explore import ExploreConfig, explore
from ltsmc.hashtable import (HALF_BUCKET, PLAIN, StateTable, TableConfig, hash_constants,
                             slots_per_bucket)
from ltsmc.network import build_network, expand, load_network
from ltsmc.oracle import sequential_bfs

OUT = Path(__file__).resolve().parent
MODELS = OUT / "models"
REF_FIG = Path("/root/reference/pkg/models/producer_consumer")


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


# ---------------------------------------------------------------- hashing

def hash_kats():
    out = {"constants": {}, "fold": [], "probe": [], "spb": []}
    for seed in (0, 1, 42, 123, 2**64 - 1, 0xDEADBEEFCAFEF00D):
        consts = hash_constants(seed, 8)
        t = StateTable(TableConfig(bucket_words=4, capacity_words=4 * 8, seed=seed), 1)
        out["constants"][str(seed)] = {"pairs": [list(c) for c in consts], "salt": t._fold_salt}
    rng = random.Random(7)
    for seed in (42, 123):
        for vlen in (1, 2, 3, 4, 7, 16):
            for _ in range(6):
                p = tuple(rng.getrandbits(32) for _ in range(vlen))
                t = StateTable(TableConfig(bucket_words=32, capacity_words=32 * 8, seed=seed), vlen)
                out["fold"].append({"seed": seed, "p": list(p), "h": t.fold(p)})
    for seed, bw, vlen, nb in ((42, 32, 1, 1000), (42, 16, 3, 77), (42, 4, 1, 8),
                               (7, 8, 2, (1 << 33) + 17), (42, 32, 2, (1 << 36) - 5),
                               (99, 4, 1, 3 * (1 << 31) + 1)):
        # the table for the large bucket counts is never allocated: use a
        # small one and override num_buckets (bucket_index reads only it)
        t = StateTable(TableConfig(bucket_words=bw, capacity_words=bw * 16, seed=seed), vlen)
        t.num_buckets = nb
        for _ in range(8):
            p = tuple(rng.getrandbits(32) for _ in range(vlen))
            out["probe"].append({"seed": seed, "bw": bw, "vlen": vlen, "nb": nb, "p": list(p),
                                 "seq": t.probe_sequence(p)})
        for p in ((0,) * vlen, (7,) * vlen):
            out["probe"].append({"seed": seed, "bw": bw, "vlen": vlen, "nb": nb, "p": list(p),
                                 "seq": t.probe_sequence(p)})
    for bw in (4, 8, 16, 32):
        for vlen in range(1, 18):
            for layout in (HALF_BUCKET, PLAIN):
                try:
                    n = slots_per_bucket(bw, vlen, layout)
                except ValueError as err:
                    n = str(err)
                out["spb"].append({"bw": bw, "vlen": vlen, "layout": layout, "spb": n})
    (OUT / "hash_kats.json").write_text(json.dumps(out, indent=1))


# ----------------------------------------------------------- table runs

def table_runs():
    arrays = {}
    meta = []
    rng = np.random.default_rng(2024)
    idx = 0
    for bw in (4, 8, 16, 32):
        for vlen in (1, 2, 3, 4):
            for layout in (None, PLAIN, HALF_BUCKET):
                if layout == HALF_BUCKET and bw != 32:
                    continue
                try:
                    spb = slots_per_bucket(bw, vlen,
                                           TableConfig(bucket_words=bw, layout=layout).resolved_layout())
                except ValueError:
                    continue
                for load in (0.5, 1.3):  # second one runs into TABLE_FULL
                    nb = 64
                    cfg = TableConfig(bucket_words=bw, capacity_words=nb * bw, layout=layout,
                                      seed=42 + idx, num_hash_functions=4 if load > 1 else 8)
                    t = StateTable(cfg, vlen)
                    n_unique = max(1, int(load * nb * spb))
                    uniq = rng.integers(0, 1 << 32, size=(n_unique, vlen), dtype=np.uint64)
                    uniq[0] = 0  # the all-zero vector is valid
                    seq = uniq[rng.integers(0, n_unique, size=2 * n_unique)]
                    seq = np.concatenate([uniq, seq])[rng.permutation(3 * n_unique)]
                    codes, handles = [], []
                    for row in seq:
                        c, h = t.find_or_insert(tuple(int(x) for x in row))
                        codes.append(c)
                        handles.append(h)
                    # claim every third successful handle, then scan
                    claimed = []
                    for h in handles[::3]:
                        if h >= 0:
                            claimed.append(int(t.claim_new(h)))
                    scan = t.scan_new(0, t.num_buckets)
                    scan_half = t.scan_new(t.num_buckets // 3, t.num_buckets // 2)
                    occ = t.occupancy()
                    rows = [(b, j, st, list(w)) for b, j, st, w in t.dump_rows()]
                    key = f"r{idx}"
                    arrays[key + "_seq"] = seq.astype(np.uint32)
                    arrays[key + "_codes"] = np.array(codes, np.uint8)
                    arrays[key + "_handles"] = np.array(handles, np.int64)
                    arrays[key + "_claimed"] = np.array(claimed, np.uint8)
                    arrays[key + "_scan"] = np.array(scan, np.int64)
                    arrays[key + "_scan_half"] = np.array(scan_half, np.int64)
                    meta.append({"key": key, "bw": bw, "vlen": vlen, "layout": layout,
                                 "capacity_words": cfg.capacity_words, "seed": cfg.seed,
                                 "k": cfg.num_hash_functions, "spb": t.slots_per_bucket,
                                 "num_buckets": t.num_buckets, "occupancy": list(occ[:2]),
                                 "dump_rows_sha": sha(json.dumps(rows))})
                    idx += 1
    np.savez_compressed(OUT / "table_runs.npz", **arrays)
    (OUT / "table_runs.json").write_text(json.dumps(meta, indent=1))


# ---------------------------------------------------------------- models

def random_network(seed: int, out: Path):
    """Random networks exercising the corner cases of build_network /
    expand: self-loops, duplicate lines, '_' columns, disabled rules,
    several rules with one result, single-participant rules, internal
    steps ("i" and its alias "tau"), deadlocks."""
    rng = random.Random(seed)
    P = rng.randint(1, 5)
    alphabet = ["a", "b", "c", "i", "tau", "d"]
    out.mkdir(parents=True, exist_ok=True)
    files = []
    for p in range(P):
        ns = rng.randint(2, 6)
        lines = []
        for _ in range(rng.randint(ns, 3 * ns)):
            src = rng.randrange(ns)
            dst = src if rng.random() < 0.2 else rng.randrange(ns)
            lines.append(f'({src}, "{rng.choice(alphabet)}", {dst})')
        if rng.random() < 0.3:
            lines.append(lines[0])  # duplicate line
        text = f"des ({rng.randrange(ns)}, {len(lines)}, {ns})\n" + "\n".join(lines) + "\n"
        (out / f"p{p}.aut").write_text(text)
        files.append(f'"p{p}.aut"')
    rules = []
    for _ in range(rng.randint(0, 6)):
        cols = [rng.choice(["_", "_", "a", "b", "c", "e"]) for _ in range(P)]
        if all(c == "_" for c in cols):
            cols[rng.randrange(P)] = rng.choice(["a", "b"])
        rules.append(" * ".join(cols) + " -> " + rng.choice(["a", "sync", "x", "b"]))
    exp = "par using\n    " + ",\n    ".join(rules) + "\nin\n    " + " || ".join(files) + "\nend par\n"
    (out / "net.exp").write_text(exp)
    return out / "net.exp"


def sinks_network(n: int, out: Path):
    """n processes that each step once into one of two sinks, gated by a
    shared `go` rule with a starter: 2^n deadlock states (> 100 at n = 8)."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "s.aut").write_text('des (0, 3, 4)\n(0,"go",1)\n(1,"a",2)\n(1,"b",3)\n')
    (out / "g.aut").write_text('des (0, 1, 2)\n(0,"go",1)\n')
    (out / "net.exp").write_text("par using\n  " + " * ".join(["go"] * (n + 1)) + " -> go\nin\n  "
                                 + " || ".join(['"g.aut"'] + ['"s.aut"'] * n) + "\nend par\n")
    return out / "net.exp"


def collide_network(out: Path):
    """Two rules with one result over identical participants and
    self-loops: exercises per-source (result, target) dedup (network.py:226-230)."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "a.aut").write_text('des (0, 4, 2)\n(0, "s", 0)\n(0, "s", 1)\n(0, "t", 0)\n(1, "t", 1)\n')
    (out / "b.aut").write_text('des (0, 3, 2)\n(0, "s", 1)\n(0, "t", 1)\n(1, "u", 0)\n')
    (out / "net.exp").write_text(
        "par using\n  s * s -> go,\n  t * t -> go,\n  s * _ -> go,\n  t * _ -> stay\n"
        'in\n  "a.aut" || "b.aut"\nend par\n')
    return out / "net.exp"


def sink_network(out: Path):
    out.mkdir(parents=True, exist_ok=True)
    (out / "x.aut").write_text('des (0,2,3)\n(0,"a",1)\n(0,"b",2)\n')
    (out / "net.exp").write_text('par using in "x.aut" end par\n')
    return out / "net.exp"


def philosophers_network(n: int, out: Path):
    """Dining philosophers (left fork first): deadlocks when every
    philosopher holds its left fork."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "phil.aut").write_text(
        'des (0, 4, 4)\n(0, "takeL", 1)\n(1, "takeR", 2)\n(2, "putL", 3)\n(3, "putR", 0)\n')
    (out / "fork.aut").write_text('des (0, 2, 2)\n(0, "take", 1)\n(1, "put", 0)\n')
    total = 2 * n
    rules = []
    for i in range(n):
        left, right = n + i, n + (i + 1) % n
        for act, fork_idx, fact in (("takeL", left, "take"), ("takeR", right, "take"),
                                    ("putL", left, "put"), ("putR", right, "put")):
            cols = ["_"] * total
            cols[i] = act
            cols[fork_idx] = fact
            rules.append(" * ".join(cols) + f" -> {act}{i}")
    files = ['"phil.aut"'] * n + ['"fork.aut"'] * n
    (out / "net.exp").write_text("par using\n  " + ",\n  ".join(rules) + "\nin\n  "
                                 + " || ".join(files) + "\nend par\n")
    return out / "net.exp"


def wide_network(n: int, out: Path):
    """n two-state processes toggled by one n-ary rule (test_explore.py:116-128):
    vlen 2 at n=33, a full 32-bit first word (no spare bits)."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "p.aut").write_text('des (0,2,2)\n(0,"t",1)\n(1,"t",0)\n')
    (out / "net.exp").write_text("par using " + " * ".join(["t"] * n) + " -> sync in "
                                 + " || ".join(['"p.aut"'] * n) + " end par\n")
    return out / "net.exp"


def sparse_network(k: int, out: Path):
    """k processes declaring 2^20 states each (20-bit fields, one per word:
    vlen k) with a tiny reachable set: one k-ary rule cycles every process
    0 -> 1 -> 2 -> 0 in lockstep; for k <= 8 each process may also step
    1 -u-> 7 on its own (2^k interleavings) and return with the rule."""
    out.mkdir(parents=True, exist_ok=True)
    extra = '(1,"u",7)\n(7,"t",0)\n' if k <= 8 else ""
    ntr = 5 if k <= 8 else 3
    (out / "s.aut").write_text(f'des (0, {ntr}, 1048576)\n(0,"t",1)\n(1,"t",2)\n(2,"t",0)\n' + extra)
    (out / "net.exp").write_text("par using\n  " + " * ".join(["t"] * k) + " -> t\nin\n  "
                                 + " || ".join(['"s.aut"'] * k) + "\nend par\n")
    return out / "net.exp"


def counter_network(n: int, out: Path):
    """n independent 3-state counters (0->1->2->0): 3^n states, all
    interleavings; a 32-process instance fills two words completely."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "c.aut").write_text('des (0,3,3)\n(0,"inc",1)\n(1,"inc",2)\n(2,"inc",0)\n')
    (out / "net.exp").write_text("par using in " + " || ".join(['"c.aut"'] * n) + " end par\n")
    return out / "net.exp"


def report_tuple(rep):
    return {"states": rep.states, "transitions": rep.transitions,
            "deadlocks": [list(s) for s in rep.deadlocks], "deadlocks_total": rep.deadlocks_total,
            "expanded": rep.expanded, "iterations": rep.iterations, "outcome": rep.outcome}


def model_entries():
    models = {}
    if MODELS.exists():
        import shutil
        shutil.rmtree(MODELS)
    MODELS.mkdir(parents=True)
    paths = {}
    import shutil
    shutil.copytree(REF_FIG, MODELS / "fig1")
    paths["fig1"] = MODELS / "fig1" / "net.exp"
    for n in range(2, 11):
        gen_token_ring(n, MODELS / f"ring{n}")
        paths[f"ring{n}"] = MODELS / f"ring{n}" / "net.exp"
    for n in range(2, 9):
        gen_gas_station(n, MODELS / f"gas{n}")
        paths[f"gas{n}"] = MODELS / f"gas{n}" / "net.exp"
    paths["sink"] = sink_network(MODELS / "sink")
    paths["collide"] = collide_network(MODELS / "collide")
    for n in (2, 3, 4, 5):
        paths[f"phil{n}"] = philosophers_network(n, MODELS / f"phil{n}")
    paths["wide33"] = wide_network(33, MODELS / "wide33")
    paths["wide32"] = wide_network(32, MODELS / "wide32")
    paths["counter8"] = counter_network(8, MODELS / "counter8")
    for n in (3, 8, 10):
        paths[f"sinks{n}"] = sinks_network(n, MODELS / f"sinks{n}")
    for k in (2, 3, 4, 5, 8, 16):
        paths[f"sparse{k}"] = sparse_network(k, MODELS / f"sparse{k}")
    for s in range(60):
        paths[f"rand{s}"] = random_network(1000 + s, MODELS / f"rand{s}")
    return paths


def main():
    warnings.simplefilter("ignore")
    hash_kats()
    print("hash kats done", flush=True)
    table_runs()
    print("table runs done", flush=True)
    paths = model_entries()
    models = {}
    kats = {}
    tmp = Path(tempfile.mkdtemp())
    for name, path in paths.items():
        try:
            net = load_network(path)
        except Exception as err:  # noqa: BLE001 - recorded as a golden error
            models[name] = {"path": str(path.relative_to(OUT)), "error": f"{type(err).__name__}: {err}"}
            continue
        scheme = statevec.make_scheme(net)
        big = name in ("ring9", "ring10")
        entry = {"path": str(path.relative_to(OUT)), "vlen": scheme.vector_length,
                 "nproc": len(net.processes), "runs": []}
        orc = sequential_bfs(net, keep_states=not big)
        entry["bfs"] = {"states": orc.states, "transitions": orc.transitions,
                        "deadlocks": [list(s) for s in orc.deadlocks[:100]],
                        "deadlocks_total": len(orc.deadlocks)}
        if not big:
            packed = [statevec.pack(scheme, s) for s in orc.state_set]
            entry["bfs"]["dump_sha"] = sha(statevec.dump_states(packed))
        cfgs = [dict(bucket_words=32, capacity_words=1 << 16), dict(bucket_words=4, capacity_words=1 << 16)]
        if big:
            cfgs = [dict(bucket_words=32, capacity_words=1 << 22)]
        if name in ("ring6", "ring5", "gas4", "phil4", "sinks10"):
            cfgs.append(dict(bucket_words=4, capacity_words=4 * 64))          # TABLE_FULL
            cfgs.append(dict(bucket_words=8, capacity_words=1 << 14, max_iterations=3))  # cap
        for c in cfgs:
            max_it = c.pop("max_iterations", None)
            if big:
                continue  # explore at ring9/10 is minutes in Python; bfs counts pin them
            cfg = ExploreConfig(workers=1, table=TableConfig(**c), detect_deadlocks=True,
                                max_iterations=max_it)
            ds, dt = tmp / "s.txt", tmp / "t.csv"
            try:
                rep = explore(net, cfg, dump_states=ds, dump_table=dt)
            except ValueError as err:
                entry["runs"].append({"table": c, "max_iterations": max_it, "error": str(err)})
                continue
            run = {"table": c, "max_iterations": max_it, "report": report_tuple(rep),
                   "dump_states_sha": sha(ds.read_text()), "dump_table_sha": sha(dt.read_text())}
            entry["runs"].append(run)
        models[name] = entry
        print(name, entry["bfs"]["states"], flush=True)
        # expand KATs on every reachable state of the small models
        if not big and orc.states <= 3000:
            rows = []
            for s in orc.state_set:
                succ, count = expand(net, s)
                rows.append([list(s), count, [[net.actions[a], list(t)] for a, t in succ]])
            kats[name] = rows
    (OUT / "models.json").write_text(json.dumps(models, indent=1))
    (OUT / "expand_kats.json").write_text(json.dumps(kats))


if __name__ == "__main__":
    sys.exit(main())
