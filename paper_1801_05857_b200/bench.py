"""Benchmark harness and model generators.

Mirrors /root/reference/pkg/src/ltsmc/bench.py: the duplication-sequence
insertion benchmark (`DuplicationSpec` :35, `gen_duplication_sequence`
:90, `insert_bench_table_config` :99, `run_insert_bench` :120,
`duplication_grid` :210), the bucket-size sweep (`bucket_size_sweep`
:380) and the scalable model generators (`gen_token_ring` :245,
`gen_gas_station` :291).  New here: generator caps raised for the
B200-scale configurations (token ring up to N=20, gas station up to 16),
the Peterson mutual-exclusion family (`gen_peterson`), and the fully
on-device insertion benchmark (`device_insert_bench`).
"""

from __future__ import annotations

import csv
import ctypes as C
import statistics
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from ._lib import check, lib
from .explore import ExploreConfig, explore
from .hashtable import DEFAULT_SEED, TABLE_FULL, StateTable, TableConfig, slots_per_bucket
from .network import Network, load_network

DUPLICATION_GRID = (1,) + tuple(range(10, 101, 10))


@dataclass(frozen=True)
class DuplicationSpec:
    total: int = 1_000_000
    duplication: int = 1
    vector_length: int = 1
    seed: int = DEFAULT_SEED

    def __post_init__(self):
        if min(self.total, self.duplication, self.vector_length) < 1:
            raise ValueError("total, duplication and vector_length must be >= 1")
        if self.duplication > self.total:
            raise ValueError("duplication exceeds sequence length")

    @property
    def unique_count(self) -> int:
        return self.total // self.duplication


@dataclass(frozen=True)
class BenchRecord:
    total: int
    duplication: int
    vector_length: int
    seed: int
    bucket_words: int
    threads: int
    wall_ms: float
    inserts_per_sec: float
    found_count: int
    inserted_count: int


def gen_duplication_array(spec: DuplicationSpec) -> np.ndarray:
    """(total, vlen) u32: total//d distinct random vectors, each repeated d
    times (the last one padded up to total), globally shuffled."""
    rng = np.random.default_rng(spec.seed)
    u = spec.unique_count
    rows = np.unique(rng.integers(0, 1 << 32, size=(u + u // 8 + 16, spec.vector_length),
                                  dtype=np.uint64), axis=0)
    while len(rows) < u:
        more = rng.integers(0, 1 << 32, size=(u, spec.vector_length), dtype=np.uint64)
        rows = np.unique(np.vstack([rows, more]), axis=0)
    rows = rows[rng.permutation(len(rows))[:u]].astype(np.uint32)
    picks = np.minimum(rng.permutation(spec.total) // spec.duplication, u - 1)
    return rows[picks]


def gen_duplication_sequence(spec: DuplicationSpec) -> list:
    return [tuple(int(w) for w in row) for row in gen_duplication_array(spec)]


def insert_bench_table_config(spec: DuplicationSpec, bucket_words: int = 32,
                              layout: str | None = None, num_hash_functions: int = 8,
                              table_seed: int = DEFAULT_SEED) -> TableConfig:
    """Table sized so duplication 1 stays at <= 50% load."""
    probe = TableConfig(bucket_words=bucket_words, layout=layout)
    spb = slots_per_bucket(bucket_words, spec.vector_length, probe.resolved_layout())
    buckets = max(num_hash_functions, -(-2 * spec.total // spb))
    return TableConfig(bucket_words=bucket_words, num_hash_functions=num_hash_functions,
                       capacity_words=buckets * bucket_words, layout=layout, seed=table_seed)


def run_insert_bench(spec: DuplicationSpec, table_cfg: TableConfig, threads: int = 1,
                     sequence=None) -> BenchRecord:
    """Insert the whole sequence into one device table and time only the
    insertion: CUDA events around the FINDORPUT kernel (gx_find_or_put_timed),
    with the sequence upload and the codes download outside the timed
    region, as the reference times only its insert loop (bench.py:161-169).
    `threads` is recorded for CSV compatibility.  Verifies found + inserted
    == total and inserted == occupancy (bench.py:176-190)."""
    from ._lib import ptr
    table = StateTable(table_cfg, spec.vector_length)
    try:
        arr = gen_duplication_array(spec) if sequence is None else \
            np.asarray(sequence, np.uint32).reshape(-1, spec.vector_length)
        arr = np.ascontiguousarray(arr, np.uint32)
        codes = np.zeros(len(arr), np.uint8)
        ms = C.c_double()
        check(lib().gx_find_or_put_timed(table.handle, ptr(arr), len(arr), ptr(codes, C.c_uint8),
                                         C.byref(ms)))
        wall = ms.value / 1e3
        if (codes == TABLE_FULL).any():
            raise RuntimeError("table full during benchmark; sizing precondition violated")
        inserted = int((codes == 1).sum())
        occupied = table.occupancy()[0]
        if inserted != occupied:
            raise RuntimeError(f"insert accounting mismatch: {inserted} inserts vs occupancy {occupied}")
    finally:
        table.close()
    return BenchRecord(total=spec.total, duplication=spec.duplication,
                       vector_length=spec.vector_length, seed=spec.seed,
                       bucket_words=table_cfg.bucket_words, threads=threads, wall_ms=wall * 1e3,
                       inserts_per_sec=spec.total / wall if wall > 0 else 0.0,
                       found_count=spec.total - inserted, inserted_count=inserted)


def device_insert_bench(table: StateTable, total: int, duplication: int = 1, seed: int = 1,
                        key_bits: int = 31, probe_group: int = 0, row_base: int = 0) -> dict:
    """The paper's Fig. 4 protocol entirely on the device: `total` FINDORPUT
    operations over total//duplication unique random vectors (key_bits
    bits per word), generated inside the kernel; CUDA-event time."""
    ms = C.c_double()
    found, ins, full, loads = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(lib().gx_bench_find_or_put_rows(table.handle, total, duplication, row_base, seed,
                                          key_bits, probe_group, C.byref(ms), C.byref(found),
                                          C.byref(ins), C.byref(full), C.byref(loads)))
    return {"ms": ms.value, "found": found.value, "inserted": ins.value, "full": full.value,
            "ops_per_sec": total / (ms.value / 1e3) if ms.value > 0 else 0.0,
            "buckets_per_op": loads.value / total if total else 0.0}


def random_access_roofline(granularity: int, buffer_bytes: int = 32 << 30, reads: int = 1 << 28,
                           with_cas: bool = False, repeats: int = 3) -> dict:
    """R(g): aligned random g-byte reads over a buffer >> L2 (SURVEY.md
    §8(d) denominator).  Returns {"g", "gbs", "ms", "segments_per_sec"}."""
    ms, gbs = C.c_double(), C.c_double()
    check(lib().gx_random_access_bench(buffer_bytes, granularity, reads, int(with_cas), repeats,
                                       C.byref(ms), C.byref(gbs)))
    return {"g": granularity, "gbs": gbs.value, "ms": ms.value, "with_cas": with_cas,
            "segments_per_sec": reads / (ms.value / 1e3), "buffer_bytes": buffer_bytes}


BENCH_CSV_COLUMNS = ("total", "duplication", "vector_length", "bucket_words", "threads", "seed",
                     "rep", "wall_ms", "inserts_per_sec", "found", "inserted")


def duplication_grid(total: int = 1_000_000, duplications=DUPLICATION_GRID, bucket_sizes=(4, 32),
                     repetitions: int = 5, threads: int = 1, vector_length: int = 1,
                     seed: int = DEFAULT_SEED, csv_path=None, progress=None) -> list:
    records = []
    for dup in duplications:
        spec = DuplicationSpec(total=total, duplication=dup, vector_length=vector_length, seed=seed)
        seq = gen_duplication_array(spec)
        for bw in bucket_sizes:
            cfg = insert_bench_table_config(spec, bw)
            for rep in range(repetitions):
                rec = run_insert_bench(spec, cfg, threads=threads, sequence=seq)
                records.append((rep, rec))
                if progress is not None:
                    progress(rec)
    if csv_path is not None:
        with open(csv_path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(BENCH_CSV_COLUMNS)
            for rep, r in records:
                w.writerow([r.total, r.duplication, r.vector_length, r.bucket_words, r.threads,
                            r.seed, rep, f"{r.wall_ms:.3f}", f"{r.inserts_per_sec:.1f}",
                            r.found_count, r.inserted_count])
    return [r for _, r in records]


# ------------------------------------------------------------ generators

def _write_net(out: Path, rules, files, comment: str) -> Path:
    exp = (f"-- {comment}\npar using\n    " + ",\n    ".join(rules) + "\nin\n    "
           + "\n    || ".join(files) + "\nend par\n")
    path = out / "net.exp"
    path.write_text(exp, encoding="utf-8")
    return path


def _rule(total: int, parts, result: str) -> str:
    cols = ["_"] * total
    for idx, act in parts:
        cols[idx] = act
    return " * ".join(cols) + f" -> {result}"


def gen_token_ring(nodes: int, out_dir) -> tuple:
    """Token ring (docs/models.md of the reference): N five-state nodes,
    rule i = put_i x get_(i+1 mod N) -> pass.  states(N) = 2 N 3^(N-1).
    Supports 2..20 nodes (the reference stops at 16)."""
    if not 2 <= nodes <= 20:
        raise ValueError("token ring supports 2..20 nodes")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    node = lambda init: (f"des ({init}, 5, 5)\n" '(0, "i", 1)\n(1, "put", 2)\n(2, "i", 3)\n'
                         '(3, "i", 4)\n(4, "get", 0)\n')
    holder, idler = out / "node_token.aut", out / "node_idle.aut"
    holder.write_text(node(0), encoding="utf-8")
    idler.write_text(node(2), encoding="utf-8")
    rules = [_rule(nodes, [(i, "put"), ((i + 1) % nodes, "get")], "pass") for i in range(nodes)]
    files = ['"node_token.aut"'] + ['"node_idle.aut"'] * (nodes - 1)
    return [holder, idler], _write_net(out, rules, files,
                                       f"token ring with {nodes} nodes: one token passed around the ring")


def gen_gas_station(customers: int, out_dir) -> tuple:
    """Gas station: operator, two pumps, N customers, 6N+2 binary rules
    (construction of the reference's docs/models.md).  2..16 customers."""
    if not 2 <= customers <= 16:
        raise ValueError("gas station supports 2..16 customers")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    texts = {
        "operator.aut": 'des (0, 3, 2)\n(0, "pay", 1)\n(1, "activate", 0)\n(0, "change", 0)\n',
        "pump.aut": 'des (0, 3, 3)\n(0, "activate", 1)\n(1, "start", 2)\n(2, "finish", 0)\n',
        "customer.aut": ('des (0, 4, 4)\n(0, "pay", 1)\n(1, "start", 2)\n(2, "finish", 3)\n'
                         '(3, "change", 0)\n'),
    }
    paths = []
    for name, text in texts.items():
        (out / name).write_text(text, encoding="utf-8")
        paths.append(out / name)
    n = customers
    total = n + 3
    rules = [_rule(total, [(0, "pay"), (3 + c, "pay")], "pay") for c in range(n)]
    rules += [_rule(total, [(0, "activate"), (1 + p, "activate")], "activate") for p in range(2)]
    for c in range(n):
        for p in range(2):
            rules.append(_rule(total, [(1 + p, "start"), (3 + c, "start")], "start"))
            rules.append(_rule(total, [(1 + p, "finish"), (3 + c, "finish")], "finish"))
    rules += [_rule(total, [(0, "change"), (3 + c, "change")], "change") for c in range(n)]
    files = ['"operator.aut"', '"pump.aut"', '"pump.aut"'] + ['"customer.aut"'] * n
    return paths, _write_net(out, rules, files, f"gas station: one operator, two pumps, {n} customers")


def gen_philosophers(n: int, out_dir) -> tuple:
    """Dining philosophers, left fork first: the deadlocking family of
    SURVEY §8(f2) (a generator in the reference's pattern, bench.py:245-359).
    N philosophers (takeL, takeR, putL, putR) and N forks (take, put); rule
    (i, a) synchronises philosopher i's action a with fork i (left) or fork
    i+1 mod N (right).  Exactly one deadlock: every philosopher holding its
    left fork.  2..16 philosophers (vlen 1 up to 10, 2 beyond)."""
    if not 2 <= n <= 16:
        raise ValueError("philosophers supports 2..16")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    phil, fork = out / "phil.aut", out / "fork.aut"
    phil.write_text('des (0, 4, 4)\n(0, "takeL", 1)\n(1, "takeR", 2)\n(2, "putL", 3)\n'
                    '(3, "putR", 0)\n', encoding="utf-8")
    fork.write_text('des (0, 2, 2)\n(0, "take", 1)\n(1, "put", 0)\n', encoding="utf-8")
    total = 2 * n
    rules = []
    for i in range(n):
        left, right = n + i, n + (i + 1) % n
        for act, f, fact in (("takeL", left, "take"), ("takeR", right, "take"),
                             ("putL", left, "put"), ("putR", right, "put")):
            rules.append(_rule(total, [(i, act), (f, fact)], f"{act}{i}"))
    files = ['"phil.aut"'] * n + ['"fork.aut"'] * n
    return [phil, fork], _write_net(out, rules, files,
                                    f"dining philosophers, {n} philosophers, left fork first")


def gen_peterson(procs: int, out_dir) -> tuple:
    """Peterson's N-process filter lock as a network of LTSs (the BEEM
    "peterson" family the paper's peterson7 row comes from).

    Shared variables are processes: level[i] (values 0..N-1) and victim[l]
    (l = 1..N-1, values 0..N-1).  Process i, for l = 1..N-1: level[i] := l,
    victim[l] := i, then scans k = 0..N-1 (k != i): it passes k when
    level[k] < l, and leaves the wait early when victim[l] != i.  After
    level N-1 it enters the critical section, then resets level[i] := 0.
    Every step is a binary synchronisation (process x variable) or an
    internal move, so the product exercises many rules per state.
    """
    n = procs
    if not 2 <= n <= 8:
        raise ValueError("peterson supports 2..8 processes")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    # process program counters
    pcs = {"idle": 0}

    def pc(key):
        if key not in pcs:
            pcs[key] = len(pcs)
        return pcs[key]

    paths = []
    rules = []
    nvar_level = n
    nvar_victim = n - 1
    total = n + nvar_level + nvar_victim
    lvl_idx = lambda k: n + k
    vic_idx = lambda l: n + nvar_level + (l - 1)
    # one automaton per process (labels are process specific)
    for i in range(n):
        pcs.clear()
        pcs["idle"] = 0
        tr = []
        cur = pc("idle")
        for l in range(1, n):
            a = pc(("setvic", l))
            tr.append((cur, f"setlv{l}", a))
            ks = [k for k in range(n) if k != i]
            w0 = pc(("wait", l, ks[0]))
            tr.append((a, f"setvic{l}", w0))
            nxt = pc(("lvl_done", l))
            for j, k in enumerate(ks):
                w = pc(("wait", l, k))
                after = pc(("wait", l, ks[j + 1])) if j + 1 < len(ks) else nxt
                tr.append((w, f"lt{l}_{k}", after))
                tr.append((w, f"nv{l}", nxt))
            cur = nxt
        cs = cur
        tr.append((cs, "cs", pc("exit")))
        tr.append((pc("exit"), "reset", pcs["idle"]))
        text = f"des (0, {len(tr)}, {len(pcs)})\n" + "".join(f'({s}, "{a}", {d})\n' for s, a, d in tr)
        p = out / f"proc{i}.aut"
        p.write_text(text, encoding="utf-8")
        paths.append(p)
        for l in range(1, n):
            rules.append(_rule(total, [(i, f"setlv{l}"), (lvl_idx(i), f"set{l}")], f"level{i}"))
            rules.append(_rule(total, [(i, f"setvic{l}"), (vic_idx(l), f"set{i}")], f"victim{l}"))
            for k in range(n):
                if k != i:
                    rules.append(_rule(total, [(i, f"lt{l}_{k}"), (lvl_idx(k), f"lt{l}")], f"check{i}"))
            rules.append(_rule(total, [(i, f"nv{l}"), (vic_idx(l), f"ne{i}")], f"check{i}"))
        rules.append(_rule(total, [(i, "reset"), (lvl_idx(i), "set0")], f"level{i}"))
    # level variable: set{x} from anywhere, lt{l} self-loop where value < l
    tr = [(v, f"set{x}", x) for v in range(n) for x in range(n)]
    tr += [(v, f"lt{l}", v) for l in range(1, n) for v in range(n) if v < l]
    lv = out / "level.aut"
    lv.write_text(f"des (0, {len(tr)}, {n})\n" + "".join(f'({s}, "{a}", {d})\n' for s, a, d in tr),
                  encoding="utf-8")
    # victim variable: set{i} from anywhere, ne{i} self-loop where value != i
    tr = [(v, f"set{x}", x) for v in range(n) for x in range(n)]
    tr += [(v, f"ne{i}", v) for i in range(n) for v in range(n) if v != i]
    vc = out / "victim.aut"
    vc.write_text(f"des (0, {len(tr)}, {n})\n" + "".join(f'({s}, "{a}", {d})\n' for s, a, d in tr),
                  encoding="utf-8")
    paths += [lv, vc]
    files = [f'"proc{i}.aut"' for i in range(n)] + ['"level.aut"'] * nvar_level + \
        ['"victim.aut"'] * nvar_victim
    return paths, _write_net(out, rules, files, f"Peterson filter lock, {n} processes")


# ------------------------------------------------------- bucket sweep

SWEEP_CSV_COLUMNS = ("model", "bucket", "mean_ms", "normalized", "reps", "outcome")
BASELINE_BUCKET_WORDS = 32


@dataclass(frozen=True)
class SweepCell:
    model: str
    bucket_words: int
    mean_ms: float
    normalized: float
    repetitions: int
    outcome: str
    states: int
    transitions: int


def bucket_size_sweep(network, model_name: str = "model", sizes=(4, 8, 16, 32),
                      repetitions: int = 5, explore_cfg: ExploreConfig | None = None,
                      csv_path=None) -> list:
    """Explore once per bucket size, `repetitions` times, normalised to 32."""
    if not isinstance(network, Network):
        model_name = Path(network).stem if model_name == "model" else model_name
        network = load_network(network)
    base = explore_cfg or ExploreConfig()
    cells = []
    for bw in sizes:
        cfg = ExploreConfig(
            workers=base.workers,
            table=TableConfig(bucket_words=bw, num_hash_functions=base.table.num_hash_functions,
                              capacity_words=base.table.capacity_words, layout=None,
                              seed=base.table.seed),
            cache_slots=base.cache_slots, detect_deadlocks=base.detect_deadlocks,
            max_iterations=base.max_iterations, backend=base.backend,
            frontier_capacity=base.frontier_capacity, probe_group=0)
        times, outcome, st, tr = [], "COMPLETE", 0, 0
        for _ in range(repetitions):
            rep = explore(network, cfg)
            times.append(rep.wall_time * 1e3)
            st, tr = rep.states, rep.transitions
            if rep.outcome != "COMPLETE":
                outcome = rep.outcome
        cells.append([model_name, bw, statistics.mean(times), repetitions, outcome, st, tr])
    base_ms = next((c[2] for c in cells if c[1] == BASELINE_BUCKET_WORDS and c[4] == "COMPLETE"), None)
    res = [SweepCell(m, bw, ms, ms / base_ms if base_ms else float("nan"), r, o, s, t)
           for m, bw, ms, r, o, s, t in cells]
    if csv_path is not None:
        with open(csv_path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(SWEEP_CSV_COLUMNS)
            for c in res:
                w.writerow([c.model, c.bucket_words, f"{c.mean_ms:.3f}", f"{c.normalized:.4f}",
                            c.repetitions, c.outcome])
    return res
