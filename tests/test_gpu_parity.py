"""Parity of the B200 path (libgx via the Python API) with the oracle and the
reference's golden vectors.  GPU only."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden_models, model_path
from oracle import oracle as O

pytestmark = pytest.mark.gpu

gx = pytest.importorskip("paper_1801_05857_b200")
from paper_1801_05857_b200 import statevec  # noqa: E402
from paper_1801_05857_b200.explore import DeviceNetwork, ExploreConfig, Explorer  # noqa: E402
from paper_1801_05857_b200.hashtable import StateTable, TableConfig  # noqa: E402

MODELS = golden_models()
REF_DIGESTS = json.loads((GOLDEN / "ref_digests.json").read_text())


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


# ------------------------------------------------------------------ table

def table_cases():
    return json.loads((GOLDEN / "table_runs.json").read_text())


@pytest.mark.parametrize("case", table_cases(), ids=lambda c: c["key"])
def test_serial_table_runs_match_reference(case):
    """Serial FINDORPUT reproduces the reference's placement handle for
    handle, then claim / scan / occupancy / dump equal the golden run."""
    arr = np.load(GOLDEN / "table_runs.npz")
    k = case["key"]
    t = StateTable(TableConfig(bucket_words=case["bw"], num_hash_functions=case["k"],
                               capacity_words=case["capacity_words"], layout=case["layout"],
                               seed=case["seed"]), case["vlen"])
    try:
        codes, handles = t.find_or_insert_batch(arr[k + "_seq"], serial=True)
        assert np.array_equal(codes, arr[k + "_codes"])
        assert np.array_equal(handles, arr[k + "_handles"])
        hs = handles[::3]
        claimed = [int(t.claim_new(int(h))) for h in hs[hs >= 0]]  # sequential, as the reference
        assert claimed == arr[k + "_claimed"].tolist()
        assert t.scan_new(0, t.num_buckets) == arr[k + "_scan"].tolist()
        assert t.scan_new(t.num_buckets // 3, t.num_buckets // 2) == arr[k + "_scan_half"].tolist()
        assert list(t.occupancy()[:2]) == case["occupancy"]
        rows = [(b, j, st, list(w)) for b, j, st, w in t.dump_rows()]
        assert sha(json.dumps(rows)) == case["dump_rows_sha"]
    finally:
        t.close()


@pytest.mark.parametrize("bw", [4, 8, 16, 32])
@pytest.mark.parametrize("vlen", [1, 2, 4])
def test_mark_mode_serial_placement(bw, vlen):
    """In-band (mark bit) tables place keys exactly where the reference does."""
    if vlen > bw:
        pytest.skip("vector longer than bucket")
    rng = np.random.default_rng(bw * 10 + vlen)
    n = 2000
    keys = (rng.integers(0, 1 << 31, size=(n, vlen), dtype=np.uint64)).astype(np.uint32)
    keys = np.concatenate([keys, keys[: n // 2]])
    cap = bw * max(16, (2 * n) // max(1, bw // vlen))
    t = StateTable(TableConfig(bucket_words=bw, capacity_words=cap), vlen, mark=(vlen - 1, 31))
    assert t.mode == "mark"
    o = O.Table(bw, 8, cap, None, 42, vlen)
    try:
        codes, handles = t.find_or_insert_batch(keys, serial=True)
        ocodes, ohandles = o.find_or_insert_batch(keys)
        assert np.array_equal(codes, ocodes)
        assert np.array_equal(handles, ohandles)
        _, words = t.read_slots(handles[codes != 2])
        assert np.array_equal(words, keys[codes != 2])
    finally:
        t.close()


@pytest.mark.parametrize("mark", [None, (0, 31)])
@pytest.mark.parametrize("bw", [4, 8, 16, 32])
def test_concurrent_batch_semantics(mark, bw):
    """One parallel batch with heavy duplication: exactly one INSERTED per
    distinct key, equal keys share one handle, occupancy exact, dump
    duplicate-free (test_hashtable.py:187-211, acceptance criterion 4)."""
    rng = np.random.default_rng(bw)
    uniq = np.unique(rng.integers(0, 1 << 31, size=100_000, dtype=np.uint64)).astype(np.uint32)
    seq = np.concatenate([uniq] * 8)[rng.permutation(8 * len(uniq))]
    cap = bw * (4 * len(uniq) // max(1, bw) + 64)
    t = StateTable(TableConfig(bucket_words=bw, capacity_words=cap), 1, mark=mark)
    try:
        codes, handles = t.find_or_insert_batch(seq)
        assert (codes != 2).all()
        assert int((codes == 1).sum()) == len(uniq)
        by_key = {}
        for kk, h in zip(seq.tolist(), handles.tolist()):
            assert by_key.setdefault(kk, h) == h
        assert t.occupancy()[0] == len(uniq)
        hs, st, ws = t.dump_arrays()
        assert len(hs) == len(uniq)
        assert np.array_equal(np.sort(ws[:, 0]), uniq)
        assert (st == 2).all()
    finally:
        t.close()


@pytest.mark.parametrize("mark", [None, (0, 31)])
def test_table_full_preserves_contents(mark):
    t = StateTable(TableConfig(bucket_words=4, capacity_words=4 * 32, num_hash_functions=4), 1,
                   mark=mark)
    try:
        rng = np.random.default_rng(1)
        keys = rng.integers(0, 1 << 31, size=(5000, 1), dtype=np.uint64).astype(np.uint32)
        codes, _ = t.find_or_insert_batch(keys, serial=True)
        assert (codes == 2).any()
        kept = keys[codes == 1]
        codes2, _ = t.find_or_insert_batch(kept)
        assert (codes2 == 0).all()
        assert t.occupancy()[0] == len(kept)
    finally:
        t.close()


def test_all_zero_vector_and_status_lifecycle():
    for mark in (None, (1, 31)):
        t = StateTable(TableConfig(bucket_words=16, capacity_words=16 * 64), 2, mark=mark)
        c, h = t.find_or_insert((0, 0))
        assert c == 1 and t.find_or_insert((0, 0)) == (0, h)
        assert t.slot_status(h) == 2
        assert t.claim_new(h) and not t.claim_new(h)
        assert t.slot_status(h) == 3
        assert t.occupancy()[:2] == (1, 0)
        assert t.read_slot(h) == (0, 0)
        t.close()


def test_claim_race_exactly_once():
    t = StateTable(TableConfig(bucket_words=8, capacity_words=8 * 1024), 1)
    try:
        _, handles = t.find_or_insert_batch(np.arange(2000, dtype=np.uint32).reshape(-1, 1))
        won = t.claim_new_batch(np.concatenate([handles] * 16))
        assert won.sum() == 2000
        per = won.reshape(16, 2000).sum(axis=0)
        assert (per == 1).all()
    finally:
        t.close()


def test_hash_constants_and_probe_sequence():
    t = StateTable(TableConfig(capacity_words=32 * 1000), 1)
    try:
        pairs, salt = t.device_hash_constants()
        opairs, osalt = O.hash_constants(42, 8)
        assert pairs == opairs and salt == osalt
        assert t.probe_sequence((7,)) == [81, 582, 616, 994, 156, 824, 1, 632]
    finally:
        t.close()


# ---------------------------------------------------------------- explore

def _run(name, table, max_iterations=None, **kw):
    net = gx.load_network(model_path(name))
    cfg = ExploreConfig(table=TableConfig(**table), detect_deadlocks=True,
                        max_iterations=max_iterations, **kw)
    ex = Explorer(net, cfg)
    try:
        rep = ex.run()
        return rep, ex.dump_states(), ex
    except Exception:
        ex.close()
        raise


@pytest.mark.parametrize("name", sorted(n for n in MODELS if "error" not in MODELS[n]))
def test_explore_matches_reference(name):
    g = MODELS[name]
    runs = g["runs"] or [{"table": {"bucket_words": 32, "capacity_words": 1 << 22},
                          "max_iterations": None, "report": None}]
    for run in runs:
        if "error" in run:
            with pytest.raises(ValueError, match="too long"):
                _run(name, run["table"])
            continue
        rep, dump, ex = _run(name, run["table"], run["max_iterations"])
        try:
            want = run["report"]
            if want is None:  # large model: sequential_bfs counts pin it
                b = g["bfs"]
                assert (rep.states, rep.transitions, rep.deadlocks_total) == \
                    (b["states"], b["transitions"], b["deadlocks_total"])
                assert rep.outcome == "COMPLETE"
                continue
            if want["outcome"] == "TABLE_FULL":
                # placement (hence the fill cliff) is schedule dependent: a
                # run may complete, then it must be exact; else invariants
                if rep.outcome == "COMPLETE":
                    b = g["bfs"]
                    assert (rep.states, rep.transitions, rep.deadlocks_total) == \
                        (b["states"], b["transitions"], b["deadlocks_total"])
                    continue
                assert rep.outcome == "TABLE_FULL"
                assert 0 < rep.states < g["bfs"]["states"]
                lines = dump.splitlines()
                assert len(lines) == len(set(lines)) == rep.states
                continue
            if want["deadlocks_total"] > 100:
                # the reference keeps the first 100 *recorded* (order dependent);
                # the device keeps the 100 smallest = sequential_bfs's sorted head
                want = dict(want, deadlocks=g["bfs"]["deadlocks"][:100])
            got = {"states": rep.states, "transitions": rep.transitions,
                   "deadlocks": [list(s) for s in rep.deadlocks],
                   "deadlocks_total": rep.deadlocks_total, "expanded": rep.expanded,
                   "iterations": rep.iterations, "outcome": rep.outcome}
            assert got == want, (name, run["table"])
            assert sha(dump) == run["dump_states_sha"], (name, run["table"])
            if rep.outcome == "COMPLETE":
                assert list(rep.digest) == REF_DIGESTS[name], (name, run["table"])
            hs, st, _ = ex.table.dump_arrays()
            occ, new, _ = ex.table.occupancy()
            assert occ == rep.states and new == int((st == 2).sum())
        finally:
            ex.close()


def test_expand_kats_on_device():
    """Device successor generation: transition count and successor set of
    every reachable state of the small golden models (network.py:184-238)."""
    kats = json.loads((GOLDEN / "expand_kats.json").read_text())
    for name, rows in kats.items():
        net = gx.load_network(model_path(name))
        sc = statevec.make_scheme(net)
        dn = DeviceNetwork(net, sc)
        try:
            packed = np.array([statevec.pack(sc, s) for s, _, _ in rows], np.uint32)
            counts, nsucc, succ = dn.expand_batch(packed)
            off = 0
            for (s, count, succ_ref), c, n in zip(rows, counts, nsucc):
                assert int(c) == count, (name, s)
                got = {tuple(int(x) for x in r) for r in succ[off:off + n]}
                off += int(n)
                want = {statevec.pack(sc, tuple(t)) for _, t in succ_ref}
                me = statevec.pack(sc, tuple(s))
                assert got - {me} == want - {me}, (name, s)
        finally:
            dn.close()


@pytest.mark.parametrize("bw", [4, 8, 16, 32])
@pytest.mark.parametrize("group", [0, 1])
def test_bucket_sizes_and_probe_groups(bw, group):
    for name in ("ring8", "gas7", "phil5", "counter8", "sinks8", "wide33"):
        b = MODELS[name]["bfs"]
        rep, dump, ex = _run(name, {"bucket_words": bw, "capacity_words": 1 << 22}, probe_group=group)
        ex.close()
        assert (rep.states, rep.transitions, rep.deadlocks_total, rep.outcome) == \
            (b["states"], b["transitions"], b["deadlocks_total"], "COMPLETE"), (name, bw)
        if "dump_sha" in b:
            assert sha(dump) == b["dump_sha"]


@pytest.mark.parametrize("n", [11, 12, 13, 14])
def test_token_ring_closed_forms(n, tmp_path):
    """states 2N 3^(N-1), transitions 4N^2 3^(N-2),
    levels 6N-4 (iterations = levels + 1)."""
    from paper_1801_05857_b200.bench import gen_token_ring
    _, p = gen_token_ring(n, tmp_path / f"ring{n}")
    net = gx.load_network(p)
    cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 28), detect_deadlocks=True)
    rep = gx.explore(net, cfg)
    assert rep.states == 2 * n * 3 ** (n - 1)
    assert rep.transitions == 4 * n * n * 3 ** (n - 2)
    assert rep.iterations == 6 * n - 4 + 1
    assert rep.deadlocks_total == 0 and rep.outcome == "COMPLETE"


@pytest.mark.parametrize("bw", [4, 8, 16, 32])
@pytest.mark.parametrize("group,cache", [(0, 1), (0, 4096), (2, 4096)])
def test_level_kernel_contention(bw, group, cache, tmp_path):
    """Exact state count under heavy insert contention: token ring N=13
    (4.78M states) in a table at load ~0.7 with K=32, so lost CASes, full
    first buckets and the rehash path are all exercised, with and without
    the block-local cache, staged (group 0) and register-group kernels."""
    from paper_1801_05857_b200.bench import gen_token_ring
    from paper_1801_05857_b200.hashtable import slots_per_bucket
    n = 13
    if group > 1 and bw < 8:
        pytest.skip("group wider than the bucket")
    _, p = gen_token_ring(n, tmp_path / "ring")
    net = gx.load_network(p)
    states = 2 * n * 3 ** (n - 1)
    spb = slots_per_bucket(bw, 2, "half" if bw == 32 else "plain")
    cap = (int(states / 0.7 / spb) + 64) * bw
    cfg = ExploreConfig(table=TableConfig(bucket_words=bw, num_hash_functions=32, capacity_words=cap),
                        detect_deadlocks=True, probe_group=group, cache_slots=cache)
    ex = Explorer(net, cfg)
    try:
        for _ in range(2):
            rep = ex.run()
            assert (rep.states, rep.transitions, rep.outcome) == \
                (states, 4 * n * n * 3 ** (n - 2), "COMPLETE")
        assert ex.table.occupancy()[0] == states
    finally:
        ex.close()


@pytest.mark.parametrize("kind,n", [("peterson", 3), ("peterson", 4), ("peterson", 5), ("gas", 9)])
def test_generated_models_match_oracle(kind, n, tmp_path):
    from paper_1801_05857_b200.bench import gen_gas_station, gen_peterson
    gen = gen_peterson if kind == "peterson" else gen_gas_station
    _, p = gen(n, tmp_path / f"{kind}{n}")
    want = O.Net.from_file(p).bfs()
    net = gx.load_network(p)
    rep = gx.explore(net, ExploreConfig(table=TableConfig(capacity_words=1 << 26),
                                        detect_deadlocks=True))
    assert (rep.states, rep.transitions, rep.iterations - 1, rep.deadlocks_total) == \
        (want["states"], want["transitions"], want["levels"], want["deadlocks"])


def test_deadlock_keep_smallest():
    """sinks10 has 1024 deadlocks: the report keeps the 100 smallest
    composite states (the reference keeps the first 100 recorded, which is
    schedule dependent above 100)."""
    rep, _, ex = _run("sinks10", {"capacity_words": 1 << 20})
    ex.close()
    assert rep.deadlocks_total == 1024
    from itertools import product
    want = sorted((1,) + bits for bits in product((2, 3), repeat=10))[:100]
    assert [tuple(s) for s in rep.deadlocks] == want


def test_cli_explore_json(capsys):
    """`python -m paper_1801_05857_b200 explore NET --json --deadlock` prints
    the reference's JSON report (docs/cli.md:28-55) with the golden counts."""
    from paper_1801_05857_b200.cli import main
    for name, extra in (("fig1", []), ("sinks8", ["--shards", "2"])):
        rc = main(["explore", str(model_path(name)), "--json", "--deadlock", "--table-mb", "4", *extra])
        assert rc == 0
        doc = json.loads(capsys.readouterr().out)
        b = MODELS[name]["bfs"]
        assert (doc["states"], doc["transitions"], doc["deadlocks_total"], doc["outcome"]) == \
            (b["states"], b["transitions"], b["deadlocks_total"], "COMPLETE")
        assert doc["config"]["bucket_words"] == 32


@pytest.mark.parametrize("bw", [4, 8, 16, 32])
@pytest.mark.parametrize("vlen", [1, 2])
def test_device_bench_reference_pins(bw, vlen):
    """The on-device duplication benchmark (the configs[1] numbers) counts
    exactly: found=4500 inserted=500 at (5000, d=10) (reference
    tests/test_cli.py:140-148), 47619 unique at (10^6, d=21)
    (tests/test_bench.py:37-39), and inserted == total // d == occupancy
    (bench.py:176-190) at every duplication."""
    from paper_1801_05857_b200.bench import (DuplicationSpec, device_insert_bench,
                                             insert_bench_table_config)
    for total, d in ((5000, 10), (10 ** 6, 21), (1 << 20, 1), (10 ** 6, 100), (3 << 20, 7)):
        spec = DuplicationSpec(total=total, duplication=d, vector_length=vlen)
        t = StateTable(insert_bench_table_config(spec, bw), vlen, mark=(vlen - 1, 31))
        try:
            r = device_insert_bench(t, total, d, seed=11)
            occ = t.occupancy()[0]
        finally:
            t.close()
        if r["full"]:
            # the reference's sizing (<= 50% load at d = 1, K = 8) overfills
            # buckets of <= 4 slots at these sizes: bw 4 / vlen 1,
            # bw 4 and 8 / vlen 2
            assert bw // vlen <= 4, (bw, vlen, total, d)
            continue
        assert (r["found"], r["inserted"], occ) == (total - total // d, total // d, total // d), (total, d)
        if (total, d) == (5000, 10):
            assert (r["found"], r["inserted"]) == (4500, 500)
        if (total, d) == (10 ** 6, 21):
            assert r["inserted"] == 47619


def test_run_insert_bench_and_cli_pins(tmp_path, capsys):
    """run_insert_bench on the reference's sequence semantics and the CLI's
    `bench-hash --total 5000 --dup 10` line (tests/test_cli.py:140-148)."""
    from paper_1801_05857_b200.bench import DuplicationSpec, insert_bench_table_config, run_insert_bench
    from paper_1801_05857_b200.cli import main
    spec = DuplicationSpec(total=10 ** 6, duplication=21)
    rec = run_insert_bench(spec, insert_bench_table_config(spec, 32))
    assert (rec.inserted_count, rec.found_count) == (47619, 10 ** 6 - 47619)
    assert rec.wall_ms > 0
    rc = main(["bench-hash", "--total", "5000", "--dup", "10", "--reps", "1", "--csv",
               str(tmp_path / "b.csv")])
    assert rc == 0
    assert "found=4500 inserted=500" in capsys.readouterr().out
    assert (tmp_path / "b.csv").exists()
