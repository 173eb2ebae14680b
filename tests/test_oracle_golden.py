"""Pin the CPU oracle (oracle/gx_oracle.c) to the real reference through the
golden vectors in tests/golden/ (made by tests/golden/make_golden.py from
/root/reference/pkg/src).  CPU only."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden_models, model_path
from oracle import oracle as O

HALF = {"half": O.HALF, "plain": O.PLAIN}


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


@pytest.fixture(scope="module")
def kats():
    return json.loads((GOLDEN / "hash_kats.json").read_text())


def test_hash_constants(kats):
    for seed, entry in kats["constants"].items():
        pairs, salt = O.hash_constants(int(seed), 8)
        assert [list(p) for p in pairs] == entry["pairs"]
        assert salt == entry["salt"]


def test_fold(kats):
    for e in kats["fold"]:
        _, salt = O.hash_constants(e["seed"], 1)
        assert O.fold(salt, e["p"]) == e["h"]


def test_probe_sequences(kats):
    for e in kats["probe"]:
        assert O.probe_raw(e["seed"], 8, e["nb"], e["p"]) == e["seq"], e


def test_survey_hash_kats():
    # SURVEY.md Appendix B.3, derived from the reference
    pairs, salt = O.hash_constants(42, 2)
    assert pairs[0] == (0xBDD732262FEB6E95, 0x28EFE333B266F103)
    assert salt == 0xFB3B2A8C40D00A64
    assert O.fold(salt, (0,)) == 0x43E52476AC286991
    assert O.probe_raw(42, 8, 1000, (7,)) == [81, 582, 616, 994, 156, 824, 1, 632]


def test_slots_per_bucket(kats):
    for e in kats["spb"]:
        if isinstance(e["spb"], int):
            assert O.slots_per_bucket(e["bw"], e["vlen"], HALF[e["layout"]]) == e["spb"]
        else:
            with pytest.raises(ValueError, match="too long|even"):
                O.slots_per_bucket(e["bw"], e["vlen"], HALF[e["layout"]])


def test_py_tuple_hash_matches_cpython():
    for p in [(0,), (7,), (1, 2), (2**32 - 1, 5, 9), tuple(range(16))]:
        assert O.py_tuple_hash(p) == hash(p)


def table_cases():
    meta = json.loads((GOLDEN / "table_runs.json").read_text())
    return meta


@pytest.mark.parametrize("case", table_cases(), ids=lambda c: c["key"])
def test_table_runs(case):
    arr = np.load(GOLDEN / "table_runs.npz")
    k = case["key"]
    t = O.Table(case["bw"], case["k"], case["capacity_words"], case["layout"], case["seed"],
                case["vlen"])
    assert (t.slots_per_bucket, t.num_buckets) == (case["spb"], case["num_buckets"])
    codes, handles = t.find_or_insert_batch(arr[k + "_seq"])
    assert np.array_equal(codes, arr[k + "_codes"])
    assert np.array_equal(handles, arr[k + "_handles"])
    claimed = [int(t.claim_new(int(h))) for h in handles[::3] if h >= 0]
    assert claimed == arr[k + "_claimed"].tolist()
    assert t.scan_new(0, t.num_buckets) == arr[k + "_scan"].tolist()
    assert t.scan_new(t.num_buckets // 3, t.num_buckets // 2) == arr[k + "_scan_half"].tolist()
    assert list(t.occupancy()[:2]) == case["occupancy"]
    hs, st, ws = t.occupied()
    spb = t.slots_per_bucket
    rows = [(int(h) // spb, int(h) % spb, "NEW" if s == O.NEW else "OLD", [int(x) for x in w])
            for h, s, w in zip(hs, st, ws)]
    assert sha(json.dumps(rows)) == case["dump_rows_sha"]


MODELS = golden_models()


@pytest.mark.parametrize("name", sorted(MODELS))
def test_model_bfs_counts(name):
    g = MODELS[name]
    if "error" in g:
        with pytest.raises(ValueError):
            O.Net.from_file(model_path(name))
        return
    if g["bfs"]["states"] > 200_000:
        pytest.skip("large model covered by the explore run / GPU tests")
    net = O.Net.from_file(model_path(name))
    got = net.bfs()
    assert got["states"] == g["bfs"]["states"]
    assert got["transitions"] == g["bfs"]["transitions"]
    assert got["deadlocks"] == g["bfs"]["deadlocks_total"]


@pytest.mark.parametrize("name", sorted(MODELS))
def test_model_explore_runs(name):
    """explore(workers=1) restated: report, --dump-states and --dump-table
    byte-identical to the reference (placement included)."""
    g = MODELS[name]
    if "error" in g or not g["runs"]:
        pytest.skip("no explore run recorded")
    net = O.Net.from_file(model_path(name))
    for run in g["runs"]:
        tc = run["table"]
        if "error" in run:
            with pytest.raises(ValueError, match="too long"):
                O.explore(net, detect_deadlocks=True, max_iterations=run["max_iterations"], **tc)
            continue
        r = O.explore(net, detect_deadlocks=True, max_iterations=run["max_iterations"], **tc)
        want = run["report"]
        got = {"states": r.states, "transitions": r.transitions,
               "deadlocks": [list(s) for s in r.deadlocks], "deadlocks_total": r.deadlocks_total,
               "expanded": r.expanded, "iterations": r.iterations, "outcome": r.outcome}
        assert got == want, (name, tc)
        assert sha(r.dump_states()) == run["dump_states_sha"], (name, tc)
        assert sha(r.dump_table()) == run["dump_table_sha"], (name, tc)


def test_expand_kats():
    kats = json.loads((GOLDEN / "expand_kats.json").read_text())
    for name, rows in kats.items():
        net = O.Net.from_file(model_path(name))
        for s, count, succ in rows:
            got, c = net.expand(s)
            assert c == count, (name, s)
            assert [[a, list(t)] for a, t in got] == succ, (name, s)


def test_iterations_are_levels_plus_one():
    for name in ("fig1", "ring5", "gas4"):
        net = O.Net.from_file(model_path(name))
        r = O.explore(net)
        assert r.iterations == net.bfs()["levels"] + 1
