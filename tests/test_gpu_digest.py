"""Set identity on the device: the reachable-set digest (gx_table_digest)
of every engine equals the reference's (tests/golden/ref_digests.json) and
the oracle's / closed-form goldens for the large models
(tests/golden/digests.json: configs[2] peterson6, rings up to 16 here and
ring19 in bench.py).  Also the exact 100-smallest deadlocks when one level
has more deadlocks than the device record buffer holds.  GPU only."""
import json
from itertools import product

import pytest

from conftest import GOLDEN, golden_models, model_path

pytestmark = pytest.mark.gpu

gx = pytest.importorskip("paper_1801_05857_b200")
from paper_1801_05857_b200 import statevec  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig, slots_per_bucket  # noqa: E402

REF = json.loads((GOLDEN / "ref_digests.json").read_text())


def big():
    return json.loads((GOLDEN / "digests.json").read_text())
MODELS = golden_models()


@pytest.mark.parametrize("shards", [1, 2, 3])
def test_golden_model_digests(shards):
    for name in sorted(REF):
        net = gx.load_network(model_path(name))
        sc = statevec.make_scheme(net)
        v = statevec.device_vlen(sc)
        if shards > 1 and (v not in (1, 2, 4) or statevec.mark_bit(sc, v) is None):
            continue  # status-byte tables: single-table engine only
        rep = gx.explore(net, ExploreConfig(table=TableConfig(capacity_words=1 << 20),
                                            detect_deadlocks=True, shards=shards))
        assert rep.outcome == "COMPLETE", name
        assert list(rep.digest) == REF[name], (name, shards)
        b = MODELS[name]["bfs"]
        assert (rep.states, rep.transitions, rep.deadlocks_total) == \
            (b["states"], b["transitions"], b["deadlocks_total"]), name


def _gen(name, tmp_path):
    from paper_1801_05857_b200.bench import (gen_gas_station, gen_peterson, gen_philosophers,
                                             gen_token_ring)
    kind = name.rstrip("0123456789")
    gen = {"ring": gen_token_ring, "gas": gen_gas_station, "peterson": gen_peterson,
           "phil": gen_philosophers}[kind]
    return gen(int(name[len(kind):]), tmp_path / name)[1]


def _cap(states, vlen, load=0.5, bw=32):
    spb = slots_per_bucket(bw, vlen, "half" if bw == 32 else "plain")
    return (int(states / load / spb) + 64) * bw


BIG_NAMES = ["ring11", "ring12", "ring13", "ring14", "ring15", "ring16", "gas9", "gas10", "gas11",
             "peterson5", "peterson6", "phil12", "phil14"]


@pytest.mark.parametrize("shards", [1, 2])
@pytest.mark.parametrize("name", BIG_NAMES)
def test_large_models_equal_oracle(name, shards, tmp_path):
    """configs[2] (peterson6, 2.1e8 states) and the scaled rings / gas
    stations: states, transitions, levels, deadlocks and the set digest
    equal the oracle's full exploration (rings past 14: the closed-form
    enumeration of the reachable set)."""
    e = big()[name]
    net = gx.load_network(_gen(name, tmp_path))
    per = e["states"] // shards + (e["states"] >> 6) + 4096
    cfg = ExploreConfig(table=TableConfig(capacity_words=_cap(per, 2 if e["vlen"] == 2 else e["vlen"]),
                                          num_hash_functions=16),
                        detect_deadlocks=True, shards=shards)
    rep = gx.explore(net, cfg)
    assert rep.outcome == "COMPLETE"
    assert (rep.states, rep.transitions, rep.deadlocks_total) == \
        (e["states"], e["transitions"], e["deadlocks_total"])
    if "iterations" in e:
        assert rep.iterations == e["iterations"]
        assert [list(s) for s in rep.deadlocks] == e["deadlocks"]
    assert list(rep.digest) == e["digest"]


def _sinks(n, out):
    """n processes that each step once into one of two sinks after a
    shared `go`: 2^n deadlocks, all in the last level."""
    out.mkdir(parents=True, exist_ok=True)
    (out / "s.aut").write_text('des (0, 3, 4)\n(0,"go",1)\n(1,"a",2)\n(1,"b",3)\n')
    (out / "g.aut").write_text('des (0, 1, 2)\n(0,"go",1)\n')
    (out / "net.exp").write_text("par using\n  " + " * ".join(["go"] * (n + 1)) + " -> go\nin\n  "
                                 + " || ".join(['"g.aut"'] + ['"s.aut"'] * n) + "\nend par\n")
    return out / "net.exp"


@pytest.mark.parametrize("shards", [1, 2])
def test_deadlocks_beyond_record_buffer(shards, tmp_path):
    """2^17 = 131072 deadlocks in one level, twice the device's per-level
    record buffer (65536): the report still holds the exact 100 smallest
    (explore.py:220-226, 361-367) and the exact total."""
    n = 17
    net = gx.load_network(_sinks(n, tmp_path / "sinks"))
    states = 1 + 3 ** n
    rep = gx.explore(net, ExploreConfig(table=TableConfig(capacity_words=_cap(states // shards + 4096, 2)),
                                        detect_deadlocks=True, shards=shards))
    assert rep.outcome == "COMPLETE" and rep.states == states
    assert rep.deadlocks_total == 2 ** n
    want = sorted((1,) + bits for bits in product((2, 3), repeat=n))[:100]
    assert [tuple(s) for s in rep.deadlocks] == want


@pytest.mark.parametrize("name", ["ring13", "peterson5", "phil12"])
def test_device_sorted_dump_at_scale(name, tmp_path):
    """gx_dump_sorted (the canonical dump's order, statevec.py:93-100) on
    1e6-1e7 states: strictly increasing rows whose digest is the golden one."""
    import numpy as np
    from paper_1801_05857_b200.explore import Explorer
    e = big()[name]
    net = gx.load_network(_gen(name, tmp_path))
    ex = Explorer(net, ExploreConfig(table=TableConfig(capacity_words=_cap(e["states"], 4), num_hash_functions=16),
                                     state_digest=False), status=False)
    try:
        ex.run()
        rows = ex.table.sorted_vectors(ex.scheme.vector_length).astype(np.uint64)
    finally:
        ex.close()
    assert len(rows) == e["states"]
    key = np.zeros(len(rows), dtype=object) if rows.shape[1] > 2 else None
    if rows.shape[1] <= 2:
        k = rows[:, 0] << np.uint64(32) if rows.shape[1] == 2 else rows[:, 0]
        if rows.shape[1] == 2:
            k = k | rows[:, 1]
        assert (np.diff(k.astype(np.uint64)) > 0).all()
    else:
        order = np.lexsort(rows.T[::-1])
        assert (order == np.arange(len(rows))).all()
    assert list(statevec.state_digest(rows.astype(np.uint32))) == e["digest"]
    del key
