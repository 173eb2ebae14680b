"""The reachable-set digest (include/gx.h gx_table_digest) on CPU: the
oracle's digest equals the one of the reference's own state sets
(tests/golden/ref_digests.json, made by make_reference_digests.py from
ltsmc.oracle.sequential_bfs), the numpy restatement in statevec equals the
C one, and the closed-form token-ring enumeration equals an exploration."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden_models, model_path
from oracle import oracle as O
from paper_1801_05857_b200 import statevec

REF = json.loads((GOLDEN / "ref_digests.json").read_text())


def big():
    return json.loads((GOLDEN / "digests.json").read_text())


@pytest.mark.parametrize("name", sorted(REF))
def test_oracle_digest_equals_reference_state_set(name):
    net = O.Net.from_file(model_path(name))
    r = O.explore(net, capacity_words=1 << 22)
    assert list(r.table.digest()) == REF[name]
    _, _, words = r.table.occupied()
    assert list(statevec.state_digest(words)) == REF[name]


def test_state_hash_restatements_agree():
    rng = np.random.default_rng(3)
    for v in (1, 2, 3, 4, 7, 16):
        w = rng.integers(0, 1 << 32, size=(50, v), dtype=np.uint64).astype(np.uint32)
        hs = statevec.state_hashes(w)
        assert [int(h) for h in hs] == [O.state_hash(row) for row in w]


def test_digest_is_order_independent_and_set_sensitive():
    rng = np.random.default_rng(4)
    w = rng.integers(0, 1 << 32, size=(1000, 2), dtype=np.uint64).astype(np.uint32)
    d = statevec.state_digest(w)
    assert statevec.state_digest(w[::-1]) == d
    w2 = w.copy()
    w2[17, 1] ^= 1  # one state traded for another: same count, different digest
    d2 = statevec.state_digest(w2)
    assert d2[0] == d[0] and d2[1:] != d[1:]
    assert statevec.state_digest(np.zeros((0, 2), np.uint32)) == (0, 0, 0)


@pytest.mark.parametrize("n", [2, 3, 4, 6, 9, 10, 11, 12])
def test_ring_enumeration_equals_exploration(n, tmp_path):
    from paper_1801_05857_b200.bench import gen_token_ring
    p = gen_token_ring(n, tmp_path / "r")[1]
    r = O.explore(O.Net.from_file(p), capacity_words=1 << 25, workers=4)
    assert r.table.digest() == O.ring_digest(n)
    if f"ring{n}" in REF:
        assert list(O.ring_digest(n)) == REF[f"ring{n}"]


def test_big_goldens_are_consistent():
    """digests.json: closed forms for the rings; explored and enumerated
    ring digests agree (the generator asserts it; re-checked here for N=11)."""
    for n in range(11, 21):
        e = big()[f"ring{n}"]
        assert e["states"] == 2 * n * 3 ** (n - 1) == e["digest"][0]
        assert e["transitions"] == 4 * n * n * 3 ** (n - 2)
    assert list(O.ring_digest(11)) == big()["ring11"]["digest"]
    for name in ("peterson3", "gas9", "phil8"):
        assert big()[name]["digest"][0] == big()[name]["states"]


@pytest.mark.parametrize("name", ["peterson3", "peterson4", "gas9", "phil8"])
def test_big_goldens_reproduce(name, tmp_path):
    from paper_1801_05857_b200.bench import gen_gas_station, gen_peterson, gen_philosophers
    kind = name.rstrip("0123456789")
    gen = {"peterson": gen_peterson, "gas": gen_gas_station, "phil": gen_philosophers}[kind]
    p = gen(int(name[len(kind):]), tmp_path / name)[1]
    r = O.explore(O.Net.from_file(p), capacity_words=1 << 25, workers=4, detect_deadlocks=True,
                  num_hash_functions=16)
    e = big()[name]
    assert (r.states, r.transitions, r.iterations, r.deadlocks_total) == \
        (e["states"], e["transitions"], e["iterations"], e["deadlocks_total"])
    assert list(r.table.digest()) == e["digest"]


def test_reference_digests_cover_golden_models():
    models = golden_models()
    assert set(REF) == {n for n in models if "error" not in models[n]}
