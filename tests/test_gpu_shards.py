"""The fused hash-owner sharded engine (gx_shard.cu, distributed.py
FusedShard) with all shards in one process on one GPU: the level kernel
routes successors owned by other shards into their inboxes (the code path
that stores over NVLink on a multi-GPU box), so sharded results must equal
the reference's for every shard count.  GPU only."""
import pytest

from conftest import golden_models, model_path
from oracle import oracle as O

pytestmark = pytest.mark.gpu

gx = pytest.importorskip("paper_1801_05857_b200")
from paper_1801_05857_b200 import distributed as D  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402

MODELS = golden_models()
NAMES = ["fig1", "ring6", "ring8", "gas6", "gas7", "phil5", "sinks8", "sinks10", "counter8", "wide33",
         "collide"]


def _cfg(bw=32, cap=1 << 22, **kw):
    return ExploreConfig(table=TableConfig(bucket_words=bw, capacity_words=cap), detect_deadlocks=True,
                         **kw)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", [n for n in NAMES if n in MODELS])
def test_sharded_matches_reference(name, world):
    g = MODELS[name]["bfs"]
    net = gx.load_network(model_path(name))
    rep = D.explore_local_shards(net, _cfg(), world)
    assert (rep.states, rep.transitions, rep.deadlocks_total, rep.outcome) == \
        (g["states"], g["transitions"], g["deadlocks_total"], "COMPLETE"), (name, world)
    assert [list(s) for s in rep.deadlocks] == g["deadlocks"][:100]
    assert rep.expanded == rep.states
    single = gx.explore(net, _cfg())
    assert rep.iterations == single.iterations


@pytest.mark.parametrize("bw", [4, 8, 16, 32])
@pytest.mark.parametrize("cache", [1, 4096])
def test_sharded_token_ring_closed_form(bw, cache, tmp_path):
    from paper_1801_05857_b200.bench import gen_token_ring
    n = 12
    _, p = gen_token_ring(n, tmp_path / "ring")
    net = gx.load_network(p)
    rep = D.explore_local_shards(net, _cfg(bw=bw, cap=1 << 24, cache_slots=cache), 4)
    assert rep.states == 2 * n * 3 ** (n - 1)
    assert rep.transitions == 4 * n * n * 3 ** (n - 2)
    assert rep.iterations == 6 * n - 4 + 1


def test_sharded_iteration_cap_and_table_full():
    net = gx.load_network(model_path("ring8"))
    single = gx.explore(net, _cfg(max_iterations=5))
    rep = D.explore_local_shards(net, _cfg(max_iterations=5), 4)
    assert (rep.outcome, rep.iterations, rep.states, rep.transitions) == \
        (single.outcome, single.iterations, single.states, single.transitions) == \
        ("ITERATION_CAP", 5, single.states, single.transitions)
    # a table far too small for the state space: every shard fills
    rep = D.explore_local_shards(net, _cfg(bw=4, cap=4 * 64), 2)
    assert rep.outcome == "TABLE_FULL"
    assert 0 < rep.states < MODELS["ring8"]["bfs"]["states"]


def test_sharded_generated_models(tmp_path):
    from paper_1801_05857_b200.bench import gen_gas_station, gen_peterson
    for gen, n in ((gen_peterson, 4), (gen_gas_station, 8)):
        _, p = gen(n, tmp_path / f"m{n}")
        want = O.Net.from_file(p).bfs()
        rep = D.explore_local_shards(gx.load_network(p), _cfg(cap=1 << 24), 3)
        assert (rep.states, rep.transitions, rep.iterations - 1, rep.deadlocks_total) == \
            (want["states"], want["transitions"], want["levels"], want["deadlocks"])


@pytest.mark.parametrize("bw", [4, 8, 32])
@pytest.mark.parametrize("world", [3, 4])
def test_sharded_contention(bw, world, tmp_path):
    """Token ring N=13 split over shards whose tables run at load ~0.7 with
    K=32: lost CASes, staged rehash rounds and inbox routing together; the
    exploration-only (no status array) tables are used as in the 150 GB
    bench configuration."""
    from paper_1801_05857_b200.bench import gen_token_ring
    from paper_1801_05857_b200.hashtable import slots_per_bucket
    n = 13
    _, p = gen_token_ring(n, tmp_path / "ring")
    net = gx.load_network(p)
    states = 2 * n * 3 ** (n - 1)
    spb = slots_per_bucket(bw, 2, "half" if bw == 32 else "plain")
    cap = (int(states / world / 0.7 / spb) + 256) * bw
    cfg = ExploreConfig(table=TableConfig(bucket_words=bw, num_hash_functions=32, capacity_words=cap),
                        detect_deadlocks=True)
    ex = D.LocalShardExplorer(net, cfg, world, inbox_capacity=states // 2, frontier_capacity=states // 4,
                              status=False)
    try:
        for _ in range(2):
            rep = ex.run()
            assert (rep.states, rep.transitions, rep.iterations, rep.outcome) == \
                (states, 4 * n * n * 3 ** (n - 2), 6 * n - 4 + 1, "COMPLETE")
    finally:
        ex.close()


def test_peterson6_single_table_equals_shards(tmp_path):
    """configs[2] (a peterson7-class model: Peterson's filter lock, 6
    processes, ~10^8 states) is beyond the CPU oracle, so two independent
    device engines pin each other: the single-table staged level kernel
    and the hash-owner sharded engine (routing + absorb) must agree on
    states, transitions, levels and deadlocks.  Peterson N <= 5 is pinned
    against the oracle in test_generated_models_match_oracle."""
    from paper_1801_05857_b200.bench import gen_peterson
    _, p = gen_peterson(6, tmp_path / "p6")
    net = gx.load_network(p)
    cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 31, num_hash_functions=16),
                        detect_deadlocks=True)
    one = gx.explore(net, cfg)
    cfg3 = ExploreConfig(table=TableConfig(capacity_words=(1 << 31) // 3, num_hash_functions=16),
                         detect_deadlocks=True)
    three = D.explore_local_shards(net, cfg3, 3)
    assert one.outcome == three.outcome == "COMPLETE"
    assert (one.states, one.transitions, one.iterations, one.deadlocks_total) == \
        (three.states, three.transitions, three.iterations, three.deadlocks_total)
    assert one.states > 10 ** 8


def test_owner_function_matches_restatement():
    """gx_owner_of (the device's owner_of_mix(key_mix(key))) equals the
    Python restatement the gloo driver tests use, for 1-4 word keys and
    1..16 ranks."""
    import numpy as np
    from test_distributed import owner_of
    from paper_1801_05857_b200.hashtable import StateTable
    rng = np.random.default_rng(3)
    for v in (1, 2, 3, 4):
        t = StateTable(TableConfig(capacity_words=1 << 12), v)
        try:
            keys = rng.integers(0, 1 << 32, size=(500, v), dtype=np.uint64).astype(np.uint32)
            for ranks in (1, 2, 3, 8, 16):
                import ctypes as C
                from paper_1801_05857_b200._lib import check, lib, ptr
                out = np.zeros(len(keys), np.int32)
                check(lib().gx_owner_of(t.handle, ptr(keys), len(keys), ranks, ptr(out, C.c_int32)))
                assert out.tolist() == [owner_of(k, ranks) for k in keys], (v, ranks)
        finally:
            t.close()
