"""Multi-shard and multi-process device paths on one GPU: the partitioned
dedup mode (gx_part.cuh) against the reference digests, including chunked
levels with inbox-overflow rollback; the hash-partitioned FINDORPUT
benchmark (configs[1] at N GPUs); two processes sharing cuda:0 through the
fused driver's CUDA-IPC inboxes (gloo counters); the NCCL all_to_all
driver (DeviceShard / explore_sharded) at world size 1, and its owner
binning at 3 ranks.  GPU only."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, golden_models, model_path

pytestmark = pytest.mark.gpu

gx = pytest.importorskip("paper_1801_05857_b200")
from paper_1801_05857_b200 import distributed as D  # noqa: E402
from paper_1801_05857_b200 import statevec  # noqa: E402
from paper_1801_05857_b200.explore import ExploreConfig  # noqa: E402
from paper_1801_05857_b200.hashtable import TableConfig  # noqa: E402

MODELS = golden_models()
REF = json.loads((GOLDEN / "ref_digests.json").read_text())


def _inband(net):
    sc = statevec.make_scheme(net)
    v = statevec.device_vlen(sc)
    return v in (1, 2, 4) and statevec.mark_bit(sc, v) is not None


@pytest.mark.parametrize("world", [1, 2, 3])
def test_dedup_mode_matches_reference(world):
    for name in sorted(REF):
        net = gx.load_network(model_path(name))
        if not _inband(net):
            continue
        cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 20), detect_deadlocks=True, dedup=True)
        rep = D.explore_local_shards(net, cfg, world)
        b = MODELS[name]["bfs"]
        assert list(rep.digest) == REF[name], (name, world)
        assert (rep.states, rep.transitions, rep.deadlocks_total, rep.outcome) == \
            (b["states"], b["transitions"], b["deadlocks_total"], "COMPLETE"), (name, world)
        assert [list(s) for s in rep.deadlocks] == b["deadlocks"][:100], name


@pytest.mark.parametrize("world", [1, 3])
def test_dedup_mode_small_inboxes(world, tmp_path):
    """Inboxes far smaller than a level: many chunks per level, first
    chunks sized from the network bound, sub-partitions, and overflowing
    chunks rolled back and re-run; the set is the closed-form one."""
    from oracle import oracle as O
    from paper_1801_05857_b200.bench import gen_token_ring
    n = 12
    net = gx.load_network(gen_token_ring(n, tmp_path / "r")[1])
    cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 24), detect_deadlocks=True, dedup=True,
                        dedup_set_log2=10)
    rep = D.explore_local_shards(net, cfg, world, inbox_capacity=1 << 16, frontier_capacity=1 << 20)
    assert (rep.states, rep.transitions, rep.iterations) == (2 * n * 3 ** (n - 1), 4 * n * n * 3 ** (n - 2),
                                                             6 * n - 4 + 1)
    assert rep.digest == O.ring_digest(n)
    assert rep.probes < 0.8 * rep.transitions  # even chunks of ~5e3 states filter duplicates


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("d", [1, 10])
def test_sharded_hash_bench(world, d):
    """configs[1] over shards: every key inserted exactly once into its
    owner's table however the sequence is split and routed."""
    net = gx.load_network(model_path("ring10"))  # any 1-word in-band geometry
    total = 1 << 22
    cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 24))
    ex = D.LocalShardExplorer(net, cfg, world, inbox_capacity=total, frontier_capacity=1 << 16)
    try:
        for _ in range(2):
            row = D.hash_bench_shards(ex.shards, lambda: None, lambda a: a, lambda a: a, total, d)
            assert (row["inserted"], row["found"], row["table_full"]) == (total // d, total - total // d, False)
            assert row["ms"] > 0
    finally:
        ex.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, names, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    out = []
    try:
        for name in names:
            net = gx.load_network(model_path(name))
            cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 20), detect_deadlocks=True)
            sh = D.FusedShard(net, cfg, rank, world, inbox_capacity=1 << 20, frontier_capacity=1 << 20)
            D.connect_fused([sh], dist)
            r = D.explore_fused([sh], dist, torch, True, device=torch.device("cpu"))
            sh.close()
            out.append((name, r.states, r.transitions, r.deadlocks_total, r.iterations, list(r.digest),
                        [list(x) for x in r.deadlocks]))
    except Exception as err:  # noqa: BLE001 - surfaced to the parent
        q.put(repr(err))
        raise
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_fused_two_processes_cuda_ipc():
    """Two processes on cuda:0: each maps the other's inbox through CUDA
    IPC and the level kernel stores routed successors into it (the
    multi-GPU data path); counters reduced over gloo."""
    import torch.multiprocessing as mp
    names = ["fig1", "ring8", "gas6", "phil5", "sinks8"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, names, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    for name, states, trans, dl, iters, dig, dls in res:
        b = MODELS[name]["bfs"]
        assert (states, trans, dl) == (b["states"], b["transitions"], b["deadlocks_total"]), name
        assert dig == REF[name] and dls == b["deadlocks"][:100], name
    assert all(p.exitcode == 0 for p in procs)


def _nccl_worker(port, names, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    out = []
    try:
        for name in names:
            net = gx.load_network(model_path(name))
            cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 20), detect_deadlocks=True)
            be = D.DeviceShard(net, cfg, 1, torch, capacity=1 << 20)
            sc = statevec.make_scheme(net)
            init = np.asarray(statevec.pack(sc, net.initial), np.uint32)
            r = D.explore_sharded(be, dist, torch, sc, init, True, device=torch.device("cuda", 0))
            be.close()
            out.append((name, r.states, r.transitions, r.deadlocks_total, r.iterations,
                        [list(x) for x in r.deadlocks]))
        # owner binning of gx_expand_route at 3 ranks against gx_owner_of
        net = gx.load_network(model_path("ring8"))
        be = D.DeviceShard(net, ExploreConfig(table=TableConfig(capacity_words=1 << 20)), 3, torch,
                           capacity=1 << 16)
        sc = statevec.make_scheme(net)
        init = np.asarray(statevec.pack(sc, net.initial), np.uint32)
        be.front[0] = torch.from_numpy(init.astype(np.int32))
        counts, tr, dl = be.expand_route(1, True)
        n = int(counts.sum().item())
        sent = be.send[:n].cpu().numpy().astype(np.uint32)
        owners = be.owner(sent)
        c = counts.cpu().numpy()
        bounds = np.concatenate([[0], np.cumsum(c)])
        ok = all((owners[bounds[r]:bounds[r + 1]] == r).all() for r in range(3))
        out.append(("binning", n, int(tr), bool(ok)))
        be.close()
    except Exception as err:  # noqa: BLE001
        q.put(repr(err))
        raise
    q.put(out)
    dist.destroy_process_group()


def test_nccl_all_to_all_driver_world1():
    """The collective driver (expand -> bin by owner -> NCCL all_to_all ->
    insert) on the device at world size 1, against the reference; its
    owner binning at 3 ranks."""
    import torch.multiprocessing as mp
    names = ["fig1", "ring8", "gas6", "phil5", "sinks10"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), names, q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert not isinstance(res, str), res
    for row in res[:-1]:
        name, states, trans, dl, iters, dls = row
        b = MODELS[name]["bfs"]
        assert (states, trans, dl) == (b["states"], b["transitions"], b["deadlocks_total"]), name
        assert dls == b["deadlocks"][:100], name
    assert res[-1][0] == "binning" and res[-1][3] and res[-1][1] > 0


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_pipelined_mode_matches_reference(world):
    """Fused levels with double-buffered inboxes: chunk c's launch routes
    into one half and absorbs chunk c - 1's keys from the other."""
    for name in sorted(REF):
        net = gx.load_network(model_path(name))
        if not _inband(net):
            continue
        cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 20), detect_deadlocks=True, pipeline=True)
        rep = D.explore_local_shards(net, cfg, world)
        b = MODELS[name]["bfs"]
        assert list(rep.digest) == REF[name], (name, world)
        assert (rep.states, rep.transitions, rep.deadlocks_total, rep.outcome) == \
            (b["states"], b["transitions"], b["deadlocks_total"], "COMPLETE"), (name, world)
        assert [list(s) for s in rep.deadlocks] == b["deadlocks"][:100], name


@pytest.mark.parametrize("world", [2, 3])
def test_pipelined_mode_many_chunks(world, tmp_path):
    """Small inboxes: many chunks per level, every half reused many times."""
    from oracle import oracle as O
    from paper_1801_05857_b200.bench import gen_token_ring
    n = 12
    net = gx.load_network(gen_token_ring(n, tmp_path / "r")[1])
    cfg = ExploreConfig(table=TableConfig(capacity_words=1 << 24), detect_deadlocks=True, pipeline=True)
    rep = D.explore_local_shards(net, cfg, world, inbox_capacity=1 << 17, frontier_capacity=1 << 20)
    assert (rep.states, rep.transitions, rep.iterations) == (2 * n * 3 ** (n - 1), 4 * n * n * 3 ** (n - 2),
                                                             6 * n - 4 + 1)
    assert rep.digest == O.ring_digest(n)
