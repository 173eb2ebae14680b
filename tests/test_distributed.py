"""The hash-owner sharded driver (paper_1801_05857_b200/distributed.py) on
CPU: world_size 2 over gloo, with the per-rank compute supplied by an
oracle-backed stand-in (test infrastructure) instead of libgx.  Checks
that routing, exchange, termination and the reductions reproduce the
single-process results exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, golden_models, model_path

MASK = (1 << 64) - 1


def key_mix(words) -> int:
    """Python restatement of gx_device.cuh key_mix (pinned against the
    device in test_gpu_shards.py::test_owner_function_matches_restatement)."""
    x = 0x9E3779B9
    for w in words:
        x = ((x ^ int(w)) * 0x85EBCA77) & 0xFFFFFFFF
        x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    return x ^ (x >> 16)


def owner_of(words, ranks: int) -> int:
    """gx_device.cuh owner_of_mix(key_mix(key), ranks)."""
    return (key_mix(words) * ranks) >> 32


class OracleShard:
    """CPU stand-in for DeviceShard built on the oracle (tests only)."""

    def __init__(self, path, table_kw, world, cap=1 << 16):
        from oracle import oracle as O
        from paper_1801_05857_b200 import load_network, statevec
        self.O = O
        self.net = O.Net.from_file(path)
        self.scheme = statevec.make_scheme(load_network(path))
        self.vlen = self.net.vlen
        self.table_kw = table_kw
        self.world = world
        self.cap = cap
        self.front = np.zeros((0, self.vlen), np.uint32)
        z = lambda: torch.zeros((cap, self.vlen), dtype=torch.int32)
        self.send, self.recv = z(), z()
        self.salt = O.hash_constants(table_kw.get("seed", 42), 1)[1]
        self._dl = []

    def reset(self):
        self.table = self.O.Table(vector_length=self.vlen, **self.table_kw)

    def owner(self, packed):
        arr = np.asarray(packed, np.uint32).reshape(-1, self.vlen)
        return np.array([owner_of(r, self.world) for r in arr])

    def seed_frontier(self, packed):
        code, _ = self.table.find_or_insert(packed)
        if code == 2:
            return -1
        self.front = packed.reshape(1, -1).astype(np.uint32)
        return 1

    def expand_route(self, nfront, detect):
        succ, trans, dl = [], 0, 0
        self._dl = []
        for row in self.front[:nfront]:
            s = self.net.unpack(row)
            out, c = self.net.expand(s)
            trans += c
            if not out:
                dl += 1
                self._dl.append(row.copy())
            succ += [self.net.pack(t) for _, t in out]
        arr = np.array(succ, np.uint32).reshape(-1, self.vlen)
        own = self.owner(arr) if len(arr) else np.zeros(0, np.int64)
        order = np.argsort(own, kind="stable")
        arr = arr[order]
        counts = np.bincount(own, minlength=self.world)
        self.send[: len(arr)] = torch.from_numpy(arr.astype(np.int32))
        return torch.tensor(counts, dtype=torch.int64), trans, dl

    def deadlock_vectors(self):
        return np.array(self._dl, np.uint32).reshape(-1, self.vlen)

    def insert_append(self, nrecv):
        keys = self.recv[:nrecv].numpy().astype(np.uint32)
        codes, _ = self.table.find_or_insert_batch(keys)
        self.front = keys[codes == 1]
        return int((codes == 1).sum()), bool((codes == 2).any())

    def states(self):
        return self.table.occupancy()[0]


def _worker(rank, world, port, jobs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_05857_b200.distributed import explore_sharded
    from paper_1801_05857_b200 import statevec
    out = []
    for name, table_kw, max_it in jobs:
        b = OracleShard(model_path(name), table_kw, world)
        init = np.asarray(statevec.pack(b.scheme, b.net.initial), np.uint32)
        r = explore_sharded(b, dist, torch, b.scheme, init, True, max_iterations=max_it)
        out.append((name, r.states, r.transitions, r.iterations, r.deadlocks_total,
                    tuple(map(tuple, r.deadlocks)), r.outcome, r.expanded))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_sharded(jobs, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, jobs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_sharded_matches_single_process():
    from oracle import oracle as O
    names = ["fig1", "ring6", "gas5", "phil4", "sinks8", "counter8", "sparse4", "collide", "rand3"]
    jobs = [(n, {"capacity_words": 1 << 16}, None) for n in names]
    res = run_sharded(jobs)
    models = golden_models()
    for (name, states, trans, iters, dl_total, dls, outcome, expanded) in res:
        ref = O.explore(O.Net.from_file(model_path(name)), capacity_words=1 << 16,
                        detect_deadlocks=True)
        assert (states, trans, iters, dl_total, outcome, expanded) == \
            (ref.states, ref.transitions, ref.iterations, ref.deadlocks_total, ref.outcome,
             ref.expanded), name
        b = models[name]["bfs"]
        assert sorted(map(list, dls)) == sorted(b["deadlocks"])[:100], name


def test_sharded_iteration_cap_and_table_full():
    jobs = [("ring5", {"capacity_words": 1 << 14}, 3),
            ("ring6", {"bucket_words": 4, "capacity_words": 4 * 64}, None)]
    res = run_sharded(jobs)
    from oracle import oracle as O
    cap = O.explore(O.Net.from_file(model_path("ring5")), capacity_words=1 << 14, max_iterations=3)
    name, states, trans, iters, _, _, outcome, _ = res[0]
    assert (states, trans, iters, outcome) == (cap.states, cap.transitions, 3, "ITERATION_CAP")
    name, states, _, _, _, _, outcome, _ = res[1]
    assert outcome == "TABLE_FULL" and 0 < states < 2916


# ------------------------------------------------ fused (peer-routed) driver

class OracleFusedShard:
    """CPU stand-in for FusedShard (tests only).  expand_range() probes the
    locally owned successors of a frontier chunk at once and stages the
    others per owner, as k_level_routed does; the P2P inbox stores are
    emulated by a gloo all_to_all inside absorb_chunk() (the device writes
    them during the expansion).  chunk_states is small on purpose, so the
    driver's chunked levels are exercised."""

    def __init__(self, path, table_kw, world, rank, chunk_states=7):
        self.base = OracleShard(path, table_kw, world)
        self.rank, self.world = rank, world
        self.vlen = self.base.vlen
        self.chunk_states = chunk_states

    def begin(self, detect):
        from paper_1801_05857_b200 import statevec
        b = self.base
        b.reset()
        self.detect = detect
        self.trans = self.dl_total = self.expanded = 0
        self.kept = []
        self.states = 0
        self.front = np.zeros((0, self.vlen), np.uint32)
        self._level_reset()
        init = np.asarray(statevec.pack(b.scheme, b.net.initial), np.uint32)
        if int(b.owner(init)[0]) == self.rank:
            code, _ = b.table.find_or_insert(init)
            if code == 2:
                return True
            self.front = init.reshape(1, -1)
            self.states = 1
        return False

    def _level_reset(self):
        self.next, self.full, self.outgoing = [], False, []

    def frontier(self):
        return len(self.front)

    def expand_range(self, begin, count):
        b = self.base
        rows = self.front[begin:begin + count]
        self.expanded += len(rows)
        succ = []
        for row in rows:
            out, c = b.net.expand(b.net.unpack(row))
            self.trans += c
            if not out and self.detect:
                self.dl_total += 1
                self.kept.append(b.net.unpack(row))
            succ += [b.net.pack(t) for _, t in out]
        arr = np.array(succ, np.uint32).reshape(-1, self.vlen)
        own = b.owner(arr) if len(arr) else np.zeros(0, np.int64)
        local = arr[own == self.rank]
        if len(local):
            codes, _ = b.table.find_or_insert_batch(local)
            self.next.append(local[codes == 1])
            self.full |= bool((codes == 2).any())
        self.outgoing = [arr[own == r] for r in range(self.world)]

    def absorb_chunk(self):
        b = self.base
        counts = torch.tensor([len(x) if r != self.rank else 0 for r, x in enumerate(self.outgoing)],
                              dtype=torch.int64)
        rc = torch.empty_like(counts)
        dist.all_to_all_single(rc, counts)
        send = torch.from_numpy(np.concatenate(
            [x if r != self.rank else np.zeros((0, self.vlen), np.uint32)
             for r, x in enumerate(self.outgoing)]).astype(np.int32).reshape(-1, self.vlen))
        recv = torch.empty((int(rc.sum()), self.vlen), dtype=torch.int32)
        dist.all_to_all_single(recv, send, output_split_sizes=rc.tolist(),
                               input_split_sizes=counts.tolist())
        keys = recv.numpy().astype(np.uint32)
        if len(keys):
            codes, _ = b.table.find_or_insert_batch(keys)
            self.next.append(keys[codes == 1])
            self.full |= bool((codes == 2).any())
        self.outgoing = [np.zeros((0, self.vlen), np.uint32)] * self.world

    def end_level(self):
        claims = len(self.front)
        self.front = np.concatenate(self.next).reshape(-1, self.vlen) if self.next else \
            np.zeros((0, self.vlen), np.uint32)
        self.states += len(self.front)
        st = np.zeros(8, np.uint64)
        st[0], st[1], st[2], st[3], st[4] = claims, len(self.front), self.trans, self.dl_total, \
            int(self.full)
        self._level_reset()
        return st

    def digest(self):
        return self.base.table.digest(self.vlen)

    def finish(self):
        class Rep:
            pass
        r = Rep()
        r.states, r.transitions, r.expanded = self.states, self.trans, self.expanded
        r.deadlocks_total, r.probes, r.level_ms = self.dl_total, 0, 0.0
        return r, sorted(self.kept)[:100]


def _fused_worker(rank, world, port, jobs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_05857_b200.distributed import explore_fused
    out = []
    try:
        for name, table_kw, max_it in jobs:
            s = OracleFusedShard(model_path(name), table_kw, world, rank)
            r = explore_fused(s, dist, torch, True, max_iterations=max_it, device=torch.device("cpu"))
            out.append((name, r.states, r.transitions, r.iterations, r.deadlocks_total,
                        tuple(map(tuple, r.deadlocks)), r.outcome, r.expanded, r.digest))
    except Exception as err:  # noqa: BLE001 - surfaced to the parent
        q.put(repr(err))
        raise
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_fused_driver_matches_single_process():
    """explore_fused's barrier / reduction / termination logic, world 2
    and 3 over gloo, against the single-process reference engine."""
    from oracle import oracle as O
    names = ["fig1", "ring6", "gas5", "phil4", "sinks8", "collide"]
    jobs = [(n, {"capacity_words": 1 << 16}, None) for n in names] + \
        [("ring5", {"capacity_words": 1 << 14}, 3)]
    models = golden_models()
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_fused_worker, args=(r, world, port, jobs, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = q.get(timeout=600)
        assert not isinstance(res, str), res
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        for (name, states, trans, iters, dl_total, dls, outcome, expanded, dig), job in zip(res, jobs):
            ref = O.explore(O.Net.from_file(model_path(name)), capacity_words=job[1]["capacity_words"],
                            detect_deadlocks=True, max_iterations=job[2])
            assert (states, trans, iters, dl_total, outcome, expanded) == \
                (ref.states, ref.transitions, ref.iterations, ref.deadlocks_total, ref.outcome,
                 ref.expanded), (name, world)
            if outcome == "COMPLETE":
                assert dig == ref.table.digest(), (name, world)
            if job[2] is None:
                assert sorted(map(list, dls)) == sorted(models[name]["bfs"]["deadlocks"])[:100], name


# ------------------------------------- partitioned (dedup) driver protocol

class OraclePartShard(OracleFusedShard):
    """CPU stand-in for a FusedShard in the partitioned dedup mode: the
    expansion routes EVERY successor (own ones too) and touches no table;
    chunk_status flags an inbox overflow when a chunk sends more than
    inbox/world keys to one owner (the device flags the receiver's
    reservation), and rollback discards the chunk; absorb_chunk exchanges,
    de-duplicates (the L2 set) and inserts.  Exercises ChunkPlanner and
    _level_partitioned, including repeated rollbacks, over gloo."""

    def __init__(self, path, table_kw, world, rank, inbox=48):
        super().__init__(path, table_kw, world, rank)
        from types import SimpleNamespace

        from paper_1801_05857_b200 import load_network
        self.dedup = True
        self.inbox_capacity = inbox
        self.set_slots = 64
        self.dnet = SimpleNamespace(net=load_network(path))
        self.rollbacks = 0
        self.nsubs = []

    def set_partitions(self, nsub):
        assert nsub & (nsub - 1) == 0
        self.nsubs.append(nsub)

    def expand_range(self, begin, count):
        b = self.base
        rows = self.front[begin:begin + count]
        self.c_exp, self.c_trans, self.c_dl, self.c_kept = len(rows), 0, 0, []
        succ = []
        for row in rows:
            out, c = b.net.expand(b.net.unpack(row))
            self.c_trans += c
            if not out and self.detect:
                self.c_dl += 1
                self.c_kept.append(b.net.unpack(row))
            succ += [b.net.pack(t) for _, t in out]
        arr = np.array(succ, np.uint32).reshape(-1, self.vlen)
        own = b.owner(arr) if len(arr) else np.zeros(0, np.int64)
        self.outgoing = [arr[own == r] for r in range(self.world)]
        self.c_ovf = int(any(len(x) > self.inbox_capacity // self.world for x in self.outgoing))
        self.c_routed = len(arr)

    def chunk_status(self):
        # cumulative counters as the device reports them (this chunk included)
        return np.array([self.c_ovf, getattr(self, "routed_total", 0) + self.c_routed,
                         self.expanded + self.c_exp], np.uint64)

    def rollback(self):
        self.rollbacks += 1
        self.outgoing = [np.zeros((0, self.vlen), np.uint32)] * self.world

    def absorb_chunk(self):
        b = self.base
        self.expanded += self.c_exp
        self.trans += self.c_trans
        self.dl_total += self.c_dl
        self.kept += self.c_kept
        self.routed_total = getattr(self, "routed_total", 0) + self.c_routed
        counts = torch.tensor([len(x) for x in self.outgoing], dtype=torch.int64)
        rc = torch.empty_like(counts)
        dist.all_to_all_single(rc, counts)
        send = torch.from_numpy(np.concatenate(self.outgoing).astype(np.int32).reshape(-1, self.vlen))
        recv = torch.empty((int(rc.sum()), self.vlen), dtype=torch.int32)
        dist.all_to_all_single(recv, send, output_split_sizes=rc.tolist(), input_split_sizes=counts.tolist())
        keys = recv.numpy().astype(np.uint32)
        if len(keys):
            keys = np.unique(keys, axis=0)  # the duplicate filter
            codes, _ = b.table.find_or_insert_batch(keys)
            self.next.append(keys[codes == 1])
            self.full |= bool((codes == 2).any())
        self.outgoing = [np.zeros((0, self.vlen), np.uint32)] * self.world

    def end_level(self):
        st = super().end_level()
        st[6] = getattr(self, "routed_total", 0)
        return st


def _part_worker(rank, world, port, jobs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_05857_b200.distributed import explore_fused
    out = []
    try:
        for name, table_kw in jobs:
            s = OraclePartShard(model_path(name), table_kw, world, rank)
            r = explore_fused(s, dist, torch, True, device=torch.device("cpu"))
            out.append((name, r.states, r.transitions, r.iterations, r.deadlocks_total, r.outcome,
                        r.digest, s.rollbacks, max(s.nsubs)))
    except Exception as err:  # noqa: BLE001 - surfaced to the parent
        q.put(repr(err))
        raise
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_driver_chunks_and_rollbacks():
    """_level_partitioned + ChunkPlanner over gloo (world 2): tiny inboxes
    force many chunks, overflowing chunks are rolled back and re-run, and
    the results equal the single-process reference engine's."""
    from oracle import oracle as O
    jobs = [("ring8", {"capacity_words": 1 << 18}), ("gas6", {"capacity_words": 1 << 18}),
            ("phil5", {"capacity_words": 1 << 16}), ("sinks8", {"capacity_words": 1 << 16})]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, 2, port, jobs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    rolled = 0
    for (name, states, trans, iters, dl, outcome, dig, rb, nsub), job in zip(res, jobs):
        ref = O.explore(O.Net.from_file(model_path(name)), capacity_words=job[1]["capacity_words"],
                        detect_deadlocks=True)
        assert (states, trans, iters, dl, outcome) == \
            (ref.states, ref.transitions, ref.iterations, ref.deadlocks_total, ref.outcome), name
        assert dig == ref.table.digest(), name
        rolled += rb
    assert rolled > 0  # the overflow path ran


def test_chunk_planner_sizes():
    from types import SimpleNamespace

    from paper_1801_05857_b200 import load_network
    from paper_1801_05857_b200.distributed import ChunkPlanner
    net = load_network(model_path("ring8"))
    sh = SimpleNamespace(world=2, inbox_capacity=1 << 20, set_slots=1 << 22, dnet=SimpleNamespace(net=net))
    p = ChunkPlanner([sh, sh])
    first = p.chunk()
    assert first == int(0.8 * (1 << 20) / p.ratio)
    p.observe(routed=5 * 1000, expanded=1000)        # 5 successors per state seen
    assert abs(p.ratio - (1.2 * 5 + 0.5)) < 1e-9 and p.chunk() > first
    p.overflowed()
    assert abs(p.ratio - 2 * (1.2 * 5 + 0.5)) < 1e-9
    assert p.nsub(10) == 1
    big = p.nsub(10 ** 9)
    assert big & (big - 1) == 0 and big == p.nsub_max == 64
