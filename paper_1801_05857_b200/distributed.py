"""Hash-owner sharded exploration across GPUs (one process per GPU).

Two drivers share the ownership rule and the level semantics:

* the fused one (`FusedShard`, `explore_fused`, `explore_local_shards`;
  gx_shard.cu): the level kernel routes successors owned by peers straight
  into their inboxes over NVLink (CUDA IPC peer mappings) while it probes
  its own, then every shard absorbs its inbox after a barrier -- the
  all-to-all is fused into successor generation;
* the collective one (`DeviceShard`, `explore_sharded`, below): expand,
  bin by owner, NCCL all_to_all of counts and payload, insert.

Every rank owns the states whose owner hash (a cheap 32-bit murmur-style
mix of the key words, independent of the table's fold and so decorrelated
from all bucket indices; gx_device.cuh `key_mix` / `owner_of_mix`) equals
its rank, holds that shard of the state table, and expands only its own
frontier.  One BFS level of the collective driver:

  1. expand + route   the local frontier's successors are generated on
                      the device and binned by owner (gx_expand_route)
  2. exchange         per-peer counts (all_to_all_single of W int64),
                      then the variable-size payload (all_to_all_single)
  3. insert           FINDORPUT of the received vectors into the local
                      shard; INSERTED ones form the next local frontier
                      (gx_insert_append)
  4. reduce           all_reduce of (claims, new, transitions, deadlocks,
                      table_full) decides termination for every rank

Rounds stay global BFS levels, so `iterations` = levels + 1 exactly as on
one GPU and in the reference (explore.py:234-268).  Transitions are
counted at the expanding rank; TABLE_FULL on any shard aborts all.

The reference's only parallelism is a bucket-range partition of one
shared table among CPU workers (explore.py:284-286); the exchange step
here replaces its shared memory.

The collective plumbing is torch.distributed (NCCL over NVLink on B200,
gloo in the CPU tests).  The per-rank compute is a `ShardBackend`; the
product backend is `DeviceShard` (libgx kernels on torch CUDA buffers).
Tests plug a CPU stand-in built on the oracle to exercise this driver
with world_size 2 over gloo.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


@dataclass
class ShardResult:
    states: int
    transitions: int
    deadlocks: tuple
    deadlocks_total: int
    expanded: int
    iterations: int
    outcome: str
    levels: int
    digest: tuple | None = None  # reachable-set digest over all ranks (gx_table_digest)
    routed: int = 0  # successors routed to another shard's inbox (all ranks)
    level_ms: float = 0.0  # CUDA-event time of the level kernels, max over ranks
    probes: int = 0  # FINDORPUTs issued (all ranks)


class DeviceShard:
    """Per-rank compute on the B200 through libgx (buffers are torch CUDA
    tensors so NCCL can move them without staging)."""

    def __init__(self, net, cfg, world: int, torch, capacity: int, stream=None):
        from . import statevec
        from .explore import DeviceNetwork
        from .hashtable import StateTable

        self.torch = torch
        self.world = world
        self.scheme = statevec.make_scheme(net)
        self.vlen = self.scheme.vector_length
        self.dnet = DeviceNetwork(net, self.scheme, stream)
        self.table = StateTable(cfg.table, self.vlen, mark=statevec.mark_bit(self.scheme),
                                stream=stream)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.cap = capacity
        mk = lambda: torch.zeros((capacity, self.vlen), dtype=torch.int32, device=dev)
        self.front, self.next, self.send, self.recv = mk(), mk(), mk(), mk()
        self.counts = torch.zeros(world, dtype=torch.int64, device=dev)
        self.offsets = torch.zeros(world, dtype=torch.int64, device=dev)
        init = np.asarray(statevec.pack(self.scheme, net.initial), np.uint32)
        self.init = init

    # -- backend protocol --------------------------------------------------
    def reset(self):
        self.table.clear()

    def owner(self, packed: np.ndarray) -> np.ndarray:
        from ._lib import check, lib, ptr
        arr = np.ascontiguousarray(packed, np.uint32).reshape(-1, self.vlen)
        out = np.zeros(arr.shape[0], np.int32)
        check(lib().gx_owner_of(self.table.handle, ptr(arr), arr.shape[0], self.world,
                                ptr(out, C.c_int32)))
        return out

    def seed_frontier(self, packed: np.ndarray) -> int:
        """Insert the initial state (if owned) and make it the frontier."""
        codes, _ = self.table.find_or_insert_batch(packed.reshape(1, -1))
        if int(codes[0]) == 2:
            return -1
        self.front[0] = self.torch.from_numpy(packed.astype(np.int32))
        return 1

    def expand_route(self, nfront: int, detect: bool):
        from ._lib import check, lib
        tr, dl = C.c_uint64(), C.c_uint64()
        check(lib().gx_expand_route(self.dnet.handle, self.table.handle, C.c_void_p(self.front.data_ptr()),
                                    nfront, self.world, C.c_void_p(self.send.data_ptr()), self.cap,
                                    C.c_void_p(self.counts.data_ptr()),
                                    C.c_void_p(self.offsets.data_ptr()), C.byref(tr), C.byref(dl),
                                    int(detect)))
        return self.counts.clone(), tr.value, dl.value

    def deadlock_vectors(self) -> np.ndarray:
        from ._lib import check, lib, ptr
        cnt = C.c_uint64()
        check(lib().gx_net_deadlocks(self.dnet.handle, None, 0, C.byref(cnt)))
        n = min(cnt.value, 1 << 16)
        out = np.zeros((max(n, 1), self.vlen), np.uint32)
        if n:
            check(lib().gx_net_deadlocks(self.dnet.handle, ptr(out), n, C.byref(cnt)))
        return out[:n]

    def insert_append(self, nrecv: int):
        from ._lib import check, lib
        nn, full = C.c_uint64(), C.c_int32()
        check(lib().gx_insert_append(self.table.handle, C.c_void_p(self.recv.data_ptr()), nrecv,
                                     C.c_void_p(self.next.data_ptr()), self.cap, C.byref(nn),
                                     C.byref(full)))
        self.front, self.next = self.next, self.front
        return nn.value, bool(full.value)

    def states(self) -> int:
        return self.table.occupancy()[0]

    def close(self):
        self.table.close()
        self.dnet.close()


GX_SH = dict(claims=0, new=1, transitions=2, deadlocks=3, table_full=4, overflow=5, routed=6,
             probes=7)
IPC_HANDLE_BYTES = 64
IPC_ZERO = bytes(IPC_HANDLE_BYTES)  # "same-process peer" in gx_shard_connect


class FusedShard:
    """One hash-owner shard on the fused level kernels (include/gx.h
    gx_shard_*): the level kernel stores successors owned by peers straight
    into their inboxes (P2P over NVLink, CUDA IPC mappings) and FINDORPUTs
    its own; after the level barrier each shard absorbs its inbox."""

    def __init__(self, net, cfg, rank: int, world: int, inbox_capacity: int = 0,
                 frontier_capacity: int = 0, stream=None, status: bool = True):
        from . import statevec
        from ._lib import check, lib
        from .explore import DeviceNetwork
        from .hashtable import StateTable

        from .explore import device_table_config
        self.rank, self.world = rank, world
        self.stream = stream
        self.scheme = statevec.make_scheme(net)
        self.vlen = statevec.device_vlen(self.scheme, cfg.pad_vlen3)
        self.dnet = DeviceNetwork(net, self.scheme, stream, self.vlen)
        self.table = StateTable(device_table_config(cfg.table, self.scheme, self.vlen), self.vlen,
                                mark=statevec.mark_bit(self.scheme, self.vlen), stream=stream,
                                status=status)
        slots = self.table.total_slots
        frontier_capacity = frontier_capacity or cfg.frontier_capacity
        if not frontier_capacity or not inbox_capacity:
            # standalone default (one shard per process and GPU): frontier and
            # inbox together take at most 40% of what this table left free
            sm, free, _tot = device_info()
            each = max(1 << 16, min(slots + 2, int(free * 0.2) // (4 * self.vlen)))
            frontier_capacity = frontier_capacity or each
            inbox_capacity = inbox_capacity or each
        self.frontier_capacity, self.inbox_capacity = frontier_capacity, inbox_capacity
        h = C.c_void_p()
        check(lib().gx_shard_create(self.dnet.handle, self.table.handle, rank, world, inbox_capacity,
                                    frontier_capacity, int(min(cfg.cache_slots, 1 << 30)),
                                    int(cfg.filter_log2), C.byref(h)))
        self._h = h
        # partitioned dedup levels (in-band tables with 1/2/4-word slots)
        self.dedup = bool(cfg.dedup) and self.vlen in (1, 2, 4) and self.table.mode == "mark"
        self.set_slots = 0
        if self.dedup:
            check(lib().gx_shard_set_mode(h, 1, int(cfg.dedup_set_log2)))
            self.set_slots = (1 << int(cfg.dedup_set_log2)) * (2 if self.vlen == 4 else 4)
        self.pipelined = bool(getattr(cfg, "pipeline", False)) and not self.dedup
        if self.pipelined:
            check(lib().gx_shard_set_pipeline(h, 1))
        self.init = np.zeros(self.vlen, np.uint32)
        packed = statevec.pack(self.scheme, net.initial)
        self.init[:len(packed)] = packed
        from .network import max_successors
        # frontier states per chunk so that no inbox can overflow even if every
        # successor of every sender's chunk went to one owner
        # (measured: sizing chunks for 16 instead of ring19's bound of 38
        # successors per state gains only 2%, profiles/README.md); a
        # pipelined shard routes into half of its peers' inboxes per chunk
        per_chunk = inbox_capacity // 2 if self.pipelined else inbox_capacity
        self.chunk_states = max(1, per_chunk // (world * max_successors(net)))

    @property
    def handle(self):
        return self._h

    def sync(self):
        """Wait for this shard's stream (its kernels and peer stores)."""
        from ._lib import check, lib
        check(lib().gx_sync(self.stream))

    def owner_of(self, packed: np.ndarray) -> int:
        from ._lib import check, lib, ptr
        arr = np.ascontiguousarray(packed, np.uint32).reshape(-1, self.vlen)
        out = np.zeros(arr.shape[0], np.int32)
        check(lib().gx_owner_of(self.table.handle, ptr(arr), arr.shape[0], self.world,
                                ptr(out, C.c_int32)))
        return int(out[0])

    def ipc_handle(self) -> bytes:
        from ._lib import check, lib, ptr
        buf = np.zeros(IPC_HANDLE_BYTES, np.uint8)
        check(lib().gx_shard_ipc_handle(self._h, ptr(buf, C.c_uint8)))
        return buf.tobytes()

    def connect(self, handles):
        from ._lib import check, lib, ptr
        buf = np.frombuffer(b"".join(handles), np.uint8).copy()
        check(lib().gx_shard_connect(self._h, ptr(buf, C.c_uint8)))

    def begin(self, detect: bool) -> bool:
        """Clear; insert the initial state if owned.  True if TABLE_FULL."""
        from ._lib import check, lib
        full = C.c_int32()
        owns = self.owner_of(self.init) == self.rank
        check(lib().gx_shard_begin(self._h, int(owns), int(detect), C.byref(full)))
        return bool(full.value)

    def expand(self):
        from ._lib import check, lib
        check(lib().gx_shard_expand(self._h))

    def frontier(self) -> int:
        from ._lib import check, lib
        n = C.c_uint64()
        check(lib().gx_shard_frontier(self._h, C.byref(n)))
        return n.value

    def expand_range(self, begin: int, count: int):
        from ._lib import check, lib
        check(lib().gx_shard_expand_range(self._h, begin, count))

    def absorb_chunk(self):
        from ._lib import check, lib
        check(lib().gx_shard_absorb_chunk(self._h))

    def bench_route(self, total: int, duplication: int, seed: int, first: int, count: int,
                    key_bits: int = 31):
        """Hash-partitioned FINDORPUT benchmark, this shard's positions
        [first, first + count) of the global sequence (gx_shard_bench_route)."""
        from ._lib import check, lib
        check(lib().gx_shard_bench_route(self._h, total, duplication, seed, key_bits, first, count))

    def bench_result(self):
        """(inserted, table_full, findorputs, routed, overflow), kernel ms"""
        from ._lib import check, lib, ptr
        out = np.zeros(5, np.uint64)
        ms = C.c_double()
        check(lib().gx_shard_bench_result(self._h, ptr(out, C.c_uint64), C.byref(ms)))
        return out, ms.value

    def set_partitions(self, nsub: int):
        from ._lib import check, lib
        check(lib().gx_shard_set_partitions(self._h, int(nsub)))

    def chunk_status(self) -> np.ndarray:
        """[inbox overflow flag, successors routed so far, states expanded so far]"""
        from ._lib import check, lib, ptr
        out = np.zeros(3, np.uint64)
        check(lib().gx_shard_chunk_status(self._h, ptr(out, C.c_uint64)))
        return out

    def rollback(self):
        from ._lib import check, lib
        check(lib().gx_shard_rollback(self._h))

    def end_level(self) -> np.ndarray:
        from ._lib import check, lib, ptr
        st = np.zeros(8, np.uint64)
        check(lib().gx_shard_end_level(self._h, ptr(st, C.c_uint64)))
        return st

    def absorb(self) -> np.ndarray:
        from ._lib import check, lib, ptr
        st = np.zeros(8, np.uint64)
        check(lib().gx_shard_absorb(self._h, ptr(st, C.c_uint64)))
        return st

    def digest(self) -> tuple:
        """This shard's part of the reachable-set digest (gx_table_digest)."""
        return self.table.digest(self.scheme.vector_length)

    def finish(self):
        from . import statevec
        from ._lib import Report, check, lib, ptr
        rep = Report()
        dl = np.zeros((100, self.vlen), np.uint32)
        check(lib().gx_shard_finish(self._h, C.byref(rep), ptr(dl)))
        sv = self.scheme.vector_length
        kept = [statevec.unpack(self.scheme, tuple(int(x) for x in dl[i, :sv]))
                for i in range(rep.deadlocks_kept)]
        return rep, kept

    def close(self):
        from ._lib import lib
        if getattr(self, "_h", None):
            lib().gx_shard_destroy(self._h)
            self._h = None
        self.table.close()
        self.dnet.close()


def device_info():
    from ._lib import lib
    sm, free, tot = C.c_int32(), C.c_uint64(), C.c_uint64()
    lib().gx_device_info(C.byref(sm), C.byref(free), C.byref(tot))
    return sm.value, free.value, tot.value


def connect_local(shards):
    from ._lib import check, lib
    arr = (C.c_void_p * len(shards))(*[s.handle.value for s in shards])
    check(lib().gx_shard_connect_local(arr, len(shards)))


def _run_levels(shards, barrier, reduce, detect: bool, max_iterations=None, reduce_max=None):
    """The level protocol shared by the in-process and multi-process
    drivers (explore.py:251-265 semantics).  A level is expanded in
    frontier chunks small enough that no inbox can overflow: for each chunk
    every shard expands, a barrier, every shard absorbs (and a barrier
    before the next chunk's peer stores); then the level's stats are
    reduced over all ranks."""
    reduce_max = reduce_max or (lambda a: a)
    full = reduce(np.array([sum(int(s.begin(detect)) for s in shards)], np.uint64))[0]
    chunk = min(s.chunk_states for s in shards)
    dedup = all(getattr(s, "dedup", False) for s in shards)
    planner = ChunkPlanner(shards) if dedup else None
    rounds = 0
    routed = 0
    outcome = "COMPLETE"
    if full:
        outcome = "TABLE_FULL"
    else:
        while True:
            widest = int(reduce_max(np.array([max(s.frontier() for s in shards)], np.uint64))[0])
            if dedup:
                _level_partitioned(shards, barrier, reduce, planner, widest)
            elif all(getattr(s, "pipelined", False) for s in shards):
                # chunk c's launch also absorbs chunk c - 1's inbox half
                chunks = max(1, -(-widest // chunk))
                for c in range(chunks):
                    for s in shards:
                        s.expand_range(c * chunk, chunk)
                    barrier()
                for s in shards:
                    s.absorb_chunk()
            else:
                chunks = max(1, -(-widest // chunk))
                for c in range(chunks):
                    for s in shards:
                        s.expand_range(c * chunk, chunk)
                    barrier()
                    for s in shards:
                        s.absorb_chunk()
                    if c + 1 < chunks:
                        barrier()
            st = np.zeros(8, np.uint64)
            for s in shards:
                st += s.end_level()
            st = reduce(st)
            routed = int(st[GX_SH["routed"]])
            rounds += 1
            if st[GX_SH["overflow"]]:
                raise RuntimeError("frontier capacity exceeded in sharded exploration; "
                                   "raise frontier_capacity")
            if st[GX_SH["table_full"]]:
                outcome = "TABLE_FULL"
                break
            if st[GX_SH["claims"]] == 0:
                break
            if max_iterations is not None and rounds >= max_iterations:
                outcome = "ITERATION_CAP"
                break
    tot = np.zeros(5, np.uint64)
    kept = []
    level_ms = 0.0
    for s in shards:
        rep, k = s.finish()
        tot += np.array([rep.states, rep.transitions, rep.expanded, rep.deadlocks_total, rep.probes],
                        np.uint64)
        level_ms += rep.level_ms
        kept.extend(k)
    return tot, sorted(kept)[:100], rounds, outcome, level_ms, routed


class ChunkPlanner:
    """Frontier chunk and sub-partition sizes of the partitioned levels.

    Every shard receives about (states expanded per shard) x (successors
    per state) keys per chunk; the chunk is sized so that this fills at
    most 80% of an inbox, from the largest successors-per-state ratio seen
    so far (initially the network's bound, network.max_successors).  The
    sub-partition count makes each sub-partition at most twice the dedup
    set's slots (set load <= 1/2 for >= 4x duplication; less duplication
    only costs redundant probes).  An overflowing chunk is rolled back and
    re-run at half the size, so the estimate never affects results."""

    def __init__(self, shards):
        from .network import max_successors
        s0 = shards[0]
        self.world = s0.world
        self.inbox = min(s.inbox_capacity for s in shards)
        self.set_slots = min(s.set_slots for s in shards)
        self.ratio = float(max_successors(s0.dnet.net))
        self.seen = 0.0
        self.routed = 0
        self.expanded = 0
        self.nsub_max = max(1, min(256, 128 // self.world))

    def chunk(self) -> int:
        return max(1, int(0.8 * self.inbox / max(self.ratio, 1e-9)))

    def nsub(self, n: int) -> int:
        keys = n * self.ratio
        want = max(1, int(-(-keys // (2 * self.set_slots))))
        p = 1
        while p < want and p < self.nsub_max:
            p *= 2
        return p

    def observe(self, routed: int, expanded: int):
        dr, de = routed - self.routed, expanded - self.expanded
        self.routed, self.expanded = routed, expanded
        if de > 0:
            self.seen = max(self.seen, dr / de)
            self.ratio = min(self.ratio, max(1.0, 1.2 * self.seen + 0.5))

    def overflowed(self):
        self.ratio *= 2.0


def _level_partitioned(shards, barrier, reduce, planner, widest: int):
    """One level of the partitioned dedup engine: frontier chunks of
    planner.chunk() states per shard; per chunk every shard expands and
    routes (gx_shard_expand_range), the overflow flags and counters are
    reduced (the barrier), then every shard filters + probes its
    sub-partitions (gx_shard_absorb_chunk)."""
    c = 0
    while c < widest:
        n = min(widest - c, planner.chunk())
        nsub = planner.nsub(n)
        for s in shards:
            s.set_partitions(nsub)
            s.expand_range(c, n)
        st = np.zeros(3, np.uint64)
        for s in shards:
            st += s.chunk_status()
        st = reduce(st)
        if st[0]:
            for s in shards:
                s.rollback()
            planner.overflowed()
            continue
        planner.observe(int(st[1]), int(st[2]))
        for s in shards:
            s.absorb_chunk()
        c += n
        if c < widest:
            barrier()


class LocalShardExplorer:
    """`world` hash-owner shards of one network in this process (one GPU),
    built once and explored any number of times (each run clears the
    tables).  On one GPU this keeps every shard's random probes inside the
    TLB reach (profiles/README.md: random access drops from 36 to 9 G/s
    once a table outgrows ~64 GiB); across GPUs it is the same protocol
    with peer inboxes over NVLink."""

    def __init__(self, net, cfg, world: int, inbox_capacity: int = 0, frontier_capacity: int = 0,
                 status: bool = True, stream=None):
        self.cfg = cfg
        self.shards = []
        frontier_capacity = frontier_capacity or cfg.frontier_capacity
        if not frontier_capacity or not inbox_capacity:
            f, i = local_buffer_sizes(net, cfg, world, status)
            frontier_capacity = frontier_capacity or f
            inbox_capacity = inbox_capacity or i
        try:
            for r in range(world):
                self.shards.append(FusedShard(net, cfg, r, world, inbox_capacity, frontier_capacity,
                                              stream=stream, status=status))
            connect_local(self.shards)
        except Exception:
            self.close()
            raise

    def run(self):
        import time

        from .explore import ExplorationReport

        t0 = time.perf_counter()
        tot, kept, rounds, outcome, level_ms, routed = _run_levels(self.shards, lambda: None, lambda a: a,
                                                                   self.cfg.detect_deadlocks,
                                                                   self.cfg.max_iterations)
        wall = time.perf_counter() - t0
        states = int(tot[0])
        return ExplorationReport(
            states=states, transitions=int(tot[1]), deadlocks=tuple(kept),
            deadlocks_total=int(tot[3]), expanded=int(tot[2]), iterations=rounds, wall_time=wall,
            throughput=states / wall if wall > 0 else 0.0, outcome=outcome, probes=int(tot[4]),
            level_ms=float(level_ms), routed=routed,
            digest=self.digest() if self.cfg.state_digest else None)

    def digest(self) -> tuple:
        """The reachable set's digest over all shards (include/gx.h
        gx_table_digest): equal to one table's for the same set."""
        return combine_digests(s.digest() for s in self.shards)

    def close(self):
        for s in self.shards:
            s.close()
        self.shards = []


def combine_digests(parts) -> tuple:
    """(count, sum, xor) digests of disjoint shards -> the digest of their union."""
    c = sm = x = 0
    for pc, ps, px in parts:
        c += int(pc)
        sm = (sm + int(ps)) & 0xFFFFFFFFFFFFFFFF
        x ^= int(px)
    return c, sm, x


def local_buffer_sizes(net, cfg, world: int, status: bool = True):
    """Default (frontier, inbox) capacities in vectors for `world` shards on
    this GPU: the tables of ALL shards are budgeted first (each shard's
    table is cfg.table, padded as device_table_config does), then 40% of the
    memory they leave is split evenly over the shards' frontiers and
    inboxes."""
    from . import statevec
    from .explore import device_table_config
    from .hashtable import slots_per_bucket
    scheme = statevec.make_scheme(net)
    vlen = statevec.device_vlen(scheme, cfg.pad_vlen3)
    tc = device_table_config(cfg.table, scheme, vlen)
    nb = tc.capacity_words // tc.bucket_words
    spb = slots_per_bucket(tc.bucket_words, vlen, tc.resolved_layout())
    table_b = nb * (4 * tc.bucket_words + ((((spb + 7) & ~7)) if status else 0))
    _sm, free, _tot = device_info()
    left = max(0, free - world * table_b - (256 << 20))
    each = max(1 << 16, int(left * 0.2) // (world * 4 * vlen))
    each = min(each, nb * spb + 2)
    return each, each


def explore_local_shards(net, cfg, world: int, inbox_capacity: int = 0, frontier_capacity: int = 0,
                         status: bool = True):
    """Hash-owner sharded exploration with all `world` shards in this
    process (one GPU): the multi-GPU protocol and kernels, with peer
    inboxes as local device memory.  Returns an ExplorationReport; its
    results equal explore(net, cfg)'s."""
    ex = LocalShardExplorer(net, cfg, world, inbox_capacity, frontier_capacity, status=status)
    try:
        return ex.run()
    finally:
        ex.close()


def explore_fused(shards, dist, torch, detect: bool, max_iterations=None,
                  device=None, digest: bool = True) -> ShardResult:
    """Multi-process driver (one process per GPU, holding one shard or
    several): shards were connected with their peers' IPC handles; the
    barrier and the stats reductions are NCCL all_reduces on the shards'
    stream."""
    if not isinstance(shards, (list, tuple)):
        shards = [shards]
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    flag = torch.zeros(1, dtype=torch.int64, device=dev)

    def barrier():
        # this process's shard kernels (and their peer stores) complete
        # before the collective, whatever stream or backend it runs on: a
        # gloo all_reduce of a host tensor would not wait for them
        for s in shards:
            if hasattr(s, "sync"):
                s.sync()
        dist.all_reduce(flag)

    def reduce(a, op=None):
        t = torch.from_numpy(a.astype(np.int64)).to(dev)
        dist.all_reduce(t, op=op or dist.ReduceOp.SUM)
        return t.cpu().numpy().astype(np.uint64)

    tot, kept, rounds, outcome, lms, routed = _run_levels(list(shards), barrier, reduce, detect, max_iterations,
                                                          reduce_max=lambda a: reduce(a, dist.ReduceOp.MAX))
    tot = reduce(tot)
    lms = float(reduce(np.array([int(lms * 1e6)], np.uint64), dist.ReduceOp.MAX)[0]) / 1e6
    gathered = [None] * dist.get_world_size()
    mine = [s.digest() for s in shards] if digest else []
    dist.all_gather_object(gathered, (kept, mine))
    dls = tuple(sorted(s for part, _ in gathered for s in part)[:100])
    dig = combine_digests(d for _, ds in gathered for d in ds) if digest else None
    return ShardResult(states=int(tot[0]), transitions=int(tot[1]), deadlocks=dls,
                       deadlocks_total=int(tot[3]), expanded=int(tot[2]), iterations=rounds,
                       outcome=outcome, levels=rounds - 1, digest=dig, routed=routed, level_ms=lms,
                       probes=int(tot[4]))


def connect_fused(shards, dist):
    """Exchange the shards' inbox IPC handles and map the peers': shards in
    other processes through CUDA IPC, shards of this process directly."""
    from ._lib import check, lib
    if not isinstance(shards, (list, tuple)):
        shards = [shards]
    mine = {s.rank: s.ipc_handle() for s in shards}
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, mine)
    world = shards[0].world
    table = [IPC_ZERO] * world
    for part in parts:
        for r, h in part.items():
            table[r] = h
    for s in shards:
        s.connect([IPC_ZERO if r in mine else table[r] for r in range(world)])
        for p in shards:
            if p is not s:
                check(lib().gx_shard_link(s.handle, p.handle))


def explore_sharded(backend, dist, torch, scheme, initial_packed: np.ndarray, detect: bool,
                    max_iterations=None, device=None) -> ShardResult:
    """Run the level loop of the module docstring on every rank."""
    from .statevec import unpack

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    backend.reset()
    own = int(backend.owner(initial_packed)[0])
    nfront = 0
    aborted = torch.zeros(1, dtype=torch.int64, device=dev)
    if own == rank:
        r = backend.seed_frontier(initial_packed)
        if r < 0:
            aborted[0] = 1
        else:
            nfront = r
    dist.all_reduce(aborted)
    rounds = 0
    trans_total = dl_total = expanded = 0
    outcome = "COMPLETE"
    kept = []
    if aborted.item():
        outcome = "TABLE_FULL"
    else:
        while True:
            counts, tr, dl = backend.expand_route(nfront, detect)
            if dl and detect:
                kept.extend(tuple(int(x) for x in row) for row in backend.deadlock_vectors())
            recv_counts = torch.empty_like(counts)
            dist.all_to_all_single(recv_counts, counts)
            s_split = counts.cpu().tolist()
            r_split = recv_counts.cpu().tolist()
            ns, nr = sum(s_split), sum(r_split)
            if nr > backend.cap:
                raise RuntimeError(f"receive buffer ({backend.cap} vectors) too small for {nr}")
            dist.all_to_all_single(backend.recv[:nr], backend.send[:ns],
                                   output_split_sizes=r_split, input_split_sizes=s_split)
            n_next, full = backend.insert_append(nr)
            stats = torch.tensor([nfront, n_next, tr, dl, int(full)], dtype=torch.int64, device=dev)
            dist.all_reduce(stats)
            claims, new, tr_sum, dl_sum, full_sum = (int(x) for x in stats.cpu().tolist())
            expanded += claims
            trans_total += tr_sum
            dl_total += dl_sum
            rounds += 1
            nfront = n_next
            if full_sum:
                outcome = "TABLE_FULL"
                break
            if claims == 0:
                break
            if max_iterations is not None and rounds >= max_iterations:
                outcome = "ITERATION_CAP"
                break
    st = torch.tensor([backend.states()], dtype=torch.int64, device=dev)
    dist.all_reduce(st)
    # deadlocks: the 100 smallest composite states over all ranks
    gathered = [None] * world
    dist.all_gather_object(gathered, sorted(unpack(scheme, p) for p in kept)[:100])
    dls = tuple(sorted(s for part in gathered for s in part)[:100])
    return ShardResult(states=int(st.item()), transitions=trans_total, deadlocks=dls,
                       deadlocks_total=dl_total, expanded=expanded, iterations=rounds,
                       outcome=outcome, levels=rounds - 1)


def hash_bench_shards(shards, barrier, reduce, reduce_max, total: int, duplication: int, seed: int = 11):
    """One run of the hash-partitioned FINDORPUT benchmark over `shards`
    (this process's; the peers' run in theirs): the global sequence of
    `total` ops is split evenly over all shards, each routes the keys it
    does not own, then every shard absorbs.  Returns the global
    (inserted, found, table_full, max kernel ms over shards and ranks)."""
    from ctypes import c_int32
    from ._lib import check, lib
    world = shards[0].world
    for s in shards:
        full = c_int32()
        check(lib().gx_shard_begin(s.handle, 0, 0, C.byref(full)))
    barrier()  # every inbox is cleared before any peer routes into it
    for s in shards:
        per = total // world
        first = s.rank * per
        count = per if s.rank < world - 1 else total - first
        s.bench_route(total, duplication, seed, first, count)
    barrier()
    for s in shards:
        s.absorb_chunk()
    st = np.zeros(5, np.uint64)
    ms = 0.0
    for s in shards:
        o, m = s.bench_result()
        st += o
        ms = max(ms, m)
    st = reduce(st)
    ms = float(reduce_max(np.array([int(ms * 1e6)], np.uint64))[0]) / 1e6
    if st[4]:
        raise RuntimeError("inbox overflow in the sharded hash benchmark; raise inbox_capacity")
    inserted = int(st[0])
    return {"ops": total, "duplication": duplication, "inserted": inserted, "found": total - inserted,
            "table_full": bool(st[1]), "routed": int(st[3]), "ms": ms,
            "ops_per_sec": total / (ms / 1e3) if ms > 0 else 0.0}


def bench_sharded(args, torch, dist, model_path, closed_form, table_capacity, clock_sampler=None,
                  cpu_fn=None, peaks=None, golden=None):
    """bench.py's N > 1 leg: one model hash-partitioned over N GPUs (strong
    scaling), fused peer-routed levels.  Device time = CUDA events around
    the K timed explorations, max over ranks; e2e = the same through
    shard construction (CSR upload from host memory, table + inbox
    allocation, IPC mapping) per step.  Also the hash-partitioned isolated
    FINDORPUT benchmark (configs[1] at N GPUs, weak scaling: 2^28 ops per
    GPU), the roofline of the level kernels, the reachable-set digest
    against the golden one, and (rank 0) the CPU reference sample."""
    import tempfile
    import time
    from pathlib import Path

    from . import _lib, statevec
    from .explore import DeviceNetwork, ExploreConfig
    from .hashtable import TableConfig

    from .network import load_network

    rank, world = dist.get_rank(), dist.get_world_size()
    tmp = Path(tempfile.mkdtemp())
    net = load_network(model_path(args.workload, tmp))
    scheme = statevec.make_scheme(net)
    vlen = scheme.vector_length
    cf = closed_form(args.workload)
    # shards per GPU: enough that each table stays inside the TLB reach
    # (profiles/README.md); global shard id = rank * local + l
    per_gpu = cf[0] // world
    gpu_bytes = table_capacity(per_gpu, vlen, args.bucket_words, args.load) * 4
    local = args.shards or max(1, -(-gpu_bytes // (80 << 30)))
    gworld = world * local
    per_shard = cf[0] // gworld + (cf[0] >> 8) // gworld + 4096
    cap_words = table_capacity(per_shard, vlen, args.bucket_words, args.load)
    cfg = ExploreConfig(table=TableConfig(bucket_words=args.bucket_words,
                                          num_hash_functions=args.hash_functions,
                                          capacity_words=cap_words), detect_deadlocks=True,
                        cache_slots=max(1, args.cache_slots), dedup=getattr(args, "dedup", False))
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream().cuda_stream
    # frontier: two adjacent levels with margin; inbox: most of what is left
    # after the tables, so that levels need few chunks
    frontier = max(1 << 20, int(per_shard * 0.05))
    free = torch.cuda.mem_get_info()[0]
    if torch.cuda.device_count() < world:  # ranks sharing a GPU (functional check)
        free //= world
    table_b = cap_words * 4 * local  # data; the status array is dropped when it does not fit
    status = table_b * 9 // 8 + 0.3 * (free - table_b) < free
    table_b = table_b * 9 // 8 if status else table_b
    inbox = max(1 << 20, int((free - table_b - local * frontier * 4 * vlen) * 0.7) // (4 * vlen * local))

    def make():
        shards = [FusedShard(net, cfg, rank * local + l, gworld, inbox_capacity=inbox,
                             frontier_capacity=frontier, stream=stream, status=status)
                  for l in range(local)]
        connect_fused(shards, dist)
        return shards

    def close(shards):
        for sh in shards:
            sh.close()

    shard = make()
    res = None
    for _ in range(args.warmup):
        res = explore_fused(shard, dist, torch, True, device=dev, digest=False)
    torch.cuda.synchronize()
    dist.barrier()
    l0 = _lib.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = clock_sampler if clock_sampler is not None else _Null()
    lms = []
    with ctx:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            res = explore_fused(shard, dist, torch, True, device=dev, digest=False)
            lms.append(res.level_ms)
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    launches = _lib.kernel_launches() - l0
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # set identity of the last timed run (all shards' tables still hold it)
    mine = [s.digest() for s in shard]
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    digest = list(combine_digests(d for p in parts for d in p))
    close(shard)
    assert (res.states, res.transitions) == cf, (res.states, res.transitions, cf)
    if golden and golden.get("digest"):
        assert digest == golden["digest"], (digest, golden["digest"])
    # e2e: shards built (CSR from host memory, tables, inboxes, IPC) every step
    e2e = []
    for i in range(args.e2e_steps + 1):
        dist.barrier()
        t0 = time.perf_counter()
        sh = make()
        r = explore_fused(sh, dist, torch, True, device=dev, digest=False)
        close(sh)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i:
            e2e.append(float(t.item()))
    e2e_value = r.states * len(e2e) / sum(e2e) if e2e else None
    dn = DeviceNetwork(net, scheme)
    csr_bytes = (dn.csr_bytes + 4 * vlen) * gworld
    dn.close()

    # roofline of the level kernels (all GPUs): SURVEY §8(d) bytes, plus the
    # probe-based bytes and the NVLink bytes of the routed successors
    hbm = (peaks or {}).get("hbm_gbs", 6650.0)
    sbw = max(32, 4 * args.bucket_words)
    level_ms = sum(lms) / len(lms)
    alg = res.transitions * sbw + res.states * 12 * vlen
    probe_b = res.probes * sbw + res.states * 12 * vlen + res.routed * 8 * vlen
    achieved = alg / (level_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm * world, "unit": "GB/s",
            "frac": achieved / (hbm * world), "traffic": None,
            "kernel": "k_level_routed + k_absorb (all GPUs)", "algorithmic_bytes_per_step": alg,
            "kernel_ms_per_step": level_ms, "bytes_model": "transitions*max(32,4*bw) + states*12*vlen",
            "probe_bytes_per_step": probe_b,
            "frac_probe_based": probe_b / (level_ms / 1e3) / 1e9 / (hbm * world),
            "nvlink_bytes_per_step": res.routed * 4 * vlen,
            "peak_note": f"{hbm} GB/s per GPU (MEASURED_PEAKS.json) x {world}"}

    # the hash-partitioned FINDORPUT benchmark: 2^28 ops per GPU, 2-word keys
    hash_rows = []
    if not getattr(args, "no_hash_bench", False):
        ops = (1 << 28) * world
        for d in (1, 10):
            per = (ops // d) // gworld + ((ops // d) >> 6) // gworld + 4096
            hcfg = ExploreConfig(table=TableConfig(bucket_words=32, num_hash_functions=8,
                                                   capacity_words=table_capacity(per, 2, 32, 0.5)))
            # any network with 2-word states and a spare top bit gives the
            # table geometry (keys are 31-bit words): the token ring N=19
            hnet = load_network(model_path("ring19", tmp))
            hs = [FusedShard(hnet, hcfg, rank * local + l, gworld, inbox_capacity=ops // gworld + (1 << 20),
                             frontier_capacity=1 << 16, stream=stream, status=False) for l in range(local)]
            connect_fused(hs, dist)

            flag = torch.zeros(1, dtype=torch.int64, device=dev)

            def barrier():
                # stream-ordered: the all_reduce runs after this rank's
                # kernels, so no peer absorbs before our stores landed
                torch.cuda.current_stream().synchronize()
                dist.all_reduce(flag)
                torch.cuda.current_stream().synchronize()

            def red(a, op=None):
                t = torch.from_numpy(a.astype(np.int64)).to(dev)
                dist.all_reduce(t, op=op or dist.ReduceOp.SUM)
                return t.cpu().numpy().astype(np.uint64)

            hash_bench_shards(hs, barrier, red, lambda a: red(a, dist.ReduceOp.MAX), ops, d)  # warm-up
            row = hash_bench_shards(hs, barrier, red, lambda a: red(a, dist.ReduceOp.MAX), ops, d)
            for h in hs:
                h.close()
            assert row["inserted"] == ops // d and not row["table_full"], row
            row.update({"bw": 32, "vlen": 2, "n_gpus": world, "ops_per_gpu": ops // world,
                        "gbs_alg": ops * sbw / (row["ms"] / 1e3) / 1e9})
            hash_rows.append(row)
    cpu = cpu_fn() if (cpu_fn is not None and rank == 0) else None
    return {
        "metric": "states explored/sec", "value": res.states * args.steps / (ms / 1e3),
        "unit": "states/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (generated model, exact state space)",
        "config": {"workload": f"configs[4] token ring N={args.workload[4:]} hash-partitioned",
                   "states": res.states, "transitions": res.transitions, "levels": res.levels,
                   "vector_words": vlen, "bucket_words": args.bucket_words,
                   "hash_functions": args.hash_functions, "table_words_per_shard": cap_words,
                   "shards_per_gpu": local, "status_array": bool(status),
                   "block_cache_slots": args.cache_slots,
                   "l2_policy": "tables re-zeroed every step; tables >> 126 MB L2",
                   "parallelism": f"hash-owner sharding x{gworld} ({local} per GPU): successors "
                                  "routed to the owner's inbox by P2P stores inside the level "
                                  "kernel (CUDA IPC over NVLink), NCCL all_reduce of level "
                                  "counters"},
        "roofline": roof, "cpu_baseline": cpu,
        "digest": {"value": digest, "golden": (golden or {}).get("digest"),
                   "equal": digest == (golden or {}).get("digest")},
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": csr_bytes,
                "d2h_bytes_per_step": (res.levels + 2) * 64 * gworld + 400 * vlen,
                "api": "FusedShard + connect_fused + explore_fused per step"},
        "hash_bench_sharded": hash_rows,
        "routed_per_step": res.routed, "probes_per_step": res.probes,
        "gpu_launches": launches,
        "clocks": clock_sampler.summary() if clock_sampler is not None else None,
    }


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
