"""Level-synchronous BFS reachability on the B200.

Python surface of /root/reference/pkg/src/ltsmc/explore.py (`ExploreConfig`
:47-62, `ExplorationReport` :65-88, `explore` :300-395, outcome constants
:33-35, DEADLOCK_KEEP :38).  One call to `gx_explore` (include/gx.h) runs
the whole search on the device: per level one kernel expands the frontier
(successor generation per process LTS and per synchronisation rule from
the network CSR), FINDORPUTs every successor into the state table and
appends the inserted ones to the next frontier.  Rounds are exact BFS
levels, so `iterations` = levels + 1 on a complete run, as in the
reference (explore.py:234-240, 255-268).

`cache_slots` keeps its meaning as the size of the per-worker dedup cache
(`LocalCache`, explore.py:91-144): on the device it sizes each thread
block's shared-memory cache (at most 8192 slots and what the three
resident blocks per SM leave of shared memory, ~1000 at bw 32; below 32
the cache is off).  The CPU worker knobs (`workers`,
`backend`) are accepted and validated for compatibility; they do not change
device execution.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import statevec
from ._lib import ExploreCfg, NetworkCsr, Report, check, lib, ptr
from .hashtable import OCCUPIED_NEW, StateTable, TableConfig, TableFullError  # noqa: F401
from .network import Network, to_csr

COMPLETE = "COMPLETE"
OUTCOME_TABLE_FULL = "TABLE_FULL"
ITERATION_CAP = "ITERATION_CAP"
OUTCOMES = (COMPLETE, OUTCOME_TABLE_FULL, ITERATION_CAP)
DEADLOCK_KEEP = 100
BACKENDS = ("auto", "threads", "processes", "cuda")


@dataclass(frozen=True)
class ExploreConfig:
    workers: int = 1
    table: TableConfig = field(default_factory=TableConfig)
    cache_slots: int = 4096
    detect_deadlocks: bool = False
    max_iterations: int | None = None
    backend: str = "auto"
    # device knobs (new): frontier buffer capacity in vectors (0 = sized
    # from free HBM) and lanes per bucket probe (0 = one 16-byte chunk each)
    frontier_capacity: int = 0
    probe_group: int = 0
    # GPU-wide L2-resident dedup filter of 2^filter_log2 entries in front of
    # the table (0 = off): duplicate successors generated anywhere on the GPU
    # skip their random table probe
    filter_log2: int = 0
    # store 3-word states padded to 4 words (in-band table, one 128-bit CAS
    # per insert) instead of the status-byte protocol; the table then has
    # vlen-4 slots (8 per 32-word bucket instead of 10)
    pad_vlen3: bool = True
    # > 1: hash-partition the state space into this many shards on this GPU
    # (the multi-GPU engine with local inboxes); `table` then sizes EACH
    # shard.  Keeps each probed table range inside the TLB reach when one
    # table would be tens of GB.  Dumps need shards == 1.
    shards: int = 1
    # compute the order-independent digest of the reachable set
    # (gx_table_digest) after the search and put it on the report
    state_digest: bool = True
    # sharded engine: partitioned levels with the level-wide duplicate
    # filter (gx_part.cuh; only the first copy of each successor in a chunk
    # probes the table) instead of the fused probe-as-you-expand kernels;
    # the filter set has 2^dedup_set_log2 32-byte groups (L2 resident)
    dedup: bool = False
    dedup_set_log2: int = 20
    # sharded engine, fused levels: split each inbox in two halves and
    # absorb chunk c - 1's keys inside chunk c's expansion launch
    pipeline: bool = False

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.cache_slots < 1:
            raise ValueError("cache_slots must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"unknown backend {self.backend!r}")
        if self.shards < 1:
            raise ValueError("shards must be >= 1")


@dataclass(frozen=True)
class ExplorationReport:
    states: int
    transitions: int
    deadlocks: tuple
    deadlocks_total: int
    expanded: int
    iterations: int
    wall_time: float
    throughput: float
    outcome: str
    device_ms: float = 0.0
    max_frontier: int = 0
    kernels: int = 0
    level_ms: float = 0.0
    probes: int = 0
    # (count, sum, xor) of the per-state hashes of the reachable set
    # (include/gx.h gx_table_digest); None when not computed
    digest: tuple | None = None
    # sharded engine: successors stored into another shard's inbox
    routed: int = 0

    def to_dict(self) -> dict:
        return {
            "states": self.states,
            "transitions": self.transitions,
            "deadlocks": [list(s) for s in self.deadlocks],
            "deadlocks_total": self.deadlocks_total,
            "expanded": self.expanded,
            "iterations": self.iterations,
            "wall_time": self.wall_time,
            "throughput": self.throughput,
            "outcome": self.outcome,
        }


class DeviceNetwork:
    """A Network's CSR uploaded to the device once (gx_net_create)."""

    def __init__(self, net: Network, scheme=None, stream=None, vlen: int | None = None):
        self.net = net
        self.scheme = scheme or statevec.make_scheme(net)
        self.vlen = vlen or self.scheme.vector_length  # device words per state (padding)
        csr = to_csr(net, self.scheme, self.vlen)
        self._arrays = csr
        init = np.zeros(self.vlen, np.uint32)
        packed = statevec.pack(self.scheme, net.initial)
        init[:len(packed)] = packed
        self._init = init
        c = NetworkCsr()
        c.nproc, c.nrules, c.vlen = csr["nproc"], csr["nrules"], csr["vlen"]
        for name in ("proc", "qtab", "im_dst", "trig", "rules", "parts", "rq", "rdst", "dedup"):
            a = csr[name]
            setattr(c, name, ptr(a))
            setattr(c, "n_" + name, a.size)
        c.n_proc = 4 * csr["nproc"]
        c.n_rules = 4 * csr["nrules"]
        if csr["nrules"] == 0:
            c.n_rules = 0
        c.initial = ptr(init)
        self.csr_bytes = sum(csr[k].nbytes for k in csr if isinstance(csr[k], np.ndarray))
        h = C.c_void_p()
        check(lib().gx_net_create(C.byref(c), stream, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().gx_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def expand_batch(self, states_packed, with_successors=True):
        """Device expand of packed states -> (counts, nsucc, successors)."""
        v = self.scheme.vector_length
        s = np.ascontiguousarray(np.asarray(states_packed, np.uint32).reshape(-1, v))
        n = s.shape[0]
        counts = np.zeros(n, np.uint64)
        nsucc = np.zeros(n, np.uint32)
        total = C.c_uint64()
        check(lib().gx_expand(self._h, ptr(s), n, ptr(counts, C.c_uint64), ptr(nsucc), None, 0,
                              C.byref(total)))
        succ = None
        if with_successors:
            cap = max(int(total.value), 1)
            succ = np.zeros((cap, v), np.uint32)
            check(lib().gx_expand(self._h, ptr(s), n, None, None, ptr(succ), cap, C.byref(total)))
            succ = succ[:total.value]
        return counts, nsucc, succ


class Explorer:
    """Reusable device explorer: network CSR + state table stay resident
    across runs (the table is cleared at the start of every run)."""

    def __init__(self, net: Network, cfg: ExploreConfig, stream=None, status: bool = True):
        self.net = net
        self.cfg = cfg
        self.scheme = statevec.make_scheme(net)
        self.vlen = statevec.device_vlen(self.scheme, cfg.pad_vlen3)
        self.dnet = DeviceNetwork(net, self.scheme, stream, self.vlen)
        self.table = StateTable(device_table_config(cfg.table, self.scheme, self.vlen), self.vlen,
                                mark=statevec.mark_bit(self.scheme, self.vlen), stream=stream,
                                status=status)
        self.last = None

    def run(self) -> ExplorationReport:
        cfg = self.cfg
        # max_iterations: None = no cap; any integer caps as in the reference
        # (explore.py:256-261: rounds >= max_iterations, so 0 stops after round 1)
        cap = -1 if cfg.max_iterations is None else max(0, int(cfg.max_iterations))
        ecfg = ExploreCfg(int(cfg.detect_deadlocks), int(cfg.filter_log2), cap,
                          int(cfg.frontier_capacity), int(cfg.probe_group),
                          int(min(cfg.cache_slots, 1 << 30)))
        rep = Report()
        v = self.vlen
        dl = np.zeros((DEADLOCK_KEEP, v), np.uint32)
        t0 = time.perf_counter()
        check(lib().gx_explore(self.dnet.handle, self.table.handle, C.byref(ecfg), C.byref(rep),
                               ptr(dl)))
        wall = time.perf_counter() - t0
        sv = self.scheme.vector_length
        kept = [statevec.unpack(self.scheme, tuple(int(x) for x in dl[i, :sv]))
                for i in range(rep.deadlocks_kept)]
        self.last = rep
        return ExplorationReport(
            states=int(rep.states), transitions=int(rep.transitions), deadlocks=tuple(sorted(kept)),
            deadlocks_total=int(rep.deadlocks_total), expanded=int(rep.expanded),
            iterations=int(rep.iterations), wall_time=wall,
            throughput=rep.states / wall if wall > 0 else 0.0, outcome=OUTCOMES[rep.outcome],
            device_ms=float(rep.device_ms), max_frontier=int(rep.max_frontier),
            kernels=int(rep.kernels), level_ms=float(rep.level_ms), probes=int(rep.probes),
            digest=self.digest() if cfg.state_digest else None)

    def digest(self) -> tuple:
        """(count, sum, xor) digest of the reachable set now in the table."""
        return self.table.digest(self.scheme.vector_length)

    def dump_states(self) -> str:
        """The canonical dump (statevec.py:93-100), sorted on the device."""
        return statevec.dump_states_array(self.table.sorted_vectors(self.scheme.vector_length),
                                          presorted=True)

    def dump_table(self) -> str:
        hs, st, ws = self.table.dump_arrays()
        ws = ws[:, :self.scheme.vector_length]
        spb = self.table.slots_per_bucket
        lines = ["bucket,slot,status,words\n"]
        for h, s, w in zip(hs, st, ws):
            lines.append(f"{int(h) // spb},{int(h) % spb},{'NEW' if s == OCCUPIED_NEW else 'OLD'},"
                         f"{statevec.format_packed(w)}\n")
        return "".join(lines)

    def close(self):
        self.table.close()
        self.dnet.close()


def device_table_config(table: TableConfig, scheme, vlen: int) -> TableConfig:
    """The table geometry for `vlen`-word device slots.  A padded 3-word
    state (vlen 4) needs more words per slot than the reference's 3, so the
    bucket count grows until the table has at least the reference's slot
    count for the same TableConfig (hashtable.py:89-111,155-159): the same
    number of states fits before TABLE_FULL."""
    sv = scheme.vector_length
    if vlen == sv:
        return table
    from dataclasses import replace

    from .hashtable import slots_per_bucket
    layout = table.resolved_layout()
    bw = table.bucket_words
    ref_slots = (table.capacity_words // bw) * slots_per_bucket(bw, sv, layout)
    spb = slots_per_bucket(bw, vlen, layout)
    buckets = -(-ref_slots // spb)
    return replace(table, capacity_words=max(buckets, 1) * bw)


def explore(net: Network, cfg: ExploreConfig, dump_states=None, dump_table=None):
    """Run the device reachability analysis and return its report
    (explore.py:300-395); optional canonical state dump and table CSV."""
    if cfg.shards > 1:
        if dump_states is not None or dump_table is not None:
            raise ValueError("dump_states / dump_table need ExploreConfig(shards=1)")
        from .distributed import explore_local_shards
        return explore_local_shards(net, cfg, cfg.shards)
    ex = Explorer(net, cfg)
    try:
        report = ex.run()
        if dump_states is not None:
            with open(dump_states, "w", encoding="utf-8") as fh:
                fh.write(ex.dump_states())
        if dump_table is not None:
            with open(dump_table, "w", encoding="utf-8") as fh:
                fh.write(ex.dump_table())
        return report
    finally:
        ex.close()
