"""Hash-owner sharded exploration across GPUs (one process per GPU).

Every rank owns the states whose owner hash (a splitmix finaliser of the
table's fold value, decorrelated from all bucket indices; gx_device.cuh
`owner_of`) equals its rank, holds that shard of the state table, and
expands only its own frontier.  One BFS level:

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
            if max_iterations and rounds >= max_iterations:
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


def bench_sharded(args, torch, dist, model_path, closed_form, table_capacity):
    """bench.py's N > 1 leg: strong scaling of one model over N GPUs."""
    import statistics
    import tempfile
    import time
    from pathlib import Path

    from . import _lib, statevec
    from .explore import ExploreConfig
    from .hashtable import TableConfig
    from .network import load_network

    rank, world = dist.get_rank(), dist.get_world_size()
    tmp = Path(tempfile.mkdtemp())
    net = load_network(model_path(args.workload, tmp))
    scheme = statevec.make_scheme(net)
    cf = closed_form(args.workload)
    per_rank = cf[0] // world + (cf[0] >> 6) + 1024
    cap_words = table_capacity(per_rank, scheme.vector_length, args.bucket_words, args.load)
    cfg = ExploreConfig(table=TableConfig(bucket_words=args.bucket_words,
                                          num_hash_functions=args.hash_functions,
                                          capacity_words=cap_words), detect_deadlocks=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    backend = DeviceShard(net, cfg, world, torch, capacity=max(1 << 20, per_rank // 4),
                          stream=torch.cuda.current_stream().cuda_stream)
    init = np.asarray(statevec.pack(scheme, net.initial), np.uint32)
    res = None
    for _ in range(args.warmup):
        res = explore_sharded(backend, dist, torch, scheme, init, True, device=dev)
    torch.cuda.synchronize()
    dist.barrier()
    l0 = _lib.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = explore_sharded(backend, dist, torch, scheme, init, True, device=dev)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    backend.close()
    return {
        "metric": "states explored/sec", "value": res.states * args.steps / (ms / 1e3),
        "unit": "states/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (generated model, exact state space)",
        "config": {"workload": args.workload, "states": res.states, "transitions": res.transitions,
                   "levels": res.levels, "parallelism": f"hash-owner sharding x{world}, "
                   "per-level NCCL all_to_all + all_reduce"},
        "gpu_launches": _lib.kernel_launches() - l0,
    }
