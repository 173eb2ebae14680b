"""Benchmark driver (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ring16]
  python bench.py --impl reference ...        # CPU reference arm

Metric: states explored/sec of a full level-synchronous reachability run
(BASELINE.json configs[3], the synthetically scaled token ring, rescaled
to the chosen size).  A step = one complete exploration of the model from
its initial state: table cleared, every BFS level expanded on the device,
statuses finalised, report read back.

  value      states / (device time of the K timed steps)  [inputs resident]
  e2e        the same through the public API `explore(net, cfg)`: network
             CSR uploaded from host memory, table allocated, report copied
             back, every step
  roofline   dominant kernel k_level: algorithmic bytes = transitions x
             S(bw) + states x 12 vlen over the summed
             CUDA-event time of its launches
  cpu_baseline / --impl reference
             the reference's bucket-partitioned parallel engine, ported to C
             (oracle/gx_oracle.c, explore.py:212-351 restated), on the host
             cores with all threads, on a bounded sample (token ring N=12)

Between timed steps the table is re-zeroed (> L2 in size), so every step
starts cold; inputs larger than L2 are stated in config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = ROOT / "MEASURED_PEAKS.json"
TLB_REACH = 60 << 30    # one table beyond this: shard it on the GPU (profiles/README.md)
SHARD_BYTES = 80 << 30  # table bytes per shard at most (ring19 sweep: 2 x 79 GB > 3 x 52 GB > 4 x 39 GB)
TRAFFIC = ROOT / "profiles" / "traffic.json"
GOLDEN_DIGESTS = ROOT / "tests" / "golden" / "digests.json"
METRIC = "states explored/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default="ring19",
                    help="ringN | gasN | petersonN (generated models); default ring19 = "
                         "BASELINE configs[3], a ~157 GB table")
    ap.add_argument("--bucket-words", type=int, default=32)
    ap.add_argument("--hash-functions", type=int, default=32,
                    help="K (the reference default is 8; load >= 0.6 needs more, SURVEY §0.3)")
    ap.add_argument("--load", type=float, default=0.8,
                    help="target table load factor (ring19 sweep with the refill probe: 0.8 > 0.85 > 0.75 > 0.9)")
    ap.add_argument("--engine", choices=("auto", "table", "shards"), default="auto",
                    help="one table, or hash-owner shards on this GPU (auto: shards once one "
                         "table would outgrow the TLB reach)")
    ap.add_argument("--shards", type=int, default=0, help="shard count (0 = auto)")
    ap.add_argument("--inbox-frac", type=float, default=0.3,
                    help="sharded engine: inbox keys per shard = frac * states / shards")
    ap.add_argument("--frontier-frac", type=float, default=0.035,
                    help="frontier vectors per shard = frac * states / shards")
    ap.add_argument("--no-status", action="store_true",
                    help="exploration-only tables without the per-slot status array")
    ap.add_argument("--probe-group", type=int, default=0)
    ap.add_argument("--cache-slots", type=int, default=4096,
                    help="per-block shared-memory dedup cache entries (< 32 = off)")
    ap.add_argument("--filter-log2", type=int, default=0,
                    help="GPU-wide L2 dedup filter of 2^k entries (0 = off)")
    ap.add_argument("--dedup", action="store_true",
                    help="sharded engine: partitioned levels with the level-wide L2 duplicate filter")
    ap.add_argument("--dedup-set-log2", type=int, default=20)
    ap.add_argument("--pipeline", type=int, default=0,
                    help="sharded engine: absorb chunk c-1's inbox inside chunk c's expansion launch")
    ap.add_argument("--cpu-sample", default="ring14",
                    help="token ring the CPU reference arm explores (ring14: 4.5e7 states, ~12 s on 16 cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hash-bench", action="store_true",
                    help="skip the isolated hash-table sweeps (configs[1])")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--crosscheck", type=int, default=1,
                    help="sharded headline: re-explore once on one table and assert the same digest")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the configs[2] (peterson6) and ring16 side measurements")
    return ap.parse_args()


def model_path(name: str, root: Path) -> Path:
    from paper_1801_05857_b200.bench import gen_gas_station, gen_peterson, gen_token_ring
    kind = name.rstrip("0123456789")
    n = int(name[len(kind):])
    gen = {"ring": gen_token_ring, "gas": gen_gas_station, "peterson": gen_peterson}[kind]
    return gen(n, root / name)[1]


def closed_form(name: str):
    """(states, transitions) known in closed form."""
    if name.startswith("ring"):
        n = int(name[4:])
        return 2 * n * 3 ** (n - 1), 4 * n * n * 3 ** (n - 2)
    return None


def table_capacity(states_estimate: int, vlen: int, bw: int, load: float) -> int:
    from paper_1801_05857_b200.hashtable import slots_per_bucket
    layout = "half" if bw == 32 else "plain"
    spb = slots_per_bucket(bw, vlen, layout)
    buckets = int(states_estimate / load / spb) + 64
    return buckets * bw


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_hash_baseline(total: int = 1 << 22):
    """run_insert_bench's CPU counterpart (reference bench.py:120-202 with
    threads=1): the reference's table restated in C
    (oracle/gx_oracle.c find_or_insert, one thread) inserting a
    duplication sequence of `total` one-word keys, per bucket size and
    d in {1, 10, 100}; the table sized as insert_bench_table_config."""
    import numpy as np

    from oracle import oracle as O
    from paper_1801_05857_b200.bench import DuplicationSpec, insert_bench_table_config
    rows = []
    for bw in (4, 8, 16, 32):
        for d in (1, 10, 100):
            spec = DuplicationSpec(total=total, duplication=d, vector_length=1)
            cfg = insert_bench_table_config(spec, bw)
            rng = np.random.default_rng(11)
            u = total // d
            keys = rng.integers(0, 1 << 32, size=u, dtype=np.uint64).astype(np.uint32)
            seq = keys[np.minimum(rng.permutation(total) // d, u - 1)]
            t = O.Table(bw, 8, cfg.capacity_words, None, 42, 1)
            t0 = time.perf_counter()
            codes, _ = t.find_or_insert_batch(seq)
            dt = time.perf_counter() - t0
            rows.append({"bw": bw, "d": d, "ops": total, "ops_per_sec": total / dt,
                         "inserted": int((codes == 1).sum())})
    return {"kind": "port", "cores": 1, "unit": "FINDORPUT ops/s", "rows": rows,
            "sample": f"{total} one-word keys per cell, oracle/gx_oracle.c table (hashtable.py:224-280 "
                      "restated), 1 thread, K=8, table sized for <= 50% load at d=1"}


def cpu_reference(sample: str, steps: int, warmup: int, tmp: Path):
    """The reference engine's C port on all host threads, bounded sample."""
    from oracle import oracle as O
    path = model_path(sample, tmp)
    net = O.Net.from_file(path)
    threads = os.cpu_count() or 1
    cf = closed_form(sample)
    states_est = cf[0] if cf else 1 << 22
    cap = table_capacity(states_est, net.vlen, 32, 0.5)
    times, r = [], None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        r = O.explore(net, capacity_words=cap, workers=threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    total = sum(times)
    return {
        "value": r.states * len(times) / total,
        "unit": "states/s",
        "cores": threads,
        "kind": "port",
        "sample": f"token ring N={sample[4:]} ({r.states} states, {r.transitions} transitions) "
                  f"full exploration, {threads} worker threads, reference explore.py engine "
                  f"restated in C (oracle/gx_oracle.c); {len(times)} timed runs",
        "states": r.states,
        "seconds_per_run": total / len(times),
    }


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    with tempfile.TemporaryDirectory() as td:
        base = cpu_reference(args.cpu_sample, args.steps, args.warmup, Path(td))
    line = {
        "impl": "reference",
        "metric": METRIC, "value": base["value"], "unit": "states/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * base["seconds_per_run"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (generated token-ring model)",
        "config": {"workload": f"token ring N={args.cpu_sample[4:]} (bounded CPU sample of "
                               f"configs[3])", "engine": "reference explore() port, C threads"},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": base["value"], "unit": "states/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def s_bw(bw: int) -> int:
    """Bytes one bucket probe moves, rounded up to a 32-byte sector."""
    return max(32, 4 * bw)


def hash_sweep(ra: dict):
    """Isolated FINDORPUT throughput vs bucket size and fill (configs[1],
    SURVEY §8(d) protocol 2): a 32 GiB table of 2-word vectors (>> L2;
    1-word keys have only 2^31 distinct values next to the mark bit, too
    few to fill it) filled step by step with fresh random keys.  At each
    fill f: an untimed fill to f - 2%, then a timed insert batch of 2% of
    the slots (8.6e7 ops at bw 32, 6.9e7 at bw 4: 2^28 inserts would move
    the fill by ~6%), then a timed lookup batch of 2^28 FINDORPUTs of keys
    already present (the last 2^28 rows inserted).  K = 8 (the reference
    default) and K = 32 (fill >= 0.6 needs it).  Keys are
    generated inside the kernel, so the algorithmic bytes per op are the
    bucket probe S(bw) (+ one 32-byte sector written per insert); extra
    buckets probed past the first are reported (buckets_per_op) but not
    credited.  frac against R(S(bw)) measured in the same run."""
    from paper_1801_05857_b200.bench import device_insert_bench
    from paper_1801_05857_b200.hashtable import StateTable, TableConfig
    out = []
    words = 1 << 33
    for bw in (4, 8, 16, 32):
        r_g = ra.get(s_bw(bw), {}).get("gbs")
        for k in (8, 32):
            t = StateTable(TableConfig(bucket_words=bw, num_hash_functions=k, capacity_words=words),
                           2, mark=(1, 31))
            slots = t.total_slots
            rows = 0  # rows attempted so far: the next fresh keys start here
            for fill in (0.5, 0.6, 0.7, 0.8, 0.9):
                target = int(fill * slots)
                batch = int(0.02 * slots)
                occ = t.occupancy()[0]
                if target - batch > occ:  # untimed fill to (fill - 2%)
                    n = target - batch - occ
                    r = device_insert_bench(t, n, 1, seed=7, row_base=rows)
                    rows += n
                    if r["full"]:
                        out.append({"vlen": 2, "bw": bw, "k": k, "fill": fill, "table_full": True})
                        break
                r = device_insert_bench(t, batch, 1, seed=7, row_base=rows)
                rows += batch
                nl = min(1 << 28, rows)
                look = device_insert_bench(t, nl, 1, seed=7, row_base=rows - nl)
                assert look["inserted"] == 0 or r["full"], look  # every looked-up key is present
                ins_gbs = r["ops_per_sec"] * (s_bw(bw) + 32) / 1e9
                look_gbs = look["ops_per_sec"] * s_bw(bw) / 1e9
                out.append({"vlen": 2, "bw": bw, "k": k, "fill": fill,
                            "fill_after": t.occupancy()[0] / slots,
                            "insert_ops": batch, "lookup_ops": nl,
                            "insert_ops_per_sec": r["ops_per_sec"],
                            "lookup_ops_per_sec": look["ops_per_sec"],
                            "insert_buckets_per_op": r["buckets_per_op"],
                            "lookup_buckets_per_op": look["buckets_per_op"],
                            "insert_gbs_alg": ins_gbs, "lookup_gbs_alg": look_gbs,
                            "lookup_frac_of_random_roofline": look_gbs / r_g if r_g else None,
                            "table_full": bool(r["full"])})
                if r["full"]:
                    break
            t.close()
    return out


def duplication_sweep(ra: dict):
    """The paper's Fig. 4 protocol (bench.py:90-114,120-202): 2^30 FINDORPUT
    ops (n >= 2^30) over total/d unique random vectors,
    globally shuffled, table sized for <= 50% load at d = 1; bucket 4
    ("Gh-cbs") vs 32 ("Gh"), 1-word vectors (the paper's) and 2-word ones
    (SURVEY §8(d)).  Keys are generated inside the kernel: algorithmic
    bytes per op = S(bw) + 32 per insert.  The reference's checks hold:
    inserted == total // d and inserted == occupancy (bench.py:176-190).  A
    cell whose sizing overfills the buckets reports table_full (vlen 2 at
    bw 4: 2 slots per bucket at 50% load, as in the reference, SURVEY
    B.4)."""
    from paper_1801_05857_b200.bench import (DuplicationSpec, device_insert_bench,
                                             insert_bench_table_config)
    from paper_1801_05857_b200.hashtable import StateTable
    total = 1 << 30
    out = []
    for vlen in (1, 2):
        for bw in (4, 8, 16, 32):
            for d in ((1, 10, 50, 100) if vlen == 1 else (1, 10, 100)):
                spec = DuplicationSpec(total=total, duplication=d, vector_length=vlen)
                t = StateTable(insert_bench_table_config(spec, bw), vlen, mark=(vlen - 1, 31))
                try:
                    r = device_insert_bench(t, total, d, seed=11)
                    occ = t.occupancy()[0]
                finally:
                    t.close()
                u = total // d
                if not r["full"]:
                    assert r["inserted"] == u == occ and r["found"] == total - u, (vlen, bw, d, r, occ)
                alg = (total * s_bw(bw) + u * 32) / (r["ms"] / 1e3) / 1e9
                r_g = ra.get(s_bw(bw), {}).get("gbs")
                out.append({"vlen": vlen, "bw": bw, "d": d, "ops_per_sec": r["ops_per_sec"],
                            "inserted": r["inserted"], "found": r["found"], "occupancy": occ,
                            "buckets_per_op": r["buckets_per_op"], "gbs_alg": alg,
                            "frac_of_random_roofline": alg / r_g if r_g else None,
                            "table_full": bool(r["full"])})
    return out


def single_table_rate(torch, name: str, tmp: Path, runs: int = 2) -> dict:
    """states/s of ringN / gasN / petersonN on one table (the explore()
    engine), CUDA events over `runs` explorations after one warm-up; the
    digest is checked against tests/golden/digests.json when present."""
    import paper_1801_05857_b200 as gx
    from paper_1801_05857_b200.explore import ExploreConfig, Explorer
    from paper_1801_05857_b200.hashtable import TableConfig
    golden = json.loads(GOLDEN_DIGESTS.read_text()).get(name, {}) if GOLDEN_DIGESTS.exists() else {}
    states = golden.get("states") or (closed_form(name) or (1 << 24,))[0]
    net = gx.load_network(model_path(name, tmp))
    from paper_1801_05857_b200 import statevec
    v = statevec.device_vlen(statevec.make_scheme(net))
    cfg = ExploreConfig(table=TableConfig(capacity_words=table_capacity(states, v, 32, 0.5),
                                          num_hash_functions=16), detect_deadlocks=True, state_digest=False)
    ex = Explorer(net, cfg, stream=torch.cuda.current_stream().cuda_stream)
    ex.run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = [ex.run() for _ in range(runs)]
    e1.record()
    torch.cuda.synchronize()
    r = reps[-1]
    d = list(ex.digest())
    ex.close()
    ms = e0.elapsed_time(e1) / runs
    ok = None
    if golden.get("digest"):
        ok = d == golden["digest"] and r.transitions == golden["transitions"]
        assert ok, (name, d, golden)
    return {"workload": name, "states": r.states, "transitions": r.transitions, "levels": r.iterations - 1,
            "ms_per_exploration": ms, "states_per_sec": r.states / (ms / 1e3), "digest_ok": ok}


def extra_workloads(torch, tmp: Path):
    """Side measurements on one table (not the headline): configs[2], a
    peterson7-class model (Peterson's filter lock with 6 processes, 2.1e8
    states), and ring16 (8 GB table), each 1 warm-up + 2 timed runs, their
    reachable sets checked against the golden digests."""
    out = []
    for name in ("peterson6", "ring16"):
        r = single_table_rate(torch, name, tmp)
        r["workload"] = ("configs[2] " if name.startswith("peterson") else "") + name
        out.append(r)
    return out


def random_access(granularities=(32, 64, 128)):
    from paper_1801_05857_b200.bench import random_access_roofline
    out = {}
    for g in granularities:
        r = random_access_roofline(g)
        c = random_access_roofline(g, with_cas=True)
        out[g] = {"gbs": r["gbs"], "gbs_with_cas": c["gbs"], "segments_per_sec": r["segments_per_sec"]}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # more ranks than GPUs (a functional check of the multi-process path on a
    # one-GPU box): ranks share cuda:0 and the counters go over gloo, since
    # NCCL refuses two ranks on one device; the inbox IPC mappings are the
    # same calls
    oversub = world > 1 and torch.cuda.device_count() < world
    if oversub:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # NCCL's init lines (communicator size, transports) on stderr, so the
        # JSON line on stdout stays the only stdout output
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1801_05857_b200.distributed import bench_sharded
        peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
        golden = json.loads(GOLDEN_DIGESTS.read_text()).get(args.workload) if GOLDEN_DIGESTS.exists() else None

        def cpu_fn():
            if args.no_cpu_baseline:
                return None
            with tempfile.TemporaryDirectory() as td:
                c = cpu_reference(args.cpu_sample, 1, 0, Path(td))
            return {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}

        line = bench_sharded(args, torch, dist, model_path, closed_form, table_capacity,
                             ClockSampler(local), cpu_fn=cpu_fn, peaks=peaks, golden=golden)
        if oversub:
            line["config"]["oversubscribed"] = (f"{world} ranks on {torch.cuda.device_count()} GPU(s); "
                                                "gloo counters")
        if rank == 0:
            print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return

    import paper_1801_05857_b200 as gx
    from paper_1801_05857_b200 import _lib, statevec
    from paper_1801_05857_b200.explore import ExploreConfig, Explorer
    from paper_1801_05857_b200.hashtable import TableConfig

    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tmp = Path(tempfile.mkdtemp())
    path = model_path(args.workload, tmp)
    net = gx.load_network(path)
    scheme = statevec.make_scheme(net)
    vlen = scheme.vector_length
    cf = closed_form(args.workload)
    states_est = cf[0] if cf else None
    if states_est is None:
        raise SystemExit("workload without a closed form needs --states")
    # engine: one table, or W hash-owner shards on this GPU when one table
    # would outgrow the TLB reach (random access drops ~4x past ~64 GiB,
    # profiles/README.md), each shard then stays inside it
    est_bytes = table_capacity(states_est, vlen, args.bucket_words, args.load) * 4
    shards = args.shards or (1 if args.engine == "table" or est_bytes <= TLB_REACH
                             else -(-est_bytes // SHARD_BYTES))
    per = states_est // shards + (states_est >> 8 if shards > 1 else 0)
    cap = table_capacity(per, vlen, args.bucket_words, args.load)
    tcfg = TableConfig(bucket_words=args.bucket_words, num_hash_functions=args.hash_functions,
                       capacity_words=cap)
    cfg = ExploreConfig(table=tcfg, detect_deadlocks=True, probe_group=args.probe_group,
                        cache_slots=max(1, args.cache_slots), filter_log2=args.filter_log2,
                        dedup=args.dedup, dedup_set_log2=args.dedup_set_log2, state_digest=False,
                        pipeline=bool(args.pipeline))
    stream = torch.cuda.current_stream().cuda_stream
    from paper_1801_05857_b200.hashtable import slots_per_bucket
    spb0 = slots_per_bucket(args.bucket_words, vlen, "half" if args.bucket_words == 32 else "plain")
    status_bytes = cap // args.bucket_words * ((spb0 + 7) & ~7) * shards
    aux_bytes = int(states_est * (args.frontier_frac + args.inbox_frac) * 4 * vlen) if shards > 1 else \
        int(states_est * args.frontier_frac * 4 * vlen)
    # the per-slot status array (1 B per slot) only serves the claim / scan /
    # dump API; drop it when the table plus its buffers would not fit with it
    status = not args.no_status and \
        cap * 4 * shards + status_bytes + aux_bytes < 0.97 * torch.cuda.mem_get_info()[0]
    if shards == 1:
        ex = Explorer(net, cfg, stream=stream, status=status)
        total_slots = ex.table.total_slots
        spb = ex.table.slots_per_bucket
        nbk = ex.table.num_buckets
    else:
        from paper_1801_05857_b200.distributed import LocalShardExplorer
        front = int(states_est * args.frontier_frac / shards) + (1 << 20)
        inbox = int(states_est * args.inbox_frac / shards) + (1 << 20)
        # never more than what the tables and frontiers leave free
        left = torch.cuda.mem_get_info()[0] - cap * 4 * shards - status_bytes * status \
            - front * 4 * vlen * shards
        # the partitioned mode also holds a quarter-inbox buffer of first occurrences
        inbox = max(1 << 20, min(inbox, int(0.85 * left) // (4 * vlen * shards * (5 if args.dedup else 4) // 4)))
        ex = LocalShardExplorer(net, cfg, shards, inbox_capacity=inbox, frontier_capacity=front,
                                status=status, stream=stream)
        total_slots = sum(sh.table.total_slots for sh in ex.shards)
        spb = ex.shards[0].table.slots_per_bucket
        nbk = sum(sh.table.num_buckets for sh in ex.shards)
    table_bytes = nbk * (4 * args.bucket_words + (((spb + 7) & ~7) if status else 0))

    for _ in range(args.warmup):
        rep = ex.run()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            reps.append(ex.run())
        ev1.record()
        torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    rep = reps[-1]
    if cf:
        assert (rep.states, rep.transitions) == cf, (rep.states, rep.transitions, cf)
    assert rep.outcome == "COMPLETE", rep.outcome
    value = rep.states * args.steps / (ms / 1e3)

    # roofline of the level kernels, algorithmic bytes per step
    sbw = s_bw(args.bucket_words)
    alg_bytes = rep.transitions * sbw + rep.states * 12 * vlen
    level_ms = statistics.mean(r.level_ms for r in reps)
    achieved = alg_bytes / (level_ms / 1e3) / 1e9
    # probe-based bytes: the probes actually issued (self-loops are never
    # probed, block-cache hits skip theirs) plus the inbox round trip of
    # the successors routed to another shard
    routed = getattr(rep, "routed", 0) or 0
    probe_bytes = rep.probes * sbw + rep.states * 12 * vlen + routed * 8 * vlen
    traffic = None
    if TRAFFIC.exists():
        tr = json.loads(TRAFFIC.read_text())
        key = f"{args.workload}/bw{args.bucket_words}/shards{shards}"
        if key in tr:  # DRAM bytes of one exploration's level kernels (ncu, profiles/)
            traffic = tr[key]["bytes_per_step"]
    # set identity of the timed run: its digest against the golden one
    # (tests/golden/digests.json: the oracle's / the closed-form
    # enumeration of the reachable set, data only)
    digest = list(ex.digest())
    golden = json.loads(GOLDEN_DIGESTS.read_text()).get(args.workload, {}) if GOLDEN_DIGESTS.exists() else {}
    if golden.get("digest"):
        assert digest == golden["digest"], (digest, golden["digest"])
    ex.close()
    crosscheck = None
    if shards > 1 and args.crosscheck:
        # the same model on ONE table (the single-GPU engine): same set
        t0 = time.perf_counter()
        one = TableConfig(bucket_words=args.bucket_words, num_hash_functions=args.hash_functions,
                          capacity_words=table_capacity(states_est, vlen, args.bucket_words, args.load))
        ex1 = Explorer(net, ExploreConfig(table=one, detect_deadlocks=True, state_digest=False),
                       stream=stream, status=False)
        r1 = ex1.run()
        d1 = list(ex1.digest())
        ex1.close()
        assert (r1.states, r1.transitions, d1) == (rep.states, rep.transitions, digest), (r1, d1, digest)
        crosscheck = {"engine": "single table (gx_explore)", "states": r1.states, "transitions": r1.transitions,
                      "digest": d1, "equal": True, "seconds": time.perf_counter() - t0}

    # the random-access roofline R(g) on this GPU: a 32 GiB buffer (>> L2,
    # inside the TLB reach) and, for tables beyond the reach, the table size
    ra = random_access()
    table_gib = (table_bytes // shards) >> 30
    ra_table = None
    if table_gib > 48:
        from paper_1801_05857_b200.bench import random_access_roofline
        r128 = random_access_roofline(sbw, buffer_bytes=table_gib << 30)
        ra_table = {"buffer_gib": table_gib, "g": sbw, "gbs": r128["gbs"],
                    "accesses_per_s": r128["segments_per_sec"]}
    r_peak = ra_table["gbs"] if ra_table else ra[sbw]["gbs"]

    # e2e through the public API with host buffers
    torch.cuda.synchronize()
    e2e_times = []
    csr_bytes = None
    for i in range(args.e2e_steps + 1):
        t0 = time.perf_counter()
        if shards == 1:
            r = gx.explore(net, cfg)
        else:
            from paper_1801_05857_b200.distributed import explore_local_shards
            r = explore_local_shards(net, cfg, shards, inbox_capacity=inbox, frontier_capacity=front,
                                     status=status)
        dt = time.perf_counter() - t0
        if i:
            e2e_times.append(dt)
    from paper_1801_05857_b200.explore import DeviceNetwork
    dn = DeviceNetwork(net, scheme)
    csr_bytes = (dn.csr_bytes + 4 * vlen) * shards
    dn.close()
    e2e_value = r.states * len(e2e_times) / sum(e2e_times) if e2e_times else None

    cpu = None
    same = None
    hash_cpu = None
    if not args.no_cpu_baseline and rank == 0:
        cpu = cpu_reference(args.cpu_sample, 1, 0, tmp)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        # the GPU on the CPU's own sample: a same-workload pair
        gpu_same = single_table_rate(torch, args.cpu_sample, tmp)
        same = {"workload": args.cpu_sample, "gpu_states_per_sec": gpu_same["states_per_sec"],
                "cpu_states_per_sec": cpu["value"], "cpu_cores": cpu["cores"],
                "gpu_over_cpu": gpu_same["states_per_sec"] / cpu["value"],
                "gpu_engine": "single table, explore() engine", "digest_ok": gpu_same["digest_ok"]}
        if not args.no_hash_bench:
            hash_cpu = cpu_hash_baseline()

    line = {
        "metric": METRIC, "value": value, "unit": "states/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (generated model, exact state space)",
        "config": {
            "workload": f"configs[3] scaled token ring N={args.workload[4:]}" if args.workload.startswith("ring")
            else args.workload,
            "states": rep.states, "transitions": rep.transitions, "levels": rep.iterations - 1,
            "vector_words": vlen, "bucket_words": args.bucket_words,
            "hash_functions": args.hash_functions, "table_bytes": table_bytes,
            "block_cache_slots": args.cache_slots, "l2_filter_log2": args.filter_log2,
            "load_factor": rep.states / total_slots,
            "status_array": status,
            "l2_policy": "table re-zeroed every step; table >> 126 MB L2",
            "parallelism": "single GPU" if shards == 1 else
            f"single GPU, {shards} hash-owner shards (one per <= 80 GiB of table, probed one at a time; "
            "fused peer-routed levels)",
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": "k_level_staged" if shards == 1 else "k_level_routed + k_absorb",
                     "algorithmic_bytes_per_step": alg_bytes,
                     "kernel_ms_per_step": level_ms,
                     "bytes_model": "transitions*max(32,4*bw) + states*12*vlen (SURVEY §8(d))",
                     "probe_bytes_per_step": probe_bytes,
                     "probe_bytes_model": "probes*max(32,4*bw) + states*12*vlen + routed*8*vlen "
                                          "(probes actually issued; inbox write + read)",
                     "achieved_probe_based": probe_bytes / (level_ms / 1e3) / 1e9,
                     "frac_probe_based": probe_bytes / (level_ms / 1e3) / 1e9 / hbm_peak,
                     "random_access_gbs": r_peak,
                     "frac_of_random_access": achieved / r_peak,
                     "random_access": ra, "random_access_table_size": ra_table},
        "cpu_baseline": cpu,
        "same_workload_cpu_vs_gpu": same,
        "digest": {"value": digest, "golden": golden.get("digest"),
                   "golden_source": golden.get("source"), "equal": digest == golden.get("digest")},
        "engine_crosscheck": crosscheck,
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": csr_bytes,
                "d2h_bytes_per_step": 64 + 400 * vlen,
                "api": "paper_1801_05857_b200.explore(net, cfg) (allocates + frees the table)"
                if shards == 1 else "distributed.explore_local_shards (allocates + frees the shards)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "probes_per_step": rep.probes,
        "routed_per_step": routed,
        "step_breakdown_ms": {"level_kernels": level_ms,
                              "level_loop": statistics.mean(r.device_ms for r in reps) if shards == 1
                              else None,
                              "whole_step": ms / args.steps,
                              "max_frontier": rep.max_frontier},
    }
    if not args.no_hash_bench:
        line["hash_bench"] = {"fill_sweep": hash_sweep(ra), "duplication_sweep": duplication_sweep(ra),
                              "cpu_baseline": hash_cpu}
    if not args.no_extra:
        line["extra_workloads"] = extra_workloads(torch, tmp)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
