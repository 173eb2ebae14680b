"""ctypes front end of the C oracle (gx_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and CPU baseline for the
B200 engine.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
may import this module; the product package never does.

Parity is pinned against the real reference (ltsmc) through the golden
vectors in tests/golden/ (see tests/test_oracle_golden.py).

The model reader here is deliberately minimal and independent of the
product's parser (paper_1801_05857_b200/aut.py): it accepts the same
`.aut` / `par using ... end par` files (aut.py:93-164, 277-321 of the
reference) but reports no diagnostics.  Action names are interned into
global ids, "tau" folded into "i" (aut.py:30-31, 89-90).
"""

from __future__ import annotations

import ctypes as C
import os
import re
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

FOUND, INSERTED, TABLE_FULL = 0, 1, 2
EMPTY, CLAIMED, NEW, OLD = 0, 1, 2, 3
PLAIN, HALF = 0, 1
OUTCOMES = ("COMPLETE", "TABLE_FULL", "ITERATION_CAP")

_lib = None


def build(force: bool = False) -> Path:
    """Compile liboracle.so with the committed Makefile."""
    if force or not LIB_PATH.exists() or \
            LIB_PATH.stat().st_mtime < (HERE / "gx_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


class OrReport(C.Structure):
    _fields_ = [
        ("states", C.c_int64), ("transitions", C.c_int64), ("expanded", C.c_int64),
        ("iterations", C.c_int64), ("deadlocks_total", C.c_int64),
        ("outcome", C.c_int32), ("deadlocks_kept", C.c_int32),
        ("wall_time", C.c_double), ("cache_hits", C.c_int64), ("cache_lookups", C.c_int64),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB_PATH))
        P = C.POINTER
        u32p, i32p, i64p, u64p, u8p = (P(C.c_uint32), P(C.c_int32), P(C.c_int64),
                                       P(C.c_uint64), P(C.c_uint8))
        L.or_last_error.restype = C.c_char_p
        L.or_hash_constants.argtypes = [C.c_uint64, C.c_int, u64p, u64p, u64p]
        L.or_fold.restype = C.c_uint64
        L.or_fold.argtypes = [C.c_uint64, u32p, C.c_int]
        L.or_slots_per_bucket.argtypes = [C.c_int, C.c_int, C.c_int]
        L.or_table_create.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_int,
                                      P(C.c_void_p)]
        L.or_table_destroy.argtypes = [C.c_void_p]
        L.or_table_geometry.argtypes = [C.c_void_p, u64p, P(C.c_int), u64p]
        L.or_bucket_index.restype = C.c_uint64
        L.or_bucket_index.argtypes = [C.c_void_p, u32p, C.c_int]
        L.or_find_or_insert.argtypes = [C.c_void_p, u32p, i64p]
        L.or_find_or_insert_batch.argtypes = [C.c_void_p, u32p, C.c_uint64, u8p, i64p]
        L.or_claim_new.argtypes = [C.c_void_p, C.c_int64]
        L.or_scan_new.restype = C.c_int64
        L.or_scan_new.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, i64p, C.c_int64]
        L.or_occupancy.argtypes = [C.c_void_p, i64p, i64p]
        L.or_slot_status.argtypes = [C.c_void_p, C.c_int64]
        L.or_read_slot.argtypes = [C.c_void_p, C.c_int64, u32p]
        L.or_occupied_slots.restype = C.c_int64
        L.or_occupied_slots.argtypes = [C.c_void_p, i64p, u8p, u32p, C.c_int64]
        L.or_scheme_info.argtypes = [C.c_int, i32p, i32p, i32p, i32p]
        L.or_net_create.argtypes = [C.c_int, i32p, i32p, i32p, i32p, i32p, i32p, C.c_int, i32p,
                                    i32p, P(C.c_void_p)]
        L.or_net_destroy.argtypes = [C.c_void_p]
        L.or_net_vlen.argtypes = [C.c_void_p]
        L.or_expand.restype = C.c_int64
        L.or_expand.argtypes = [C.c_void_p, i32p, i32p, i32p, C.c_int64, i64p]
        L.or_explore.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int64,
                                 P(OrReport), u32p]
        L.or_bfs.argtypes = [C.c_void_p, C.c_int64, i64p, i64p, i64p, i64p]
        L.or_net_pack.argtypes = [C.c_void_p, i32p, u32p]
        L.or_net_unpack.argtypes = [C.c_void_p, u32p, i32p]
        L.or_probe_raw.argtypes = [C.c_uint64, C.c_int, C.c_uint64, u32p, C.c_int, u64p]
        L.or_py_tuple_hash.restype = C.c_int64
        L.or_py_tuple_hash.argtypes = [u32p, C.c_int]
        L.or_state_hash.restype = C.c_uint64
        L.or_state_hash.argtypes = [u32p, C.c_int]
        L.or_table_digest.argtypes = [C.c_void_p, C.c_int, u64p]
        L.or_ring_digest.argtypes = [C.c_int, C.c_int, u64p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _err() -> str:
    return lib().or_last_error().decode()


# ----------------------------------------------------------------- hashing

def hash_constants(seed: int, k: int):
    a = np.zeros(k, np.uint64)
    b = np.zeros(k, np.uint64)
    salt = np.zeros(1, np.uint64)
    lib().or_hash_constants(seed & (2**64 - 1), k, _ptr(a, C.c_uint64), _ptr(b, C.c_uint64),
                            _ptr(salt, C.c_uint64))
    return [(int(x), int(y)) for x, y in zip(a, b)], int(salt[0])


def fold(salt: int, p) -> int:
    arr = np.asarray(p, np.uint32)
    return int(lib().or_fold(salt, _ptr(arr, C.c_uint32), len(arr)))


def probe_raw(seed: int, k: int, num_buckets: int, p):
    arr = np.asarray(p, np.uint32)
    out = np.zeros(k, np.uint64)
    lib().or_probe_raw(seed & (2**64 - 1), k, num_buckets, _ptr(arr, C.c_uint32), len(arr),
                       _ptr(out, C.c_uint64))
    return [int(x) for x in out]


def slots_per_bucket(bw: int, vlen: int, layout: int) -> int:
    n = lib().or_slots_per_bucket(bw, vlen, layout)
    if n == 0:
        raise ValueError(_err())
    return n


def py_tuple_hash(p) -> int:
    arr = np.asarray(p, np.uint32)
    return int(lib().or_py_tuple_hash(_ptr(arr, C.c_uint32), len(arr)))


def state_hash(p) -> int:
    arr = np.ascontiguousarray(p, np.uint32)
    return int(lib().or_state_hash(_ptr(arr, C.c_uint32), len(arr)))


def ring_digest(n: int, threads: int = 0) -> tuple:
    """(count, sum, xor) digest of token ring N's reachable set, enumerated
    in closed form (gx_oracle.c or_ring_digest)."""
    out = np.zeros(3, np.uint64)
    if lib().or_ring_digest(n, threads or os.cpu_count() or 1, _ptr(out, C.c_uint64)):
        raise ValueError(_err())
    return int(out[0]), int(out[1]), int(out[2])


# -------------------------------------------------------------------- table

class Table:
    """Serial/atomic restatement of StateTable (hashtable.py:129-365)."""

    def __init__(self, bucket_words=32, num_hash_functions=8, capacity_words=1 << 22,
                 layout=None, seed=42, vector_length=1):
        if layout is None:
            layout = HALF if bucket_words == 32 else PLAIN
        elif isinstance(layout, str):
            layout = HALF if layout == "half" else PLAIN
        h = C.c_void_p()
        if lib().or_table_create(bucket_words, num_hash_functions, capacity_words, layout,
                                 seed & (2**64 - 1), vector_length, C.byref(h)):
            raise ValueError(_err())
        self._h = h
        self.vlen = vector_length
        nb = C.c_uint64()
        spb = C.c_int()
        ts = C.c_uint64()
        lib().or_table_geometry(h, C.byref(nb), C.byref(spb), C.byref(ts))
        self.num_buckets, self.slots_per_bucket, self.total_slots = nb.value, spb.value, ts.value
        self.num_hash_functions = num_hash_functions

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_table_destroy(self._h)
            self._h = None

    def bucket_index(self, p, i):
        arr = np.asarray(p, np.uint32)
        return int(lib().or_bucket_index(self._h, _ptr(arr, C.c_uint32), i))

    def probe_sequence(self, p):
        return [self.bucket_index(p, i) for i in range(self.num_hash_functions)]

    def find_or_insert(self, p):
        arr = np.ascontiguousarray(p, np.uint32)
        hd = C.c_int64()
        code = lib().or_find_or_insert(self._h, _ptr(arr, C.c_uint32), C.byref(hd))
        return code, hd.value

    def find_or_insert_batch(self, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, np.uint32).reshape(-1, self.vlen)
        n = keys.shape[0]
        codes = np.zeros(n, np.uint8)
        handles = np.zeros(n, np.int64)
        lib().or_find_or_insert_batch(self._h, _ptr(keys, C.c_uint32), n, _ptr(codes, C.c_uint8),
                                      _ptr(handles, C.c_int64))
        return codes, handles

    def claim_new(self, h):
        return bool(lib().or_claim_new(self._h, h))

    def scan_new(self, first, last):
        n = lib().or_scan_new(self._h, first, last, None, 0)
        out = np.zeros(max(n, 1), np.int64)
        lib().or_scan_new(self._h, first, last, _ptr(out, C.c_int64), n)
        return out[:n].tolist()

    def occupancy(self):
        o, n = C.c_int64(), C.c_int64()
        lib().or_occupancy(self._h, C.byref(o), C.byref(n))
        return o.value, n.value, (o.value / self.total_slots if self.total_slots else 0.0)

    def slot_status(self, h):
        return lib().or_slot_status(self._h, h)

    def read_slot(self, h):
        out = np.zeros(self.vlen, np.uint32)
        lib().or_read_slot(self._h, h, _ptr(out, C.c_uint32))
        return tuple(int(x) for x in out)

    def digest(self, words: int | None = None) -> tuple:
        """(count, sum, xor) set digest of the occupied slots (gx_table_digest)."""
        out = np.zeros(3, np.uint64)
        lib().or_table_digest(self._h, int(words or self.vlen), _ptr(out, C.c_uint64))
        return int(out[0]), int(out[1]), int(out[2])

    def occupied(self):
        """(handles, statuses, words[n, vlen]) in bucket-major order."""
        n = lib().or_occupied_slots(self._h, None, None, None, 0)
        hs = np.zeros(max(n, 1), np.int64)
        st = np.zeros(max(n, 1), np.uint8)
        ws = np.zeros((max(n, 1), self.vlen), np.uint32)
        lib().or_occupied_slots(self._h, _ptr(hs, C.c_int64), _ptr(st, C.c_uint8),
                                _ptr(ws, C.c_uint32), n)
        return hs[:n], st[:n], ws[:n]


# ------------------------------------------------------------ model reading

_TRANS = re.compile(r"^\((.*)\)$")


def _canon(name: str) -> str:
    return "i" if name in ("i", "tau") else name


def read_aut(text: str):
    """-> (nstates, initial, [(src, label, dst)])"""
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    head = lines[0][3:].strip()[1:-1].split(",")
    initial, _, nstates = (int(x) for x in head)
    trans = []
    for ln in lines[1:]:
        body = _TRANS.match(ln).group(1)
        src, _, rest = body.partition(",")
        mid, _, dst = rest.rpartition(",")
        lab = mid.strip()
        if len(lab) >= 2 and lab[0] == lab[-1] == '"':
            lab = lab[1:-1]
        trans.append((int(src), _canon(lab), int(dst)))
    return nstates, initial, trans


def read_exp(text: str):
    """-> ([process file], [([name or None per column], result)])"""
    text = "\n".join(ln.split("--", 1)[0] for ln in text.splitlines())
    toks = re.findall(r'"[^"]*"|\|\||->|\*|,|[^\s",*|]+', text)
    assert toks[:2] == ["par", "using"]
    i = 2
    rules = []
    while toks[i] != "in":
        cols = []
        while True:
            cols.append(None if toks[i] == "_" else _canon(toks[i]))
            i += 1
            if toks[i] == "*":
                i += 1
                continue
            assert toks[i] == "->"
            i += 1
            break
        rules.append((cols, _canon(toks[i])))
        i += 1
        if toks[i] == ",":
            i += 1
    i += 1
    files = []
    while True:
        f = toks[i]
        files.append(f[1:-1] if f.startswith('"') else f)
        i += 1
        if toks[i] == "||":
            i += 1
            continue
        break
    return files, rules


class Net:
    """Network handle for the C oracle, built from raw automata + rules."""

    def __init__(self, procs, rules):
        # procs: [(nstates, initial, [(src, name, dst)])]; rules: [([name|None], result)]
        names: dict[str, int] = {}

        def gid(s):
            if s not in names:
                names[s] = len(names)
            return names[s]

        nstates, initial, ntrans, trans, nlabels, labname = [], [], [], [], [], []
        for ns, ini, tr in procs:
            local: dict[str, int] = {}
            for src, lab, dst in tr:
                if lab not in local:
                    local[lab] = len(local)
                trans += [src, local[lab], dst]
            nstates.append(ns)
            initial.append(ini)
            ntrans.append(len(tr))
            nlabels.append(len(local))
            labname += [gid(l) for l in sorted(local, key=local.get)]
        P = len(procs)
        cols, res = [], []
        for c, r in rules:
            cols += [-1 if x is None else gid(x) for x in c]
            res.append(gid(r))
        self.nproc = P
        self.nstates = nstates
        self.initial = tuple(initial)
        self.action_names = names
        arr = lambda v: np.ascontiguousarray(np.asarray(v if v else [0], np.int32))
        self._keep = [arr(nstates), arr(initial), arr(ntrans), arr(trans), arr(nlabels),
                      arr(labname), arr(cols), arr(res)]
        k = self._keep
        h = C.c_void_p()
        if lib().or_net_create(P, *[_ptr(x, C.c_int32) for x in k[:6]], len(rules),
                               _ptr(k[6], C.c_int32), _ptr(k[7], C.c_int32), C.byref(h)):
            raise ValueError(_err())
        self._h = h
        self.vlen = lib().or_net_vlen(h)

    @classmethod
    def from_file(cls, path):
        path = Path(path)
        files, rules = read_exp(path.read_text())
        procs = []
        for f in files:
            p = Path(f)
            if not p.is_absolute():
                p = path.parent / p
            procs.append(read_aut(p.read_text()))
        return cls(procs, rules)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_net_destroy(self._h)
            self._h = None

    def expand(self, s, cap=4096):
        s = np.asarray(s, np.int32)
        acts = np.zeros(cap, np.int32)
        tgts = np.zeros((cap, self.nproc), np.int32)
        cnt = C.c_int64()
        n = lib().or_expand(self._h, _ptr(s, C.c_int32), _ptr(acts, C.c_int32),
                            _ptr(tgts, C.c_int32), cap, C.byref(cnt))
        inv = {v: k for k, v in self.action_names.items()}
        succ = [(inv[int(acts[i])], tuple(int(x) for x in tgts[i])) for i in range(min(n, cap))]
        return succ, cnt.value

    def pack(self, s):
        s = np.asarray(s, np.int32)
        out = np.zeros(self.vlen, np.uint32)
        lib().or_net_pack(self._h, _ptr(s, C.c_int32), _ptr(out, C.c_uint32))
        return tuple(int(x) for x in out)

    def unpack(self, p):
        p = np.asarray(p, np.uint32)
        out = np.zeros(self.nproc, np.int32)
        if lib().or_net_unpack(self._h, _ptr(p, C.c_uint32), _ptr(out, C.c_int32)):
            raise ValueError("corrupt packed state")
        return tuple(int(x) for x in out)

    def bfs(self, max_states=0):
        s, t, lv, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        rc = lib().or_bfs(self._h, max_states, C.byref(s), C.byref(t), C.byref(lv), C.byref(d))
        if rc:
            raise RuntimeError(f"product exceeds max_states={max_states}")
        return {"states": s.value, "transitions": t.value, "levels": lv.value, "deadlocks": d.value}


@dataclass
class OracleRun:
    states: int
    transitions: int
    deadlocks: tuple  # sorted composite states (<= 100 recorded)
    deadlocks_total: int
    expanded: int
    iterations: int
    outcome: str
    wall_time: float
    table: Table

    def dump_states(self) -> str:
        """Canonical dump (statevec.py:93-100)."""
        _, _, words = self.table.occupied()
        rows = sorted(tuple(int(x) for x in r) for r in words)
        return "".join(" ".join(f"{w:08x}" for w in r) + "\n" for r in rows) if rows else "\n"

    def dump_table(self) -> str:
        """CSV as explore.py:379-383."""
        hs, st, ws = self.table.occupied()
        spb = self.table.slots_per_bucket
        out = ["bucket,slot,status,words\n"]
        for h, s, w in zip(hs, st, ws):
            out.append(f"{int(h) // spb},{int(h) % spb},{'NEW' if s == NEW else 'OLD'},"
                       + " ".join(f"{int(x):08x}" for x in w) + "\n")
        return "".join(out)


def explore(net: Net, bucket_words=32, num_hash_functions=8, capacity_words=1 << 22, layout=None,
            seed=42, workers=1, cache_slots=4096, detect_deadlocks=False, max_iterations=None):
    """explore.py:300-395 restated (W=1 is exact, including placement)."""
    t = Table(bucket_words, num_hash_functions, capacity_words, layout, seed, net.vlen)
    rep = OrReport()
    dl = np.zeros((100, net.vlen), np.uint32)
    if lib().or_explore(net._h, t._h, workers, cache_slots, int(detect_deadlocks),
                        int(max_iterations or 0), C.byref(rep), _ptr(dl, C.c_uint32)):
        raise ValueError(_err())
    dls = tuple(sorted(net.unpack(dl[i]) for i in range(rep.deadlocks_kept)))
    return OracleRun(rep.states, rep.transitions, dls, rep.deadlocks_total, rep.expanded,
                     rep.iterations, OUTCOMES[rep.outcome], rep.wall_time, t)
