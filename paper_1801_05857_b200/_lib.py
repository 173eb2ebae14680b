"""ctypes binding of libgx.so (include/gx.h).

The shared library is built in-tree (paper_1801_05857_b200/libgx.so, see
build.py).  There is no fallback: if it is missing or no CUDA device is
usable, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
# GX_LIB (developer knob): load an alternative build of libgx.so, e.g. a
# variant compiled with other tile constants for an A/B sweep
LIB_PATH = Path(os.environ["GX_LIB"]) if os.environ.get("GX_LIB") else HERE / "libgx.so"

GX_OK, GX_EINPUT, GX_ETABLE_FULL, GX_EINTERNAL = 0, 1, 2, 3


class TableCfg(C.Structure):
    _fields_ = [("bucket_words", C.c_int32), ("num_hash_functions", C.c_int32),
                ("capacity_words", C.c_uint64), ("layout", C.c_int32),
                ("vector_length", C.c_int32), ("seed", C.c_uint64),
                ("mark_word", C.c_int32), ("mark_bit", C.c_int32),
                ("flags", C.c_int32), ("reserved", C.c_int32)]


class NetworkCsr(C.Structure):
    _fields_ = [("nproc", C.c_uint32), ("nrules", C.c_uint32), ("vlen", C.c_uint32),
                ("reserved", C.c_uint32)] + [
        (f, t) for name in ("proc", "qtab", "im_dst", "trig", "rules", "parts", "rq", "rdst", "dedup")
        for f, t in ((name, C.POINTER(C.c_uint32)), ("n_" + name, C.c_uint64))
    ] + [("initial", C.POINTER(C.c_uint32))]


class ExploreCfg(C.Structure):
    _fields_ = [("detect_deadlocks", C.c_int32), ("filter_log2", C.c_int32),
                ("max_iterations", C.c_int64), ("frontier_capacity", C.c_uint64),
                ("probe_group", C.c_int32), ("cache_slots", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("states", C.c_uint64), ("transitions", C.c_uint64), ("expanded", C.c_uint64),
                ("iterations", C.c_uint64), ("deadlocks_total", C.c_uint64),
                ("outcome", C.c_int32), ("deadlocks_kept", C.c_int32),
                ("device_ms", C.c_double), ("levels_launched", C.c_uint64),
                ("max_frontier", C.c_uint64), ("kernels", C.c_uint64),
                ("level_ms", C.c_double), ("probes", C.c_uint64)]


class GxError(RuntimeError):
    """CUDA / internal failure inside libgx (reference CLI exit code 3)."""


_lib = None

# symbol -> (restype, argtypes)
_P = C.POINTER
_u32p, _i32p, _u64p, _i64p, _u8p, _vp = (_P(C.c_uint32), _P(C.c_int32), _P(C.c_uint64),
                                         _P(C.c_int64), _P(C.c_uint8), C.c_void_p)
SIGNATURES = {
    "gx_table_create": (C.c_int, [_P(TableCfg), _vp, _P(_vp)]),
    "gx_table_destroy": (C.c_int, [_vp]),
    "gx_table_clear": (C.c_int, [_vp]),
    "gx_table_geometry": (C.c_int, [_vp, _u64p, _i32p, _u64p]),
    "gx_table_hash_constants": (C.c_int, [_vp, _u64p, _u64p, _u64p]),
    "gx_table_mode": (C.c_int, [_vp]),
    "gx_find_or_put": (C.c_int, [_vp, _u32p, C.c_uint64, _u8p, _i64p, C.c_int32]),
    "gx_find_or_put_device": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, _u64p, _u64p]),
    "gx_find_or_put_timed": (C.c_int, [_vp, _u32p, C.c_uint64, _u8p, _P(C.c_double)]),
    "gx_claim_new": (C.c_int, [_vp, _i64p, C.c_uint64, _u8p]),
    "gx_scan_new": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _i64p, C.c_uint64, _u64p]),
    "gx_occupancy": (C.c_int, [_vp, _u64p, _u64p]),
    "gx_read_slots": (C.c_int, [_vp, _i64p, C.c_uint64, _u8p, _u32p]),
    "gx_dump": (C.c_int, [_vp, _i64p, _u8p, _u32p, C.c_uint64, _u64p]),
    "gx_table_digest": (C.c_int, [_vp, C.c_int32, _u64p]),
    "gx_dump_sorted": (C.c_int, [_vp, C.c_int32, _u32p, C.c_uint64, _u64p]),
    "gx_net_create": (C.c_int, [_P(NetworkCsr), _vp, _P(_vp)]),
    "gx_net_destroy": (C.c_int, [_vp]),
    "gx_expand": (C.c_int, [_vp, _u32p, C.c_uint64, _u64p, _u32p, _u32p, C.c_uint64, _u64p]),
    "gx_explore": (C.c_int, [_vp, _vp, _P(ExploreCfg), _P(Report), _u32p]),
    "gx_expand_route": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int32, _vp, C.c_uint64, _vp, _vp,
                                  _u64p, _u64p, C.c_int32]),
    "gx_net_deadlocks": (C.c_int, [_vp, _u32p, C.c_uint64, _u64p]),
    "gx_insert_append": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64, _u64p, _i32p]),
    "gx_owner_of": (C.c_int, [_vp, _u32p, C.c_uint64, C.c_int32, _i32p]),
    "gx_bench_find_or_put": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32,
                                       _P(C.c_double), _u64p, _u64p, _u64p]),
    "gx_bench_find_or_put_rows": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_int32, C.c_int32, _P(C.c_double), _u64p, _u64p,
                                            _u64p, _u64p]),
    "gx_random_access_bench": (C.c_int, [C.c_uint64, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                         _P(C.c_double), _P(C.c_double)]),
    "gx_shard_create": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_uint64, C.c_uint64, C.c_int32,
                                  C.c_int32, _P(_vp)]),
    "gx_shard_destroy": (C.c_int, [_vp]),
    "gx_shard_ipc_handle": (C.c_int, [_vp, _u8p]),
    "gx_shard_connect": (C.c_int, [_vp, _u8p]),
    "gx_shard_connect_local": (C.c_int, [_P(_vp), C.c_int32]),
    "gx_shard_link": (C.c_int, [_vp, _vp]),
    "gx_shard_begin": (C.c_int, [_vp, C.c_int32, C.c_int32, _i32p]),
    "gx_shard_expand": (C.c_int, [_vp]),
    "gx_shard_absorb": (C.c_int, [_vp, _u64p]),
    "gx_shard_expand_range": (C.c_int, [_vp, C.c_uint64, C.c_uint64]),
    "gx_shard_absorb_chunk": (C.c_int, [_vp]),
    "gx_shard_set_mode": (C.c_int, [_vp, C.c_int32, C.c_int32]),
    "gx_shard_set_pipeline": (C.c_int, [_vp, C.c_int32]),
    "gx_shard_bench_route": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_uint64,
                                       C.c_uint64]),
    "gx_shard_bench_result": (C.c_int, [_vp, _u64p, _P(C.c_double)]),
    "gx_shard_set_partitions": (C.c_int, [_vp, C.c_uint32]),
    "gx_shard_chunk_status": (C.c_int, [_vp, _u64p]),
    "gx_shard_rollback": (C.c_int, [_vp]),
    "gx_shard_end_level": (C.c_int, [_vp, _u64p]),
    "gx_shard_frontier": (C.c_int, [_vp, _u64p]),
    "gx_shard_finish": (C.c_int, [_vp, _P(Report), _u32p]),
    "gx_random_access_bench_alloc": (C.c_int, [C.c_uint64, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                               C.c_int32, _P(C.c_double), _P(C.c_double), _u64p]),
    "gx_last_error": (C.c_char_p, []),
    "gx_kernel_launches": (C.c_uint64, []),
    "gx_device_info": (C.c_int, [_i32p, _u64p, _u64p]),
    "gx_sync": (C.c_int, [_vp]),
}


def lib():
    """Load libgx.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c "
                              "'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().gx_last_error().decode(errors="replace")


def check(rc: int):
    if rc == GX_OK:
        return
    msg = last_error()
    if rc == GX_EINPUT:
        raise ValueError(msg)
    raise GxError(f"libgx error {rc}: {msg}")


def ptr(a: np.ndarray, ctype=C.c_uint32):
    return a.ctypes.data_as(C.POINTER(ctype))


def kernel_launches() -> int:
    return int(lib().gx_kernel_launches())
