"""The state table: a fixed-capacity closed-hashing set of packed vectors in
B200 HBM, with K-function first-fit probing over buckets of 4/8/16/32 words.

Python surface of /root/reference/pkg/src/ltsmc/hashtable.py (constants
:35-51, `TableConfig` :75-86, `slots_per_bucket` :89-111, `hash_constants`
:123-126, `StateTable` :129-365, `TableFullError` :71); every operation
runs on the device through libgx (include/gx.h).  `find_or_insert` of a
single vector is kept for API compatibility; batches go through
`find_or_insert_batch` (one kernel launch, device-parallel).

Table-full is a value (TABLE_FULL), never an exception, as in the
reference (hashtable.py:5-7).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TableCfg, check, lib, ptr

EMPTY = 0
CLAIMED = 1
OCCUPIED_NEW = 2
OCCUPIED_OLD = 3

FOUND = 0
INSERTED = 1
TABLE_FULL = 2

HALF_BUCKET = "half"
PLAIN = "plain"

BUCKET_WORD_CHOICES = (4, 8, 16, 32)
DEFAULT_SEED = 42
DEFAULT_CAPACITY_WORDS = 1 << 22

MASK64 = (1 << 64) - 1


class TableFullError(RuntimeError):
    """Raised by callers that treat a full table as unrecoverable."""


@dataclass(frozen=True)
class TableConfig:
    bucket_words: int = 32
    num_hash_functions: int = 8
    capacity_words: int = DEFAULT_CAPACITY_WORDS
    layout: str | None = None
    seed: int = DEFAULT_SEED

    def resolved_layout(self) -> str:
        if self.layout is not None:
            return self.layout
        return HALF_BUCKET if self.bucket_words == 32 else PLAIN


def slots_per_bucket(bucket_words: int, vector_length: int, layout: str) -> int:
    if bucket_words <= 0 or vector_length <= 0:
        raise ValueError("bucket_words and vector_length must be positive")
    if layout == HALF_BUCKET:
        if bucket_words % 2:
            raise ValueError("half-bucket layout requires an even bucket size")
        n = 2 * ((bucket_words // 2) // vector_length)
    elif layout == PLAIN:
        n = bucket_words // vector_length
    else:
        raise ValueError(f"unknown layout {layout!r}")
    if n == 0:
        raise ValueError(f"vector too long for bucket: {vector_length} words in a "
                         f"{bucket_words}-word bucket ({layout})")
    return n


def _splitmix(x: int):
    while True:
        x = (x + 0x9E3779B97F4A7C15) & MASK64
        z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def hash_constants(seed: int, count: int) -> tuple:
    g = _splitmix(seed & MASK64)
    return tuple((next(g) | 1, next(g)) for _ in range(count))


class StateTable:
    """Device-resident concurrent set of fixed-length word vectors.

    `mark=(word, bit)` declares a bit no key will ever set (a spare bit of
    the packing scheme); the table then inserts with one CAS per key and
    probes only data sectors.  Without it every key pattern is allowed and
    the claim/publish status protocol of the reference is used.
    `status=False` (in-band tables only) drops the per-slot status array
    for exploration-only tables: 12.5% less memory at bw 32 / vlen 2; the
    claim / scan / dump methods then raise ValueError.
    """

    def __init__(self, config: TableConfig, vector_length: int, mark=None, stream=None,
                 status: bool = True):
        if config.bucket_words not in BUCKET_WORD_CHOICES:
            raise ValueError(f"bucket_words must be one of {BUCKET_WORD_CHOICES}, "
                             f"got {config.bucket_words}")
        if config.num_hash_functions < 1:
            raise ValueError("need at least one hash function")
        layout = config.resolved_layout()
        spb = slots_per_bucket(config.bucket_words, vector_length, layout)
        nb = config.capacity_words // config.bucket_words
        if nb < config.num_hash_functions:
            raise ValueError(f"capacity_words {config.capacity_words} gives {nb} buckets, "
                             f"fewer than {config.num_hash_functions} hash functions")
        self.config = config
        self.layout = layout
        self.vector_length = vector_length
        self.num_buckets = nb
        self.slots_per_bucket = spb
        self.total_slots = nb * spb
        self.mark = mark
        self.hash_constants = hash_constants(config.seed, config.num_hash_functions)
        self._fold_salt = next(_splitmix((config.seed ^ 0xA5A5A5A5A5A5A5A5) & MASK64))
        cfg = TableCfg(config.bucket_words, config.num_hash_functions, config.capacity_words,
                       1 if layout == HALF_BUCKET else 0, vector_length, config.seed & MASK64,
                       mark[0] if mark else -1, mark[1] if mark else 0,
                       0 if status else 1, 0)  # GX_TABLE_NO_STATUS: exploration-only table
        h = C.c_void_p()
        check(lib().gx_table_create(C.byref(cfg), stream, C.byref(h)))
        self._h = h
        self.mode = "mark" if lib().gx_table_mode(h) == 0 else "status"
        self._mark_mask = None
        if mark is not None and self.mode == "mark":
            m = np.zeros(vector_length, np.uint32)
            m[mark[0]] = 1 << mark[1]
            self._mark_mask = m

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().gx_table_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def clear(self):
        check(lib().gx_table_clear(self._h))

    # --- hashing (host restatement of the device formulas, for inspection)

    def fold(self, p) -> int:
        h = self._fold_salt
        for w in p:
            h = ((h ^ int(w)) * 0x9E3779B97F4A7C15) & MASK64
            h ^= h >> 29
        return h

    def bucket_index(self, p, i: int) -> int:
        assert 0 <= i < self.config.num_hash_functions, "hash function index out of range"
        a, b = self.hash_constants[i]
        return ((a * self.fold(p) + b) & MASK64) % self.num_buckets

    def probe_sequence(self, p) -> list:
        return [self.bucket_index(p, i) for i in range(self.config.num_hash_functions)]

    def device_hash_constants(self):
        k = self.config.num_hash_functions
        a = np.zeros(k, np.uint64)
        b = np.zeros(k, np.uint64)
        s = np.zeros(1, np.uint64)
        check(lib().gx_table_hash_constants(self._h, ptr(a, C.c_uint64), ptr(b, C.c_uint64),
                                            ptr(s, C.c_uint64)))
        return [(int(x), int(y)) for x, y in zip(a, b)], int(s[0])

    # --- core operations

    def _keys(self, keys) -> np.ndarray:
        arr = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, self.vector_length))
        if arr.size and (arr.max() > 0xFFFFFFFF):
            raise ValueError("vector words must be 32-bit")
        arr = arr.astype(np.uint32)
        if self._mark_mask is not None and arr.size and (arr & self._mark_mask).any():
            raise ValueError("a key sets the table's reserved mark bit")
        return arr

    def find_or_insert_batch(self, keys, serial: bool = False):
        """FINDORPUT of n vectors -> (codes u8[n], handles i64[n]).  Equal
        vectors in one batch agree on one handle and exactly one is
        INSERTED.  serial=True reproduces single-threaded placement."""
        arr = self._keys(keys)
        n = arr.shape[0]
        codes = np.zeros(n, np.uint8)
        handles = np.zeros(n, np.int64)
        if n:
            check(lib().gx_find_or_put(self._h, ptr(arr), n, ptr(codes, C.c_uint8),
                                       ptr(handles, C.c_int64), 1 if serial else 0))
        return codes, handles

    def find_or_insert(self, p) -> tuple:
        codes, handles = self.find_or_insert_batch([tuple(p)], serial=True)
        return int(codes[0]), int(handles[0])

    def claim_new_batch(self, handles) -> np.ndarray:
        hs = np.ascontiguousarray(np.asarray(handles, np.int64).reshape(-1))
        out = np.zeros(hs.shape[0], np.uint8)
        if hs.size:
            check(lib().gx_claim_new(self._h, ptr(hs, C.c_int64), hs.size, ptr(out, C.c_uint8)))
        return out.astype(bool)

    def claim_new(self, handle: int) -> bool:
        return bool(self.claim_new_batch([handle])[0])

    def scan_new(self, first_bucket: int, last_bucket: int) -> list:
        return self.scan_new_array(first_bucket, last_bucket).tolist()

    def scan_new_array(self, first_bucket: int, last_bucket: int) -> np.ndarray:
        cnt = C.c_uint64()
        check(lib().gx_scan_new(self._h, first_bucket, last_bucket, None, 0, C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), np.int64)
        if cnt.value:
            check(lib().gx_scan_new(self._h, first_bucket, last_bucket, ptr(out, C.c_int64),
                                    cnt.value, C.byref(cnt)))
        return out[:cnt.value]

    def occupancy(self) -> tuple:
        occ, new = C.c_uint64(), C.c_uint64()
        check(lib().gx_occupancy(self._h, C.byref(occ), C.byref(new)))
        o = occ.value
        return o, new.value, (o / self.total_slots if self.total_slots else 0.0)

    # --- inspection

    def read_slots(self, handles):
        hs = np.ascontiguousarray(np.asarray(handles, np.int64).reshape(-1))
        st = np.zeros(hs.size, np.uint8)
        words = np.zeros((hs.size, self.vector_length), np.uint32)
        if hs.size:
            check(lib().gx_read_slots(self._h, ptr(hs, C.c_int64), hs.size, ptr(st, C.c_uint8),
                                      ptr(words)))
        return st, words

    def slot_status(self, handle: int) -> int:
        return int(self.read_slots([handle])[0][0])

    def read_slot(self, handle: int) -> tuple:
        return tuple(int(w) for w in self.read_slots([handle])[1][0])

    def dump_arrays(self):
        """(handles, statuses, words[n, vlen]) of all published slots,
        bucket-major."""
        cnt = C.c_uint64()
        check(lib().gx_dump(self._h, None, None, None, 0, C.byref(cnt)))
        n = cnt.value
        hs = np.zeros(max(n, 1), np.int64)
        st = np.zeros(max(n, 1), np.uint8)
        ws = np.zeros((max(n, 1), self.vector_length), np.uint32)
        if n:
            check(lib().gx_dump(self._h, ptr(hs, C.c_int64), ptr(st, C.c_uint8), ptr(ws), n,
                                C.byref(cnt)))
        return hs[:n], st[:n], ws[:n]

    def digest(self, words: int | None = None) -> tuple:
        """(count, sum, xor) of the per-state hashes of the occupied slots'
        first `words` words (include/gx.h gx_table_digest); order- and
        placement-independent, so shards and engines compare exactly."""
        out = np.zeros(3, np.uint64)
        check(lib().gx_table_digest(self._h, int(words or self.vector_length), ptr(out, C.c_uint64)))
        return int(out[0]), int(out[1]), int(out[2])

    def sorted_vectors(self, words: int | None = None) -> np.ndarray:
        """The occupied slots' first `words` words, sorted lexicographically
        on the device (gx_dump_sorted): dump_states' order."""
        w = int(words or self.vector_length)
        cnt = C.c_uint64()
        check(lib().gx_dump_sorted(self._h, w, None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), w), np.uint32)
        if cnt.value:
            check(lib().gx_dump_sorted(self._h, w, ptr(out), cnt.value, C.byref(cnt)))
        return out[:cnt.value]

    def occupied_vectors(self) -> list:
        return [tuple(int(x) for x in row) for row in self.dump_arrays()[2]]

    def dump_rows(self):
        names = {OCCUPIED_NEW: "NEW", OCCUPIED_OLD: "OLD"}
        hs, st, ws = self.dump_arrays()
        spb = self.slots_per_bucket
        for h, s, w in zip(hs, st, ws):
            yield int(h) // spb, int(h) % spb, names[int(s)], tuple(int(x) for x in w)
