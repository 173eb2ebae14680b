"""Bit-packing of composite states into vectors of u32 words -- the unit the
device table stores -- and the canonical state dump.

API and layout follow /root/reference/pkg/src/ltsmc/statevec.py
(`scheme_for_sizes` :41, `pack` :69, `unpack` :79, `format_packed` :93,
`dump_states` :98): field i has max(1, bit_length(n_i - 1)) bits, fields are
placed from bit 0 of word 0 upward, a field that would cross a word
boundary starts the next word, padding is zero and the all-zero vector is
a valid state.  `mark_bit` is new: it picks the spare high bit the B200
table uses as its in-band "occupied" flag ("State table").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

WORD_BITS = 32
MAX_VECTOR_WORDS = 16


class PackingError(ValueError):
    pass


@dataclass(frozen=True)
class PackingScheme:
    widths: tuple
    num_states: tuple
    word_index: tuple
    shift: tuple
    total_bits: int
    vector_length: int


def scheme_for_sizes(sizes) -> PackingScheme:
    sizes = tuple(int(n) for n in sizes)
    widths = tuple(max(1, (n - 1).bit_length()) for n in sizes)
    words, shifts = [], []
    w_idx, fill = 0, 0
    for w in widths:
        if fill + w > WORD_BITS:
            w_idx, fill = w_idx + 1, 0
        words.append(w_idx)
        shifts.append(fill)
        fill += w
    vlen = w_idx + 1
    if vlen > MAX_VECTOR_WORDS:
        raise PackingError(f"state vector too wide: {vlen} words exceeds {MAX_VECTOR_WORDS}")
    return PackingScheme(widths=widths, num_states=sizes, word_index=tuple(words),
                         shift=tuple(shifts), total_bits=sum(widths), vector_length=vlen)


def make_scheme(net) -> PackingScheme:
    return scheme_for_sizes(p.num_states for p in net.processes)


def pack(scheme: PackingScheme, s) -> tuple:
    out = [0] * scheme.vector_length
    for v, w, sh in zip(s, scheme.word_index, scheme.shift):
        out[w] |= v << sh
    return tuple(out)


def unpack(scheme: PackingScheme, p) -> tuple:
    vals = []
    for i, (w, sh, width) in enumerate(zip(scheme.word_index, scheme.shift, scheme.widths)):
        v = (p[w] >> sh) & ((1 << width) - 1)
        if v >= scheme.num_states[i]:
            raise PackingError(f"corrupt packed state: field {i} decodes to {v} >= "
                               f"{scheme.num_states[i]}")
        vals.append(v)
    return tuple(vals)


def unpack_array(scheme: PackingScheme, words: np.ndarray) -> np.ndarray:
    """Vectorised unpack of an (n, vlen) u32 array -> (n, nproc) int64."""
    words = np.asarray(words, np.uint64).reshape(-1, scheme.vector_length)
    out = np.empty((words.shape[0], len(scheme.widths)), np.int64)
    for i, (w, sh, width) in enumerate(zip(scheme.word_index, scheme.shift, scheme.widths)):
        out[:, i] = (words[:, w] >> np.uint64(sh)) & np.uint64((1 << width) - 1)
    return out


def format_packed(p) -> str:
    return " ".join(f"{int(w):08x}" for w in p)


def dump_states(packed_states) -> str:
    return "\n".join(format_packed(p) for p in sorted(packed_states)) + "\n"


def dump_states_array(words: np.ndarray, presorted: bool = False) -> str:
    """dump_states for an (n, vlen) u32 array: sorted lexicographically over
    the words (on the host unless `presorted`, e.g. by gx_dump_sorted)."""
    words = np.asarray(words, np.uint32).reshape(len(words), -1) if len(words) else words
    if len(words) == 0:
        return "\n"
    srt = words if presorted else words[np.lexsort(words.T[::-1])]
    hexes = [np.char.zfill(np.char.mod("%x", srt[:, j]), 8) for j in range(srt.shape[1])]
    lines = hexes[0]
    for h in hexes[1:]:
        lines = np.char.add(np.char.add(lines, " "), h)
    return "\n".join(lines.tolist()) + "\n"


def device_vlen(scheme: PackingScheme, pad: bool = True) -> int:
    """Words per state on the device: a 3-word state is stored padded to 4
    words (the padding word is zero), so the exploration table can use the
    in-band mode with one 128-bit CAS per insert instead of the status-byte
    protocol.  The state set is unchanged; the table holds vlen-4 slots."""
    v = scheme.vector_length
    return 4 if (pad and v == 3) else v


def mark_bit(scheme: PackingScheme, vlen: int | None = None):
    """(word, bit) of a bit no packed state ever sets -- the top bit of the
    word with the most unused bits -- or None if every word is full.  With
    device padding (vlen > the scheme's), the always-zero padding word's top
    bit."""
    if vlen is not None and vlen > scheme.vector_length:
        return vlen - 1, WORD_BITS - 1
    used = [0] * scheme.vector_length
    for w, sh, width in zip(scheme.word_index, scheme.shift, scheme.widths):
        used[w] = max(used[w], sh + width)
    best = min(range(scheme.vector_length), key=lambda w: (used[w], w))
    if used[best] >= WORD_BITS:
        return None
    return best, WORD_BITS - 1


# ------------------------------------------------------------ set digest
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def state_hashes(words: np.ndarray) -> np.ndarray:
    """Per-state hash of packed vectors (n, vlen) u32 (include/gx.h
    gx_table_digest): h = 0x6A09E667F3BCC908 ^ vlen, then h = mix64(h ^ w)
    for each word."""
    words = np.asarray(words, np.uint32)
    words = words.reshape(len(words), -1) if words.ndim != 2 else words
    h = np.full(len(words), 0x6A09E667F3BCC908 ^ words.shape[1], np.uint64)
    with np.errstate(over="ignore"):
        for j in range(words.shape[1]):
            h = _mix64(h ^ words[:, j].astype(np.uint64))
    return h


def state_digest(words: np.ndarray) -> tuple:
    """(count, sum mod 2^64, xor) of state_hashes: the order-independent
    multiset digest of a set of packed states."""
    h = state_hashes(words)
    if len(h) == 0:
        return 0, 0, 0
    s = int(np.sum(h, dtype=np.uint64))
    x = int(np.bitwise_xor.reduce(h))
    return len(h), s, x

