"""Synchronous product of a network of LTSs, and its flattening into the
compact CSR the B200 successor kernel reads.

API mirrors /root/reference/pkg/src/ltsmc/network.py: `SyncRule` :28,
`Network` :43, `build_network` :65, `expand` :184, `successors` :241,
`is_deadlock` :247, `load_network` :252, `NetworkError` :25.

Semantics (network.py:65-181): a label of process i that appears in any
rule column i is synchronised and never fires alone (even when that rule
is disabled because another column names an unknown label); all other
labels are independent.  Network action ids: rule results in rule order,
then independent labels in (process, label id) order, deduplicated by
name.

`expand`/`successors`/`is_deadlock` are per-state point queries kept for
API compatibility (action ids included); exploration never calls them --
it runs the device kernels on the CSR produced by `to_csr`.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from itertools import product
from pathlib import Path

import numpy as np

from .aut import INTERNAL_ACTION, Lts, NetworkDescription, parse_aut, parse_network

CompositeState = tuple


class NetworkError(ValueError):
    """A description and its automata do not fit together."""


@dataclass(frozen=True)
class SyncRule:
    participants: tuple  # label id per process, None when absent
    result: int          # network action id
    enabled: bool = True


@dataclass(frozen=True)
class Network:
    processes: tuple
    rules: tuple
    actions: tuple
    independent: tuple
    # per process, per local state: ((action id, dst), ...) distinct, file order
    indep_moves: tuple = field(repr=False, default=())
    # per rule: None (disabled) or ((process, per-state dst tuples), ...)
    rule_moves: tuple = field(repr=False, default=())

    @property
    def initial(self) -> CompositeState:
        return tuple(p.initial for p in self.processes)

    def action_id(self, name: str):
        return self.actions.index(name) if name in self.actions else None


def max_successors(net: Network) -> int:
    """An upper bound on the successors of any composite state: every
    process's largest independent-move list plus every enabled rule's
    largest cartesian product (network.py expand() semantics).  Sizes the
    sharded engine's frontier chunks so no inbox can overflow."""
    bound = sum(max((len(m) for m in per), default=0) for per in net.indep_moves)
    for moves in net.rule_moves:
        if moves is None:
            continue
        prod = 1
        for _proc, per_state in moves:
            prod *= max((len(d) for d in per_state), default=0)
        bound += prod
    return max(bound, 1)


def build_network(desc: NetworkDescription, ltss) -> Network:
    ltss = tuple(ltss)
    n = len(ltss)
    if n != len(desc.process_files):
        raise NetworkError(f"{n} automata supplied for {len(desc.process_files)} process files")
    for rule in desc.rules:
        if rule.arity != n:
            raise NetworkError(f"rule arity {rule.arity} != {n} processes")
        named = [p for p in rule.participants if p is not None]
        if not named:
            raise NetworkError("rule with no participants")
        if INTERNAL_ACTION in named:
            raise NetworkError("the internal action cannot synchronize")
        if len(named) == 1:
            warnings.warn(f"rule for action {rule.result!r} has a single participant; "
                          "it behaves as a renaming", stacklevel=2)

    synced = [set() for _ in range(n)]
    for rule in desc.rules:
        for i, name in enumerate(rule.participants):
            lid = None if name is None else ltss[i].label_id(name)
            if lid is not None:
                synced[i].add(lid)
    independent = tuple(frozenset(set(range(len(l.labels))) - synced[i]) for i, l in enumerate(ltss))

    actions: list = []
    aid_of: dict = {}

    def intern(name):
        if name not in aid_of:
            aid_of[name] = len(actions)
            actions.append(name)
        return aid_of[name]

    rules = []
    for rule in desc.rules:
        res = intern(rule.result)
        lids = tuple(None if nm is None else ltss[i].label_id(nm)
                     for i, nm in enumerate(rule.participants))
        enabled = all(lid is not None for nm, lid in zip(rule.participants, lids) if nm is not None)
        rules.append(SyncRule(participants=lids, result=res, enabled=enabled))
    for i, lts in enumerate(ltss):
        for lid in sorted(independent[i]):
            intern(lts.labels[lid])

    indep_moves = []
    for i, lts in enumerate(ltss):
        per = [[] for _ in range(lts.num_states)]
        for src, lid, dst in lts.transitions:
            if lid in independent[i]:
                mv = (aid_of[lts.labels[lid]], dst)
                if mv not in per[src]:
                    per[src].append(mv)
        indep_moves.append(tuple(map(tuple, per)))

    rule_moves = []
    for rule in rules:
        if not rule.enabled:
            rule_moves.append(None)
            continue
        cols = []
        for i, lid in enumerate(rule.participants):
            if lid is None:
                continue
            per = [[] for _ in range(ltss[i].num_states)]
            for src, tl, dst in ltss[i].transitions:
                if tl == lid and dst not in per[src]:
                    per[src].append(dst)
            cols.append((i, tuple(map(tuple, per))))
        rule_moves.append(tuple(cols))

    return Network(processes=ltss, rules=tuple(rules), actions=tuple(actions),
                   independent=independent, indep_moves=tuple(indep_moves),
                   rule_moves=tuple(rule_moves))


def load_network(path) -> Network:
    path = Path(path)
    desc = parse_network(path.read_text(encoding="utf-8"))
    ltss = []
    for f in desc.process_files:
        p = Path(f)
        ltss.append(parse_aut((p if p.is_absolute() else path.parent / p).read_text(encoding="utf-8")))
    return build_network(desc, ltss)


# ------------------------------------------------------- point queries

def expand(net: Network, s: CompositeState):
    """(successor list, transition count) of one composite state, with the
    reference's ordering and counting conventions (network.py:184-238)."""
    out, seen = [], set()
    count = 0
    for i, moves in enumerate(net.indep_moves):
        here = moves[s[i]]
        count += len(here)
        for act, dst in here:
            key = (act, s[:i] + (dst,) + s[i + 1:])
            if key not in seen:
                seen.add(key)
                out.append(key)
    fired = set()
    for rule, cols in zip(net.rules, net.rule_moves):
        if cols is None:
            continue
        lists = [tbl[s[i]] for i, tbl in cols]
        if not all(lists):
            continue
        procs = [i for i, _ in cols]
        for combo in product(*lists):
            t = list(s)
            for i, d in zip(procs, combo):
                t[i] = d
            key = (rule.result, tuple(t))
            if key not in fired:
                fired.add(key)
                count += 1
            if key not in seen:
                seen.add(key)
                out.append(key)
    return out, count


def successors(net: Network, s: CompositeState):
    return expand(net, s)[0]


def is_deadlock(net: Network, s: CompositeState) -> bool:
    return not successors(net, s)


# --------------------------------------------------------- device CSR

def _may_collide(net: Network, r1: int, r2: int) -> bool:
    """Can rules r1 and r2 (same result) ever fire to the same target from
    the same source (network.py expand() dedups (result, target) pairs)?
    A common target t from source s needs, process by process:
      * in both rules: some local state q where both rules' destination
        lists intersect (t_i is in both);
      * in one rule only: a local state q that is among that rule's own
        destinations from q (the other rule leaves i at t_i = s_i = q).
    The conditions are independent per process, so if any one of them is
    unsatisfiable the pair never collides (a sound, state-blind test)."""
    m1 = dict(net.rule_moves[r1])
    m2 = dict(net.rule_moves[r2])
    for i in set(m1) | set(m2):
        if i in m1 and i in m2:
            if not any(set(a) & set(b) for a, b in zip(m1[i], m2[i])):
                return False
        else:
            per = m1[i] if i in m1 else m2[i]
            if not any(q in dsts for q, dsts in enumerate(per)):
                return False
    return True


def to_csr(net: Network, scheme, vlen: int | None = None) -> dict:
    """Flatten the move tables for the device (layout: include/gx.h,
    gx_network_csr).  Returns u32 numpy arrays."""
    P = len(net.processes)
    qbase = np.zeros(P + 1, np.int64)
    for i, lts in enumerate(net.processes):
        qbase[i + 1] = qbase[i] + lts.num_states
    proc = np.zeros((P, 4), np.uint32)
    for i in range(P):
        proc[i] = (scheme.word_index[i], scheme.shift[i], (1 << scheme.widths[i]) - 1, qbase[i])

    enabled = [r for r, mv in enumerate(net.rule_moves) if mv is not None]
    dev_id = {r: k for k, r in enumerate(enabled)}

    trig = [0]  # index 0: the empty list
    dedup = [0]
    rules = np.zeros((len(enabled), 4), np.uint32)
    parts, rq, rdst = [], [], []
    first_of: dict = {}  # (process, rule) for trigger lists
    for k, r in enumerate(enabled):
        cols = net.rule_moves[r]
        earlier = [dev_id[r0] for r0 in enabled[:k]
                   if net.rules[r0].result == net.rules[r].result and _may_collide(net, r0, r)]
        if earlier:
            dedup_off = len(dedup)
            dedup += [len(earlier)] + earlier
        else:
            dedup_off = 0
        rules[k] = (len(cols), len(parts), dedup_off, net.rules[r].result)
        for i, tbl in cols:
            base = len(rq)
            for dsts in tbl:
                rq.append((len(rdst), len(dsts)))
                rdst.extend(dsts)
            parts.append((base, scheme.word_index[i], scheme.shift[i], (1 << scheme.widths[i]) - 1))
        first_of.setdefault(cols[0][0], []).append(k)

    qtab = np.zeros((int(qbase[-1]), 4), np.uint32)
    im_dst = []
    for i, lts in enumerate(net.processes):
        mine = first_of.get(i, [])
        first_tbl = {k: net.rule_moves[enabled[k]][0][1] for k in mine}
        for q in range(lts.num_states):
            moves = net.indep_moves[i][q]
            dsts = []
            for _, d in moves:
                if d != q and d not in dsts:
                    dsts.append(d)
            fire = [k for k in mine if first_tbl[k][q]]
            if fire:
                toff = len(trig)
                trig += [len(fire)] + fire
            else:
                toff = 0
            qtab[qbase[i] + q] = (len(im_dst), len(dsts), len(moves), toff)
            im_dst.extend(dsts)

    u32 = lambda x, w=1: np.ascontiguousarray(np.asarray(x, np.uint32).reshape(-1)) if len(x) else np.zeros(w, np.uint32)
    return {
        "nproc": P, "nrules": len(enabled), "vlen": vlen or scheme.vector_length,
        "proc": u32(proc), "qtab": u32(qtab, 4), "im_dst": u32(im_dst),
        "trig": u32(trig), "rules": u32(rules, 4), "parts": u32(parts, 4),
        "rq": u32(rq, 2), "rdst": u32(rdst), "dedup": u32(dedup),
    }
