"""Host-side pieces (CPU): model parsing, network semantics, packing, the
device CSR layout, and the C ABI surface of libgx.so (symbols only)."""
import ctypes
import json
import re
import warnings

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_models, model_path
from paper_1801_05857_b200 import aut, network, statevec
from paper_1801_05857_b200.aut import ParseError, parse_aut, parse_network, unparse_aut
from paper_1801_05857_b200.hashtable import (HALF_BUCKET, PLAIN, TableConfig, hash_constants,
                                             slots_per_bucket)
from paper_1801_05857_b200.network import NetworkError, build_network, expand, load_network

MODELS = golden_models()


# ------------------------------------------------------------- parsers

def test_aut_basics():
    lts = parse_aut('des (0,1,2)\n(0,"a",1)')
    assert (lts.num_states, lts.initial, lts.labels, lts.transitions) == (2, 0, ("a",), ((0, 0, 1),))
    assert parse_aut('des (0,3,2)\n(0,"tau",1)\n(1,"i",0)\n(1,"tau",1)').labels == ("i",)
    assert parse_aut("des (0,2,2)\n(0, a, 1)\n(1, b-c!x, 0)").labels == ("a", "b-c!x")
    assert parse_aut('des (0,1,2)\n(0, "a, b (x)", 1)').labels == ("a, b (x)",)
    assert parse_aut('des (0,1,2)\r\n\r\n(0,"a",1)\r\n\r\n').transitions == ((0, 0, 1),)


@pytest.mark.parametrize("text,match", [
    ('des (0,2,2)\n(0,"a",1)', "header says 2, found 1"),
    ('des (0,2,2)\n(0,"a",1)\n(1,"b",5)', "line 3"),
    ("des 0 1 2\n", "header"),
    ("graph (0,1,2)\n", "header"),
    ("des (5,0,2)\n", "initial"),
    (f"des (0,0,{(1 << 20) + 1})\n", "range"),
    ("", "empty"),
])
def test_aut_errors(text, match):
    with pytest.raises(ParseError, match=match):
        parse_aut(text)


def test_aut_roundtrip_random():
    rng = np.random.default_rng(3)
    for _ in range(200):
        ns = int(rng.integers(1, 12))
        labs = ["a", "b", "c_d", "i", "x1"]
        tr = [(int(rng.integers(ns)), labs[int(rng.integers(5))], int(rng.integers(ns)))
              for _ in range(int(rng.integers(0, 20)))]
        text = f"des ({int(rng.integers(ns))}, {len(tr)}, {ns})\n" + \
            "".join(f'({s}, "{l}", {d})\n' for s, l, d in tr)
        lts = parse_aut(text)
        assert parse_aut(unparse_aut(lts)) == lts


def test_network_parser():
    pc = ('par using\n    send * rec *  _  -> trans,\n    send *  _  * rec -> trans\nin\n'
          '    "producer.aut"\n    || "consumer.aut"\n    || "consumer.aut"\nend par\n')
    d = parse_network(pc)
    assert d.process_files == ("producer.aut", "consumer.aut", "consumer.aut")
    assert d.rules[0].participants == ("send", "rec", None) and d.rules[0].result == "trans"
    assert parse_network('par using in "a.aut" end par').rules == ()
    d = parse_network("-- c\npar using a * b -> c -- t\nin x.aut || y.aut end par")
    assert d.process_files == ("x.aut", "y.aut")
    d = parse_network('par using _ * tau? -> tau in "x.aut" || "y.aut" end par')
    assert d.rules[0].participants == (None, "tau?") and d.rules[0].result == "i"


@pytest.mark.parametrize("text,match", [
    ('par using a * b -> c in "x.aut" || "y.aut" || "z.aut" end par', "rule arity 2 != 3 processes"),
    ('par using\n a ** b -> c\nin "x.aut" || "y.aut" end par', "line 2"),
    ('par using in "a.aut"', "end of input"),
    ('par using in "a.aut" end par extra', "trailing"),
])
def test_network_parser_errors(text, match):
    with pytest.raises(ParseError, match=match):
        parse_network(text)


# ----------------------------------------------------- network semantics

def test_build_network_errors():
    lts = parse_aut('des (0,1,2)\n(0,"i",1)')
    with pytest.raises(NetworkError, match="internal"):
        build_network(parse_network('par using i * i -> x in "x.aut" || "y.aut" end par'), [lts, lts])
    with pytest.raises(NetworkError):
        build_network(parse_network('par using in "x.aut" || "y.aut" end par'), [lts])
    a = parse_aut('des (0,1,2)\n(0,"a",1)')
    with pytest.warns(UserWarning, match="single participant"):
        build_network(parse_network('par using a * _ -> b in "x.aut" || "y.aut" end par'), [a, a])


def test_fig_independent_sets():
    net = load_network(model_path("fig1"))
    names = lambda i: sorted(net.processes[i].labels[l] for l in net.independent[i])
    assert names(0) == ["gen_work"] and names(1) == ["i", "work"] == names(2)


def test_host_expand_matches_reference_kats():
    """Point-query expand (API compatibility) equals the reference's expand
    on every reachable state of the small golden models, order included."""
    from paper_1801_05857_b200.network import max_successors
    kats = json.loads((GOLDEN / "expand_kats.json").read_text())
    warnings.simplefilter("ignore")
    for name, rows in kats.items():
        net = load_network(model_path(name))
        # network.max_successors sizes the sharded engine's frontier chunks
        # (no inbox may overflow): it must bound every reachable state
        bound = max_successors(net)
        for s, count, succ in rows:
            got, c = expand(net, tuple(s))
            assert c == count, (name, s)
            assert [[net.actions[a], list(t)] for a, t in got] == succ, (name, s)
            assert len(succ) <= bound, (name, s)


def test_golden_errors_reproduced():
    for name, g in MODELS.items():
        if "error" in g:
            with pytest.raises(ValueError):
                load_network(model_path(name))


# --------------------------------------------------------------- packing

def test_packing():
    sc = statevec.scheme_for_sizes([2, 2, 2])
    assert statevec.pack(sc, (1, 0, 1)) == (0x5,) and statevec.unpack(sc, (0x5,)) == (1, 0, 1)
    sc = statevec.scheme_for_sizes([1 << 20, 1 << 20])
    assert (sc.word_index, sc.shift, sc.vector_length) == ((0, 1), (0, 0), 2)
    with pytest.raises(statevec.PackingError, match="too wide"):
        statevec.scheme_for_sizes([1 << 20] * 30)
    with pytest.raises(statevec.PackingError, match="corrupt"):
        statevec.unpack(statevec.scheme_for_sizes([3]), (3,))
    assert statevec.dump_states([(2, 0), (1, 5), (1, 4)]) == \
        "00000001 00000004\n00000001 00000005\n00000002 00000000\n"
    arr = np.array([[2, 0], [1, 5], [1, 4]], np.uint32)
    assert statevec.dump_states_array(arr) == statevec.dump_states([tuple(r) for r in arr.tolist()])


def test_mark_bit_choice():
    assert statevec.mark_bit(statevec.scheme_for_sizes([2] * 32)) is None
    assert statevec.mark_bit(statevec.scheme_for_sizes([2] * 33)) == (1, 31)
    assert statevec.mark_bit(statevec.scheme_for_sizes([5] * 8)) == (0, 31)


def test_table_config_and_capacity():
    for L in range(1, 17):
        assert slots_per_bucket(32, L, HALF_BUCKET) == 2 * (16 // L)
    assert slots_per_bucket(16, 3, HALF_BUCKET) == 4 and slots_per_bucket(16, 3, PLAIN) == 5
    with pytest.raises(ValueError, match="too long"):
        slots_per_bucket(4, 5, PLAIN)
    assert TableConfig(bucket_words=32).resolved_layout() == HALF_BUCKET
    assert hash_constants(42, 1)[0] == (0xBDD732262FEB6E95, 0x28EFE333B266F103)


def test_csr_layout_counts():
    """The CSR's per-state transition counts and trigger lists agree with
    the host move tables (a device-free consistency check)."""
    for name in ("fig1", "gas3", "ring4", "collide", "rand3"):
        net = load_network(model_path(name))
        sc = statevec.make_scheme(net)
        c = network.to_csr(net, sc)
        proc = c["proc"].reshape(-1, 4)
        qtab = c["qtab"].reshape(-1, 4)
        for i, lts in enumerate(net.processes):
            for q in range(lts.num_states):
                e = qtab[proc[i][3] + q]
                assert e[2] == len(net.indep_moves[i][q])


# ---------------------------------------------------------------- C ABI

def declared_symbols():
    hdr = (ROOT / "include" / "gx.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char \*)\s*(gx_\w+)\s*\(", hdr, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1801_05857_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib.SIGNATURES)


def test_library_loads_and_reports_launch_counter():
    from paper_1801_05857_b200 import _lib
    assert _lib.kernel_launches() >= 0
    assert isinstance(_lib.last_error(), str)


# ------------------------------------------------------------------ CLI

def test_cli_gen_model_and_input_errors(tmp_path, capsys):
    """cli.py mirrors ltsmc's subcommands and exit codes (cli.py:28-31)."""
    from paper_1801_05857_b200.cli import main
    assert main(["gen-model", "token-ring", "--n", "3", "--out", str(tmp_path / "r3")]) == 0
    out = capsys.readouterr().out
    assert out.startswith("config[gen-model]:") and "net.exp" in out
    assert (tmp_path / "r3" / "net.exp").exists()
    assert main(["explore", str(tmp_path / "missing.exp")]) == 1
    assert main(["explore", str(tmp_path / "r3" / "net.exp"), "--oracle"]) == 1
    assert main(["explore", "--bucket-size", "5", "x"]) == 1
    assert main(["nonsense"]) == 1



def test_may_collide_is_sound_on_reachable_states():
    """network._may_collide prunes the device's same-result dedup checks; a
    pair it calls collision-free must never produce a common (result,
    target) from a reachable state.  Checked by brute force on every
    reachable state of the small golden models (expand KATs)."""
    from itertools import combinations, product
    from paper_1801_05857_b200.network import _may_collide
    kats = json.loads((GOLDEN / "expand_kats.json").read_text())
    warnings.simplefilter("ignore")
    checked = 0
    for name in ("collide", "fig1", "gas3", "phil3", "rand3", "rand7"):
        if name not in kats:
            continue
        net = load_network(model_path(name))
        live = [r for r, m in enumerate(net.rule_moves) if m is not None]
        pairs = [(a, b) for a, b in combinations(live, 2)
                 if net.rules[a].result == net.rules[b].result and not _may_collide(net, a, b)]

        def targets(r, s):
            cols = net.rule_moves[r]
            out = set()
            for combo in product(*[per[s[i]] for i, per in cols]):
                t = list(s)
                for (i, _), d in zip(cols, combo):
                    t[i] = d
                out.add(tuple(t))
            return out

        for s, _, _ in kats[name]:
            for a, b in pairs:
                assert not (targets(a, s) & targets(b, s)), (name, a, b, s)
                checked += 1
    assert checked > 0


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_philosophers_generator_equals_golden_family(n, tmp_path, capsys):
    """gen-model philosophers (the product's deadlocking family) produces the
    reference-pinned golden models phil2..5: same reachable set (dump sha
    from the real reference, tests/golden/models.json) and one deadlock."""
    import hashlib
    import json

    from conftest import GOLDEN
    from oracle import oracle as O
    from paper_1801_05857_b200.cli import main
    assert main(["gen-model", "philosophers", "--n", str(n), "--out", str(tmp_path / "p")]) == 0
    capsys.readouterr()
    r = O.explore(O.Net.from_file(tmp_path / "p" / "net.exp"), capacity_words=1 << 16, detect_deadlocks=True)
    want = json.loads((GOLDEN / "models.json").read_text())[f"phil{n}"]["runs"][0]
    assert hashlib.sha256(r.dump_states().encode()).hexdigest() == want["dump_states_sha"]
    assert (r.states, r.transitions, r.deadlocks_total) == \
        (want["report"]["states"], want["report"]["transitions"], want["report"]["deadlocks_total"]) == \
        (3 ** n - 1, want["report"]["transitions"], 1)
