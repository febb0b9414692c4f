"""Host front end (parser/resolver, compile, load/extract) against the
reference's behaviour: dispatch dumps, diagnostics, store layout, round
trips.  CPU only; goes through libtrs_b200.so's host C ABI."""
import random

import numpy as np
import pytest

from oracle import ref
from paper_2009_07174_b200 import api
from paper_2009_07174_b200 import workloads as W

PLUS = ("sort Nat = Zero() | S(Nat) | Plus(Nat, Nat);\nvar X : Nat; Y : Nat;\n"
        "eqn Plus(Zero(), X) = X;\n    Plus(S(X), Y) = S(Plus(X, Y));\ninput Plus(Zero(), Zero());\n")

FAMILIES = [W.transform(3), W.mergesort(50, 42), W.treemergesort(3, 4, 11), W.fib(10), W.buildsum(3),
            W.reverse(8), W.ackermann(2, 2), W.fib_batch(1, roots=8)]


def test_dump_dispatch_golden():
    # dispatch_tests.cpp:204-219
    assert api.System(PLUS).dump_dispatch() == (
        "symbol Plus/2: 2 rule(s)\n"
        "  rule #0: Plus(Zero(), X) = X\n"
        "    check [0] = Zero\n"
        "    bind  [1] -> X\n"
        "    root  reuse X\n"
        "  rule #1: Plus(S(X), Y) = S(Plus(X, Y))\n"
        "    check [0] = S\n"
        "    bind  [0.0] -> X\n"
        "    bind  [1] -> Y\n"
        "    new   n0 = Plus(X, Y)\n"
        "    root  n1 = S(n0)\n")


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("k", range(len(FAMILIES)))
def test_dump_dispatch_matches_reference(k):
    text = FAMILIES[k]
    assert api.System(text).dump_dispatch() == ref.dump_dispatch(text)


def test_rule_counts_and_sharing():
    s = api.System(W.mergesort(2))
    assert s.num_rules == 22 and s.max_new_slots == 4
    # structural RHS sharing: G(X, X) builds no node for X and F(X)=G(H(X),H(X)) builds one H
    t = api.System("sort T = A() | F(T) | G(T, T) | H(T);\nvar X : T;\neqn F(X) = G(H(X), H(X));\ninput F(A());\n")
    assert "new   n0 = H(X)\n    root  n1 = G(n0, n0)" in t.dump_dispatch()
    assert t.max_new_slots == 1


BAD = {
    "lex": "sort T = A();\nvar X : T;\neqn\ninput A() $;\n",
    "missing_section": "sort T = A();\neqn\ninput A();\n",
    "unknown_symbol": "sort T = A();\nvar X : T;\neqn B() = A();\ninput A();\n",
    "arity": "sort T = A() | F(T);\nvar X : T;\neqn F(A(), A()) = A();\ninput A();\n",
    "sort": "sort T = A(); U = B() | G(U);\nvar X : T;\neqn G(A()) = B();\ninput B();\n",
    "non_linear": "sort T = A() | F(T, T);\nvar X : T;\neqn F(X, X) = A();\ninput A();\n",
    "free_rhs": "sort T = A() | F(T);\nvar X : T; Y : T;\neqn F(X) = Y;\ninput A();\n",
    "lhs_var": "sort T = A() | F(T);\nvar X : T;\neqn X = A();\ninput A();\n",
    "non_ground": "sort T = A() | F(T);\nvar X : T;\neqn\ninput F(X);\n",
    "constant_without_parens": "sort T = A() | F(T);\nvar X : T;\neqn F(A) = A();\ninput A();\n",
    "duplicate": "sort T = A() | A();\nvar X : T;\neqn\ninput A();\n",
    "trailing": "sort T = A();\nvar X : T;\neqn\ninput A(); A();\n",
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_diagnostics_reject(name):
    with pytest.raises(ValueError):
        api.System(BAD[name])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("name", sorted(BAD))
def test_diagnostics_match_reference(name):
    """Same located diagnostics (file:line:col: kind: message) as parser.cpp."""
    try:
        api.System(BAD[name])
        ours = ""
    except ValueError as e:
        ours = str(e)
    assert ours == ref.diagnostics(BAD[name])


def test_load_layout_and_pin():
    # term_store_tests.cpp:22-41
    s = api.System(W.mergesort(2).split("input ")[0] + "input Cons(Zero(), Nil());\n")
    st = api.Store.load(s)
    v = st.view()
    assert v["n"] == 4 and list(v["roots"]) == [1]
    assert v["hss"][1] == s.symbol_id("Cons")
    assert list(v["refcounts"][1:4]) == [1, 1, 1]
    assert st.dump(s) == "1  Cons  2  3  rc=1  -\n2  Zero  rc=1  -\n3  Nil  rc=1  -\n"


def test_extract_inverts_load_on_random_ground_terms():
    # term_store_tests.cpp:43-52 (300 random ground terms)
    rng = random.Random(7)
    s = api.System(W.mergesort(2))
    syms = [(s.symbol_name(f), s.symbol_arity(f)) for f in range(s.num_symbols)]
    header = W.mergesort(2).split("input ")[0]
    for _ in range(300):
        def gen(depth):
            cands = [x for x in syms if depth > 0 or x[1] == 0]
            name, ar = rng.choice(cands)
            return f"{name}(" + ", ".join(gen(depth - 1) for _ in range(ar)) + ")"
        term = gen(4)
        try:
            t = api.System(header + f"input {term};\n")
        except ValueError:
            continue  # ill-sorted random term
        st = api.Store.load(t)
        np.testing.assert_array_equal(st.extract_canonical(), t.input_canonical())
        np.testing.assert_array_equal(st.canonical(), t.input_canonical())


def test_explicit_capacity_too_small():
    s = api.System(W.mergesort(2).split("input ")[0] + "input Cons(Zero(), Nil());\n")
    with pytest.raises(api.EngineError) as ei:
        api.Store.load(s, capacity=3)
    assert ei.value.fault == api.EngineFault.Capacity


def test_extract_surfaces_dangling_reference():
    # term_store_tests.cpp:198-209
    s = api.System(W.mergesort(2).split("input ")[0] + "input Cons(Zero(), Nil());\n")
    st = api.Store.load(s)
    st.poke_arg(0, 1, 0)
    with pytest.raises(api.EngineError) as ei:
        st.extract_canonical()
    assert ei.value.fault == api.EngineFault.DanglingReference


def test_deep_inputs_do_not_recurse():
    # a 20k-element list and S^2584: the resolver and load are iterative
    s = api.System(W.mergesort(2).split("input ")[0] + "input Len(" + "Cons(S(Zero()), " * 20000 + "Nil()" +
                   ")" * 20000 + ");\n")
    st = api.Store.load(s)
    assert st.view()["n"] == 20000 * 3 + 3


def test_batched_store_roots():
    texts = [W.fib_batch(s, roots=4) for s in (1, 2, 3)]
    systems = [api.System(t) for t in texts]
    st = api.Store.load(systems)
    v = st.view()
    assert v["num_roots"] == 3
    for k, s in enumerate(systems):
        np.testing.assert_array_equal(st.canonical(k), s.input_canonical())


def test_batched_store_rejects_mismatched_signatures():
    with pytest.raises(ValueError):
        api.Store.load([api.System(W.fib(3)), api.System(W.ackermann(1, 1))])


def test_print_words_round_trip():
    s = api.System(W.fib(5))
    assert s.print_words(s.input_canonical()) == s.print_input() == f"Fib({W.peano(5)})"


def _mutants(seed: int):
    """Syntax-error mutants of valid systems: a punctuation or word removed,
    doubled or swapped for another, anywhere in the text."""
    import random
    import re

    rng = random.Random(seed)
    base = [W.fib(3), W.mergesort(3, 1), W.buildsum(2), W.ackermann(1, 1),
            "sort T = struct A() | F(T) | G(T, T);\nvar X : T; Y : T;\neqn F(X) = G(X, X);\ninput F(A());\n"]
    text = rng.choice(base)
    toks = [m for m in re.finditer(r"[A-Za-z_][A-Za-z0-9_]*|[(),;=|:%$]", text)]
    out = []
    for _ in range(4):
        m = rng.choice(toks)
        a, b = m.span()
        op = rng.randrange(4)
        if op == 0:
            t = text[:a] + text[b:]
        elif op == 1:
            t = text[:a] + m.group() + " " + text[a:]
        elif op == 2:
            t = text[:a] + rng.choice(["(", ")", ",", ";", "=", "|", ":", "sort", "var", "eqn", "input", "struct",
                                       "Q", "$", "%"]) + text[b:]
        else:
            c = rng.choice(toks)
            t = text[:a] + c.group() + text[b:]
        out.append(t)
    return out


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(150))
def test_diagnostics_fuzz_match_reference(seed):
    """Error recovery equals the reference's on mutated systems: the same
    located diagnostics, in the same order, or the same acceptance."""
    for text in _mutants(seed):
        try:
            api.System(text)
            ours = ""
        except ValueError as e:
            ours = str(e)
        assert ours == ref.diagnostics(text), text
