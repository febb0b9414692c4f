"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run where /root/reference exists and `make -C oracle ref` has built
oracle/_ref/libtrs_ref.so:

    python tests/golden/make_golden.py

For every case it records the reference sweep engine's per-sweep widths and
sweep count (workers = 1; widths are schedule-independent,
sweep_engine_tests.cpp:162-186), the total rewrites, and the canonical DAG
words of the normal form.  It also asserts the reference's own seq/sweep
parity on each case (sweep_engine_tests.cpp:148-160) so a fixture is never
written from a diverging pair.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

MS2 = W.mergesort(2)


def with_input(text: str, term: str) -> str:
    """Replace the input line of a generated system (the reference tests' fixture trick)."""
    head = text[: text.index("input ")]
    return head + f"input {term};\n"


UNIT = {
    # sweep_engine_tests.cpp:42-61 (mergesort(2) signature)
    "unit_zero": with_input(MS2, "Zero()"),
    "unit_cons": with_input(MS2, "Cons(Zero(), Nil())"),
    "unit_merge_nil_nil": with_input(MS2, "Merge(Nil(), Nil())"),
    "unit_lt": with_input(MS2, "Lt(S(Zero()), S(S(Zero())))"),
    "unit_sort2": with_input(MS2, "Sort(Cons(S(Zero()), Cons(Zero(), Nil())))"),
    # sweep_engine_tests.cpp:63-82 collapse
    "unit_collapse": "sort Nat = Zero() | S(Nat) | Plus(Nat, Nat);\nvar X : Nat;\neqn Plus(Zero(), X) = X;\n"
                     "input Plus(Zero(), S(Zero()));\n",
    # :84-101 constructive
    "unit_constructive": "sort Nat = Zero() | S(Nat) | Len(List);\n     Bool = Gt(Nat, Nat);\n"
                         "     List = Nil() | Sort(List) | Sort2(Bool, List);\nvar L : List;\n"
                         "eqn Sort(L) = Sort2(Gt(Len(L), S(Zero())), L);\ninput Sort(Nil());\n",
    # :103-115 duplicated template variable
    "unit_dupvar": "sort Nat = Zero() | S(Nat) | F(Nat) | G(Nat, Nat);\nvar X : Nat;\neqn F(X) = G(X, X);\n"
                   "input F(S(Zero()));\n",
    # :117-132 erasure
    "unit_erase": "sort T = A() | B() | F(T);\nvar X : T;\neqn F(X) = A();\ninput F(F(A()));\n",
    # seq_engine_tests.cpp:116-123 zero equations
    "unit_noeqn": "sort Nat = Zero() | S(Nat);\nvar X : Nat;\neqn\ninput S(Zero());\n",
    # a shared fresh node built twice by one template (structural RHS sharing)
    "unit_shared_fresh": "sort T = A() | B() | F(T) | G(T, T) | H(T);\nvar X : T;\n"
                         "eqn F(X) = G(H(X), H(X));\n    H(A()) = B();\ninput F(F(A()));\n",
    # constant chains (A() -> B() -> C(), no rules on C) under a parent that
    # matches the chain's end, and a chain that stops at a building rule
    "unit_chain_nf": "sort T = A() | B() | C() | D() | F(T) | G(T, T);\nvar X : T;\n"
                     "eqn A() = B();\n    B() = C();\n    F(C()) = G(A(), D());\n    D() = A();\n"
                     "input G(F(A()), F(B()));\n",
    "unit_chain_into_build": "sort T = A() | B() | C() | F(T) | H(T, T);\nvar X : T;\n"
                             "eqn A() = B();\n    B() = F(C());\n    F(X) = H(X, X);\n"
                             "input H(A(), F(A()));\n",
    # a polled parent: two parents waiting on one shared non-nf node
    "unit_two_waiters": "sort T = A() | B() | F(T) | G(T, T) | K(T, T) | H(T);\nvar X : T; Y : T;\n"
                        "eqn F(X) = K(G(H(X), H(X)), H(X));\n    H(A()) = B();\n    G(X, Y) = Y;\n"
                        "    K(X, Y) = X;\ninput F(A());\n",
}

FAMILIES = {
    "transform3": W.transform(3),
    "transform6": W.transform(6),
    "mergesort10_s3": W.mergesort(10, 3),
    "mergesort50_s42": W.mergesort(50, 42),
    "mergesort64_s1": W.mergesort(64, 1),
    "treemergesort_3_4_s11": W.treemergesort(3, 4, 11),
    "treemergesort_2_3_s5": W.treemergesort(2, 3, 5),
    "treemergesort_4_5_s7": W.treemergesort(4, 5, 7),
    "fib10": W.fib(10),
    "fib12": W.fib(12),
    "buildsum3": W.buildsum(3),
    "buildsum8": W.buildsum(8),
    "reverse8": W.reverse(8),
    "reverse64": W.reverse(64),
    "ackermann22": W.ackermann(2, 2),
    "ackermann23": W.ackermann(2, 3),
    "fibbatch16_s1": W.fib_batch(1, roots=16),
    "fibbatch64_s3": W.fib_batch(3, roots=64),
}


def record(text: str) -> dict:
    sw = ref.run(text, "sweep", workers=1)
    sq = ref.run(text, "seq")
    assert sw.status == 0 and sq.status == 0, (sw.message, sq.message)
    assert sw.rewrites == sq.rewrites, "reference seq/sweep rewrite divergence"
    assert (sw.words == sq.words).all(), "reference seq/sweep DAG divergence"
    return {
        "text": text,
        "rewrites": int(sw.rewrites),
        "sweeps": int(sw.sweeps),
        "max_width": int(sw.max_width),
        "widths": [int(x) for x in sw.widths],
        "words": [int(x) for x in sw.words],
        "nodes": int(sw.n_nodes),
    }


def main():
    cases = {}
    for name, text in {**UNIT, **FAMILIES}.items():
        cases[name] = record(text)
        print(f"{name}: {cases[name]['rewrites']} rewrites, {cases[name]['sweeps']} sweeps")
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref/libtrs_ref.so (unmodified reference)",
           "cases": cases}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "small.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
