"""Synthetic workload texts for the BASELINE configs.

The three reference families are restated from the reference generator
(`proj/src/generators.cpp`): the SplitMix64 numeral stream (`:12-25`), the
merge-sort TRS header (`:27-66`), `numeral_list` (`:68-74`), `tree_input`
(`:76-82`), `transform_text` (`:84-110`), `peano` (`:114-120`) and
`generate` (`:146-174`).  The texts are byte-identical to the reference's
(`tests/test_workloads.py` checks that against the reference itself).

The configs the reference does not ship (fib, build+sum, reverse,
Ackermann, the fib batch shards) follow SURVEY.md Appendix A verbatim.
"""
from __future__ import annotations

_MASK = (1 << 64) - 1
NUMERAL_BOUND = 32  # generators.cpp:11


class SplitMix64:
    """generators.cpp:14-25 (state += golden gamma, then the mix-64 finaliser)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def numeral(self) -> int:
        return self.next() % NUMERAL_BOUND


def peano(value: int, succ: str = "S") -> str:
    return f"{succ}(" * value + "Zero()" + ")" * value


MERGESORT_HEADER = (
    "sort  Nat  = struct Zero() | S(Nat) | Len(List);\n"
    "      Bool = struct True() | False() | Lt(Nat, Nat) | Gt(Nat, Nat);\n"
    "      List = struct Nil() | Cons(Nat, List) | Merge(List, List) |\n"
    "             Merge2(Bool, Nat, List, Nat, List) | Even(List) |\n"
    "             Odd(List) | Sort(List) | Sort2(Bool, List);\n"
    "      Tree = struct Leaf(List) | Node(Tree, Tree);\n"
    "\n"
    "var X : Nat; Y : Nat; B : Bool; L : List; M : List;\n"
    "\n"
    "eqn\n"
    "  Len(Nil()) = Zero();\n"
    "  Len(Cons(X, L)) = S(Len(L));\n"
    "\n"
    "  Merge(Nil(), M) = M;\n"
    "  Merge(L, Nil()) = L;\n"
    "  Merge(Cons(X, L), Cons(Y, M)) = Merge2(Lt(X, Y), X, L, Y, M);\n"
    "\n"
    "  Merge2(True(), X, L, Y, M) = Cons(X, Merge(L, Cons(Y, M)));\n"
    "  Merge2(False(), X, L, Y, M) = Cons(Y, Merge(Cons(X, L), M));\n"
    "\n"
    "  Sort(L) = Sort2(Gt(Len(L), S(Zero())), L);\n"
    "  Sort2(False(), L) = L;\n"
    "  Sort2(True(), L) = Merge(Sort(Even(L)), Sort(Odd(L)));\n"
    "\n"
    "  Even(Nil()) = Nil();\n"
    "  Even(Cons(X, L)) = Cons(X, Odd(L));\n"
    "  Odd(Nil()) = Nil();\n"
    "  Odd(Cons(X, L)) = Even(L);\n"
    "\n"
    "  Gt(Zero(), Zero()) = False();\n"
    "  Gt(Zero(), S(Y)) = False();\n"
    "  Gt(S(X), Zero()) = True();\n"
    "  Gt(S(X), S(Y)) = Gt(X, Y);\n"
    "\n"
    "  Lt(Zero(), Zero()) = False();\n"
    "  Lt(Zero(), S(Y)) = True();\n"
    "  Lt(S(X), Zero()) = False();\n"
    "  Lt(S(X), S(Y)) = Lt(X, Y);\n"
    "\n"
)


def _numeral_list(rng: SplitMix64, length: int) -> str:
    head = "".join(f"Cons({peano(rng.numeral())}, " for _ in range(length))
    return head + "Nil()" + ")" * length


def _tree_input(rng: SplitMix64, depth: int, length: int) -> str:
    # generators.cpp:76-82, left subtree first so the numeral stream reads leaf by leaf
    if depth == 0:
        return f"Leaf(Sort({_numeral_list(rng, length)}))"
    left = _tree_input(rng, depth - 1, length)
    right = _tree_input(rng, depth - 1, length)
    return f"Node({left}, {right})"


def mergesort(length: int, seed: int = 1) -> str:
    out = f"% family: mergesort  n={length}  seed={seed}\n" + MERGESORT_HEADER
    rng = SplitMix64(seed)
    return out + f"input Sort({_numeral_list(rng, length)});\n"


def treemergesort(depth: int, length: int, seed: int = 1) -> str:
    if depth > 26:
        raise ValueError("treemergesort depth above 26 is not supported")
    out = f"% family: treemergesort  depth={depth}  k={length}  seed={seed}\n" + MERGESORT_HEADER
    rng = SplitMix64(seed)
    return out + f"input {_tree_input(rng, depth, length)};\n"


def transform(depth: int) -> str:
    letters = [chr(c) for c in range(ord("A"), ord("Z") + 1)]
    out = f"% family: transform  depth={depth}\n"
    out += "sort Nat  = struct Zero() | Suc(Nat);\n     Tree = struct "
    out += "".join(f"{c}() | " for c in letters)
    out += "End() |\n            Node(Tree, Tree) | Expand(Nat) | Expand2(Nat);\n\n"
    out += "var o : Tree; p : Tree; x : Nat;\n\neqn\n"
    out += (
        "  Expand(Zero()) = A();\n"
        "  Expand(Suc(x)) = Node(Expand(x), Expand2(x));\n"
        "  Expand2(Zero()) = A();\n"
        "  Expand2(Suc(x)) = Node(Expand(x), Expand2(x));\n"
    )
    for c in letters:
        nxt = "End()" if c == "Z" else f"{chr(ord(c) + 1)}()"
        out += f"  {c}() = {nxt};\n"
    out += "\ninput Expand(" + "Suc(" * depth + "Zero()" + ")" * depth + ");\n"
    return out


def generated_numerals(family: str, length: int, depth: int = 0, seed: int = 1) -> list[int]:
    """generators.cpp:176-183: the numeral sequence an instance embeds."""
    leaves = 1 if family == "mergesort" else (1 << depth)
    rng = SplitMix64(seed)
    return [rng.numeral() for _ in range(leaves * length)]


# ---------------------------------------------------------------------------
# SURVEY.md Appendix A configs


FIB_RULES = (
    "var X : Nat; Y : Nat;\n"
    "eqn Plus(Zero(), Y) = Y;\n"
    "    Plus(S(X), Y) = S(Plus(X, Y));\n"
    "    Fib(Zero()) = Zero();\n"
    "    Fib(S(Zero())) = S(Zero());\n"
    "    Fib(S(S(X))) = Plus(Fib(X), Fib(S(X)));\n"
)


def fib(n: int) -> str:
    """Config 1: Fib(S^n(Zero())) with Peano Plus (Appendix A)."""
    return (
        f"% family: fib  n={n}\n"
        "sort Nat = struct Zero() | S(Nat) | Plus(Nat, Nat) | Fib(Nat);\n"
        + FIB_RULES
        + f"input Fib({peano(n)});\n"
    )


def buildsum(depth: int) -> str:
    """Config 3b: Sum(Build(Suc^depth(Zero()))) -> B0^depth(B1(Z())) (Appendix A)."""
    return (
        f"% family: buildsum  depth={depth}\n"
        "sort Nat  = struct Zero() | Suc(Nat);\n"
        "     Bin  = struct Z() | B0(Bin) | B1(Bin) | Add(Bin, Bin) | Inc(Bin) | Sum(Tree);\n"
        "     Tree = struct Leaf(Bin) | Node(Tree, Tree) | Build(Nat) | Build2(Nat);\n"
        "var x : Nat; a : Bin; b : Bin; l : Tree; r : Tree;\n"
        "eqn Build(Zero()) = Leaf(B1(Z()));\n"
        "    Build(Suc(x)) = Node(Build(x), Build2(x));\n"
        "    Build2(Zero()) = Leaf(B1(Z()));\n"
        "    Build2(Suc(x)) = Node(Build(x), Build2(x));\n"
        "    Sum(Leaf(a)) = a;\n"
        "    Sum(Node(l, r)) = Add(Sum(l), Sum(r));\n"
        "    Add(Z(), b) = b;\n"
        "    Add(a, Z()) = a;\n"
        "    Add(B0(a), B0(b)) = B0(Add(a, b));\n"
        "    Add(B0(a), B1(b)) = B1(Add(a, b));\n"
        "    Add(B1(a), B0(b)) = B1(Add(a, b));\n"
        "    Add(B1(a), B1(b)) = B0(Inc(Add(a, b)));\n"
        "    Inc(Z()) = B1(Z());\n"
        "    Inc(B0(a)) = B1(a);\n"
        "    Inc(B1(a)) = B0(Inc(a));\n"
        "input Sum(Build(" + "Suc(" * depth + "Zero()" + ")" * depth + "));\n"
    )


def reverse(n: int) -> str:
    """Config 4a: Rev of an n-element list whose i-th element is S^(i mod 4)(Zero())."""
    items = "".join(f"Cons({peano(i % 4)}, " for i in range(n))
    return (
        f"% family: reverse  n={n}\n"
        "sort Nat  = struct Zero() | S(Nat);\n"
        "     List = struct Nil() | Cons(Nat, List) | Rev(List) | Rev2(List, List);\n"
        "var X : Nat; L : List; A : List;\n"
        "eqn Rev(L) = Rev2(L, Nil());\n"
        "    Rev2(Nil(), A) = A;\n"
        "    Rev2(Cons(X, L), A) = Rev2(L, Cons(X, A));\n"
        f"input Rev({items}Nil(){')' * n});\n"
    )


def ackermann(m: int, n: int) -> str:
    """Config 4b: Ack(m, n) in Peano numerals."""
    return (
        f"% family: ackermann  m={m} n={n}\n"
        "sort Nat = struct Zero() | S(Nat) | Ack(Nat, Nat);\n"
        "var M : Nat; N : Nat;\n"
        "eqn Ack(Zero(), N) = S(N);\n"
        "    Ack(S(M), Zero()) = Ack(M, S(Zero()));\n"
        "    Ack(S(M), S(N)) = Ack(M, Ack(S(M), N));\n"
        f"input Ack({peano(m)}, {peano(n)});\n"
    )


def _balanced(items: list[str]) -> str:
    # pair adjacent leaves Node(l_{2i}, l_{2i+1}) level by level up to one root
    level = items
    while len(level) > 1:
        nxt = []
        for i in range(0, len(level) - 1, 2):
            nxt.append(f"Node({level[i]}, {level[i + 1]})")
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


def fib_batch(seed: int, roots: int = 4096) -> str:
    """Config 5F shard `seed`: balanced Node tree of Leaf(Fib(S^(10 + z mod 6)(Zero())))."""
    rng = SplitMix64(seed)
    leaves = [f"Leaf(Fib({peano(10 + rng.next() % 6)}))" for _ in range(roots)]
    return (
        f"% family: fibbatch  seed={seed}  roots={roots}\n"
        "sort Nat = struct Zero() | S(Nat) | Plus(Nat, Nat) | Fib(Nat);\n"
        "     Tree = struct Leaf(Nat) | Node(Tree, Tree);\n"
        + FIB_RULES
        + f"input {_balanced(leaves)};\n"
    )


def treemergesort_batch(seed: int, depth: int = 12, length: int = 16) -> str:
    """Config 5S shard `seed`: GenSpec::treemergesort(12, 16, seed)."""
    return treemergesort(depth, length, seed)


# name -> (text factory, description); full-size BASELINE configs
CONFIGS = {
    "fib18": (lambda: fib(18), "config 1: Fib(18) as one term"),
    "mergesort16k": (lambda: mergesort(16384, 1), "config 2: mergesort of 2^14 Peano numerals"),
    "transform22": (lambda: transform(22), "config 3a: transformation tree depth 22"),
    "buildsum22": (lambda: buildsum(22), "config 3b: tree build+sum depth 22"),
    "reverse16k": (lambda: reverse(16384), "config 4a: list reverse 2^14"),
    "ackermann36": (lambda: ackermann(3, 6), "config 4b: Ackermann(3,6)"),
}


def batch_shards(kind: str, shards: int = 8) -> list[str]:
    """Config 5: the 8 shards x 4096 independent roots (seeds 1..8)."""
    if kind == "fib":
        return [fib_batch(s) for s in range(1, shards + 1)]
    if kind == "sort":
        return [treemergesort_batch(s) for s in range(1, shards + 1)]
    raise ValueError(kind)


def wide(k: int, vals=(3, 2, 4, 1, 2, 5, 1)) -> str:
    """A test family for wide records (not a BASELINE config): a k-ary symbol
    W rotating its arguments (W = 16 words for k <= 8, 32 beyond), a depth-3
    pattern (Q, interpreted matcher) and Peano addition (planned matcher)."""
    xs = [f"x{j}" for j in range(1, k + 1)]
    ts = ", ".join(["Nat"] * k)
    lines = [f"sort Nat = struct Zero() | S(Nat) | P(Nat, Nat) | W({ts}) | D(Nat) | Q(Nat);",
             "var " + " ".join(f"{x} : Nat;" for x in xs) + " y : Nat;",
             "eqn",
             "  P(Zero(), y) = y;",
             "  P(S(x1), y) = S(P(x1, y));",
             "  D(x1) = P(Q(x1), x1);",
             "  Q(S(S(S(x1)))) = Q(x1);",
             "  Q(S(S(Zero()))) = Zero();",
             "  Q(x1) = x1;",
             f"  W(Zero(), {', '.join(xs[1:])}) = P({xs[1]}, {xs[-1]});",
             f"  W(S(x1), {', '.join(xs[1:])}) = W({', '.join(xs[1:])}, D(x1));"]

    def w(off):
        vs = [vals[(off + j) % len(vals)] for j in range(k - 1)] + [0]
        return "W(" + ", ".join(peano(v) for v in vs) + ")"

    lines.append(f"input P({w(0)}, P({w(1)}, {w(2)}));")
    return "\n".join(lines) + "\n"


def many_rules(nrules: int = 40, depth: int = 8) -> str:
    """A test family (not a BASELINE config): one symbol with `nrules` rules
    (past the 32-rule match tables, so its rule choice walks the rules) next
    to ordinary planned symbols."""
    cs = [f"C{k}()" for k in range(nrules + 1)]
    lines = ["sort T = struct " + " | ".join(cs) + " | F(T) | G(T, T) | H(T);", "var x : T; y : T;", "eqn"]
    for k in range(nrules):
        lines.append(f"  F(C{k}()) = H(C{k + 1}());")
    lines.append("  H(x) = x;")
    lines.append("  G(C0(), y) = F(y);")
    lines.append("  G(x, y) = F(x);")

    def tree(d, k):
        if d == 0:
            return f"F(C{k % nrules}())"
        return f"G({tree(d - 1, 2 * k)}, {tree(d - 1, 2 * k + 1)})"

    lines.append(f"input {tree(depth, 1)};")
    return "\n".join(lines) + "\n"


def random_program(seed: int, nfun: int = 4, input_depth: int = 7, call_depth: int = 4, calls: int = 64,
                   max_arity: int = 3, input_seed: int | None = None) -> str:
    """A test family (not a BASELINE config): a random terminating system.

    Constructors K0() | K1(T) | K2(T, T) and functions F0..F{nfun-1} of
    arity 1-3, each defined by first-match rules on nested constructor
    patterns (depth <= 2, some on later arguments too) with an optional
    catch-all.  A right-hand side may call a lower function freely and its own
    function only on a variable bound strictly inside the first argument's
    pattern, so every system terminates (recursive path order with F_i > F_j
    for i > j > constructors).  Inputs are random constructor terms under
    random calls, `calls` of them joined by a balanced K2 tree (independent
    redexes side by side, so the frontier widens past one warp).  With
    `input_seed` the system is the one of `seed` and only the input differs
    (several such texts batch as roots of one store)."""
    rng = SplitMix64(seed * 0x9E3779B1 + 17)

    def rnd(n):
        return rng.next() % n

    arity = [1 + rnd(max_arity) for _ in range(nfun)]
    cons = [("K0", 0), ("K1", 1), ("K2", 2)]
    lines = ["sort T = struct K0() | K1(T) | K2(T, T) | "
             + " | ".join(f"F{i}({', '.join(['T'] * a)})" for i, a in enumerate(arity)) + ";"]
    vars_ = [f"x{k}" for k in range(12)] + ["y1", "y2"]
    lines.append("var " + " ".join(f"{v} : T;" for v in vars_))
    lines.append("eqn")

    def pattern(depth, fresh, inner):
        # a constructor pattern; `inner` collects variables bound strictly inside it
        c, a = cons[rnd(3)]
        if a == 0:
            return f"{c}()"
        subs = []
        for _ in range(a):
            if depth > 1 and rnd(3) == 0:
                subs.append(pattern(depth - 1, fresh, inner))
            else:
                v = fresh.pop(0)
                inner.append(v)
                subs.append(v)
        return f"{c}({', '.join(subs)})"

    def rhs(i, depth, scope, smaller):
        choice = rnd(10)
        if depth == 0 or choice < 3:
            if scope and rnd(4) != 0:
                return scope[rnd(len(scope))]
            return "K0()"
        if choice < 6:
            c, a = cons[1 + rnd(2)]
            return f"{c}({', '.join(rhs(i, depth - 1, scope, smaller) for _ in range(a))})"
        if choice < 9 and smaller:
            args = [smaller[rnd(len(smaller))]] + [rhs(i, depth - 1, scope, smaller) for _ in range(arity[i] - 1)]
            return f"F{i}({', '.join(args)})"
        if i > 0:
            j = rnd(i)
            return f"F{j}({', '.join(rhs(i, depth - 1, scope, smaller) for _ in range(arity[j]))})"
        return "K0()"

    for i in range(nfun):
        seen = set()
        for _ in range(1 + rnd(3)):
            fresh = list(vars_[:12])
            inner = []
            first = pattern(2, fresh, inner)
            rest = []
            for _ in range(arity[i] - 1):
                if rnd(4) == 0:
                    rest.append(pattern(1, fresh, []))
                else:
                    rest.append(fresh.pop(0))
            lhs = f"F{i}({', '.join([first] + rest)})"
            if lhs in seen:
                continue
            seen.add(lhs)
            scope = [v for v in vars_[:12] if v not in fresh]
            lines.append(f"  {lhs} = {rhs(i, 3, scope, inner)};")
        if rnd(6) != 0:
            xs = vars_[: arity[i]]
            lines.append(f"  F{i}({', '.join(xs)}) = {rhs(i, 2, xs, [])};")

    def data(depth):
        if depth == 0 or rnd(6) == 0:
            return "K0()"
        c, a = cons[1 + rnd(2)]
        return f"{c}({', '.join(data(depth - 1) for _ in range(a))})"

    def term(depth, top=False):
        if depth == 0 or (not top and rnd(2) == 0):
            return data(input_depth)
        i = rnd(nfun)
        return f"F{i}({', '.join(term(depth - 1) for _ in range(arity[i]))})"

    if input_seed is not None:
        rng = SplitMix64(input_seed * 0x85EBCA77 + 3)  # same system, another input
    items = [term(call_depth, True) for _ in range(calls)]
    while len(items) > 1:
        items = [f"K2({items[k]}, {items[k + 1]})" if k + 1 < len(items) else items[k] for k in range(0, len(items), 2)]
    lines.append(f"input {items[0]};")
    return "\n".join(lines) + "\n"
