"""The C oracle restatement (oracle/trs_oracle.c), pinned against the
golden vectors produced by the unmodified reference (tests/golden/) and,
where oracle/_ref was built, against the reference live."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref
from paper_2009_07174_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "small.json")
CASES = json.load(open(GOLDEN))["cases"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_sweep_restatement_matches_reference_golden(name):
    g = CASES[name]
    o = O.run_text(g["text"])
    assert o.status == 0
    assert o.rewrites == g["rewrites"]
    assert o.sweeps == g["sweeps"]
    np.testing.assert_array_equal(o.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(o.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.parametrize("name", sorted(CASES))
def test_seq_restatement_matches_reference_golden(name):
    g = CASES[name]
    o = O.run_seq(g["text"])
    assert o.rewrites == g["rewrites"]
    np.testing.assert_array_equal(o.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("text", [W.fib(12), W.mergesort(20, 4), W.treemergesort(3, 4, 11), W.buildsum(6)])
def test_full_trace_matches_reference_live(text):
    """With one worker the reference trace is deterministic: live_terms, n
    and free_len must match too (sweep_engine.cpp:117-128)."""
    r = ref.run(text, "sweep", workers=1)
    o = O.run_text(text)
    np.testing.assert_array_equal(o.widths, r.widths)
    np.testing.assert_array_equal(o.live, r.live)


def test_counts_match_survey_8d():
    """Counter definitions reproduce SURVEY.md §8(d): fib(18) A = 233 k
    (9.57/rw), S_min 498 B/rw; transform(16) A/rw 0.43, S_min 30 B/rw,
    3.29 slot visits per rewrite."""
    o = O.run_text(W.fib(18), words=False)
    assert o.rewrites == 24363 and o.sweeps == 5240
    assert abs(o.accesses / o.rewrites - 9.57) < 0.01
    assert abs(o.s_min(2) / o.rewrites - 498) < 1
    t = O.run_text(W.transform(16), words=False)
    assert abs(t.accesses / t.rewrites - 0.43) < 0.005
    assert abs(t.s_min(2) / t.rewrites - 30) < 0.5
    assert abs(t.counts["visits"] / t.rewrites - 3.29) < 0.01


def test_transform_count_formula():
    # seq_engine_tests.cpp:39-43, 80-88: (2^(d+1) - 1) + 26 * 2^d
    for d in (0, 1, 3, 5):
        assert O.run_seq(W.transform(d)).rewrites == (2 ** (d + 1) - 1) + 26 * 2 ** d


def test_step_budget():
    text = "sort T = A() | F(T);\nvar X : T;\neqn F(X) = F(F(X));\ninput F(A());\n"
    assert O.run_text(text, step_budget=500).status == 1
    assert O.run_seq(text, step_budget=1000).status == 1


def test_mergesort_sorts():
    # seq_engine_tests.cpp:68-78 with the independent sorting oracle
    for n in (1, 2, 10, 50):
        text = W.mergesort(n, 42)
        nums = sorted(W.generated_numerals("mergesort", n, seed=42))
        sys_words = O.run_seq(text).words[0]
        # decode Cons(peano, ...) list from canonical words
        from paper_2009_07174_b200 import api

        s = api.System(text)
        printed = s.print_words(sys_words)
        expect = "".join(f"Cons({W.peano(v)}, " for v in nums) + "Nil()" + ")" * len(nums)
        assert printed == expect


def test_workload_counts_fixture_consistent():
    """The committed algorithmic-work fixture agrees with the oracle on a shard."""
    path = os.path.join(os.path.dirname(__file__), "golden", "workload_counts.json")
    d = json.load(open(path))
    assert sum(d[f"fibbatch_s{s}"]["rewrites"] for s in range(1, 9)) == 67_968_202
    assert d["fibbatch_s1"]["rewrites"] == 8_424_285 and d["fibbatch_s1"]["sweeps"] == 1293
    assert d["sortbatch_s1"]["rewrites"] == 4_534_140 and d["sortbatch_s1"]["sweeps"] == 982
    assert d["transform22"]["rewrites"] == 117_440_511 and d["transform22"]["sweeps"] == 96
    o = O.run_text(W.fib(18), words=False)
    assert d["fib18"]["A"] == o.accesses


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(40))
def test_random_programs_match_reference(seed):
    """Random terminating systems (workloads.random_program: nested and
    multi-position patterns, first-match order, catch-alls, stuck calls):
    the C restatement and the reference's own sweep engine agree on rewrites,
    sweeps, per-sweep widths and the normal form."""
    from paper_2009_07174_b200 import workloads as W

    text = W.random_program(seed)
    o = O.run_text(text)
    r = ref.run(text, "sweep", workers=1)
    assert o.status == 0 and r.status == 0
    assert (o.rewrites, o.sweeps) == (r.rewrites, r.sweeps)
    np.testing.assert_array_equal(o.widths, r.widths)
    np.testing.assert_array_equal(o.words[0], r.words)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(30))
def test_random_wide_programs_match_reference(seed):
    """Random systems with functions of arity up to 7 (16-word records on the
    GPU): the C restatement and the reference's sweep engine agree."""
    text = W.random_program(seed, max_arity=7, nfun=5, call_depth=2, calls=32, input_depth=5)
    o = O.run_text(text)
    r = ref.run(text, "sweep", workers=1)
    assert o.status == 0 and r.status == 0
    assert (o.rewrites, o.sweeps) == (r.rewrites, r.sweeps)
    np.testing.assert_array_equal(o.widths, r.widths)
    np.testing.assert_array_equal(o.words[0], r.words)


@pytest.mark.parametrize("name", sorted(CASES))
def test_logical_restatement_matches_reference_golden(name):
    """The logical-time restatement (derive time T = max(built + 1, max
    argument nf epoch + 1), dependency order, no sweep scans) reproduces the
    reference sweep engine's trace exactly."""
    g = CASES[name]
    o = O.run_logical(g["text"])
    assert o.status == 0
    assert (o.rewrites, o.sweeps) == (g["rewrites"], g["sweeps"])
    np.testing.assert_array_equal(o.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(o.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(0, 70, 3))
def test_logical_random_programs_match_reference(seed):
    text = W.random_program(seed) if seed % 2 == 0 else W.random_program(
        seed, max_arity=7, nfun=5, call_depth=2, calls=32, input_depth=5)
    o = O.run_logical(text)
    r = ref.run(text, "sweep", workers=1)
    assert o.status == 0 and r.status == 0
    assert (o.rewrites, o.sweeps) == (r.rewrites, r.sweeps)
    np.testing.assert_array_equal(o.widths, r.widths)
    np.testing.assert_array_equal(o.words[0], r.words)


def test_logical_matches_sweep_restatement_on_batches():
    """Multi-root stores: both restatements agree per root and on widths."""
    texts = [W.fib_batch(3, roots=64), W.fib_batch(5, roots=64)]
    a, b = O.run_logical(texts), O.run_text(texts)
    assert (a.rewrites, a.sweeps) == (b.rewrites, b.sweeps)
    np.testing.assert_array_equal(a.widths, b.widths)
    for x, y in zip(a.words, b.words):
        np.testing.assert_array_equal(x, y)


def test_logical_step_budget():
    text = "sort T = A() | F(T);\nvar X : T;\neqn F(X) = F(F(X));\ninput F(A());\n"
    assert O.run_logical(text, step_budget=500).status == 1


FULLSIZE = os.path.join(os.path.dirname(__file__), "golden", "fullsize_ref.json")


@pytest.mark.skipif(not os.path.exists(FULLSIZE), reason="full-size fixture not generated")
@pytest.mark.parametrize("name", ["fib18", "reverse16k", "ackermann36", "mergesort16k", "fibbatch_s1", "sortbatch_s3"])
def test_logical_restatement_matches_fullsize_reference(name):
    """At BASELINE size the logical-time restatement reproduces the
    reference's own full-size results (tests/golden/make_fullsize.py):
    rewrites, sweeps, width-vector and normal-form hashes."""
    import hashlib

    fx = json.load(open(FULLSIZE)).get(name)
    if fx is None:
        pytest.skip(f"{name} not in the fixture yet")
    texts = {**{k: v[0] for k, v in W.CONFIGS.items()},
             "fibbatch_s1": lambda: W.fib_batch(1), "sortbatch_s3": lambda: W.treemergesort_batch(3)}
    o = O.run_logical(texts[name]())
    assert o.status == 0 and o.rewrites == fx["rewrites"]
    assert hashlib.sha1(o.words[0].astype("<u4").tobytes()).hexdigest() == fx["words_sha1"]
    if "widths_sha1" in fx:
        assert o.sweeps == fx["sweeps"]
        assert hashlib.sha1(o.widths.astype("<u8").tobytes()).hexdigest() == fx["widths_sha1"]
