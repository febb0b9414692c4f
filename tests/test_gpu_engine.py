"""GPU engine behaviour through the C ABI: error model, batched roots,
device knobs that must not change results, and the full-size BASELINE
configs (bit-exact against reference-derived fixtures)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2009_07174_b200 import api
from paper_2009_07174_b200 import workloads as W

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(__file__)
CASES = json.load(open(os.path.join(HERE, "golden", "small.json")))["cases"]
COUNTS = json.load(open(os.path.join(HERE, "golden", "workload_counts.json")))


def run(engine, texts, **opts):
    return api.normalize_texts(texts, engine=engine, options=api.make_options(**opts))


def test_step_budget_raises(engine):
    # sweep_engine_tests.cpp:223-236
    text = "sort T = A() | F(T);\nvar X : T;\neqn F(X) = F(F(X));\ninput F(A());\n"
    with pytest.raises(api.EngineError) as ei:
        run(engine, text, step_budget=500)
    assert ei.value.fault == api.EngineFault.StepBudget


def test_fixed_capacity_fails_hard(engine):
    # sweep_engine_tests.cpp:203-210 (load capacity 64 with growth disabled)
    s = api.System(W.mergesort(20, 4))
    st = api.Store.load(s)
    engine.set_program(s)
    engine.load(st, capacity=st.view()["n"] + 8)
    with pytest.raises(api.EngineError) as ei:
        engine.run(api.make_options(fixed_capacity=1, disable_gc=1))
    assert ei.value.fault == api.EngineFault.Capacity


def test_fixed_capacity_with_gc_recycles(engine):
    """A tight fixed arena still completes when compaction can reclaim garbage."""
    g = CASES["mergesort64_s1"]
    s = api.System(g["text"])
    st = api.Store.load(s)
    engine.set_program(s)
    engine.load(st)
    peak = engine.run(api.make_options(disable_gc=1))["peak_slots"]
    collected = 0
    for frac in (0.8, 0.6, 0.5):
        engine.load(st, capacity=int(peak * frac))
        stats = engine.run(api.make_options(fixed_capacity=1, validate=1))
        assert stats["total_rewrites"] == g["rewrites"]
        np.testing.assert_array_equal(engine.trace()["rewrites"], np.asarray(g["widths"], np.uint64))
        np.testing.assert_array_equal(engine.canonical(0), np.asarray(g["words"], np.uint32))
        collected += stats["gc_runs"]
    assert collected > 0


def test_growth_is_invisible(engine):
    # sweep_engine_tests.cpp:212-221: a tiny initial arena grows on demand
    g = CASES["treemergesort_4_5_s7"]
    s = api.System(g["text"])
    st = api.Store.load(s)
    engine.set_program(s)
    engine.load(st, capacity=st.view()["n"] + 1)
    stats = engine.run(api.make_options(disable_gc=1))
    assert stats["regrows"] > 0 and stats["total_rewrites"] == g["rewrites"]
    np.testing.assert_array_equal(engine.trace()["rewrites"], np.asarray(g["widths"], np.uint64))


def test_explicit_capacity_below_input_fails(engine):
    s = api.System(W.fib(5))
    st = api.Store.load(s)
    engine.set_program(s)
    with pytest.raises(api.EngineError):
        engine.load(st, capacity=2)


def test_dangling_reference_detected(engine):
    s = api.System(W.mergesort(2).split("input ")[0] + "input Cons(Zero(), Cons(Zero(), Nil()));\n")
    st = api.Store.load(s)
    st.poke_arg(1, 1, 0)  # Cons's tail -> slot 0
    engine.set_program(s)
    engine.load(st)
    engine.run()
    with pytest.raises(api.EngineError) as ei:
        engine.canonical(0)
    assert ei.value.fault == api.EngineFault.DanglingReference


def test_batched_roots_equal_individual_runs(engine):
    # one store, three independent roots (same signature): fib-batch shards
    texts = [W.fib_batch(s, roots=16) for s in (1, 2, 3)]
    res = run(engine, texts)
    total = 0
    widths = None
    for k, t in enumerate(texts):
        one = run(engine, t)
        np.testing.assert_array_equal(res.words[k], one.words[0])
        total += one.total_rewrites
        w = one.widths
        widths = w if widths is None else _pad_add(widths, w)
    assert res.total_rewrites == total
    np.testing.assert_array_equal(res.widths, widths)  # independent roots: widths add per sweep


def _pad_add(a, b):
    n = max(len(a), len(b))
    out = np.zeros(n, np.uint64)
    out[: len(a)] += a
    out[: len(b)] += b
    return out


@pytest.mark.parametrize("opts", [dict(variant=2), dict(max_blocks=1), dict(small_enter=1 << 20, small_exit=1 << 20),
                                  dict(disable_small=1, gc_interval=3), dict(blocks_per_sm=1, small_enter=4),
                                  dict(profile=1), dict(disable_warp_mode=1, max_blocks=3), dict(disable_gc=1),
                                  dict(small_enter=40, small_exit=40), dict(validate=1, gc_interval=1),
                                  dict(no_runahead=1), dict(no_runahead=1, disable_small=1),
                                  dict(validate=2), dict(validate=2, gc_interval=2)])
@pytest.mark.parametrize("name", ["treemergesort_4_5_s7", "fibbatch64_s3", "unit_two_waiters", "transform6"])
def test_knobs_do_not_change_results(engine, name, opts):
    g = CASES[name]
    res = run(engine, g["text"], **opts)
    assert res.total_rewrites == g["rewrites"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))


def test_rerun_after_normal_form(engine):
    """A second run on an already-normal store: one empty sweep, zero rewrites."""
    s = api.System(CASES["fib10"]["text"])
    engine.set_program(s)
    engine.load(api.Store.load(s))
    engine.run()
    st = engine.run()
    assert st["total_rewrites"] == 0 and st["sweeps"] == 1


def test_compact_and_fetch(engine):
    g = CASES["fibbatch64_s3"]
    s = api.System(g["text"])
    engine.set_program(s)
    engine.load(api.Store.load(s))
    engine.run()
    c = engine.compact(8)
    nbytes, words = engine.fetch_records()
    assert words == 8 and nbytes == (c["live_terms"] + 1) * 32
    np.testing.assert_array_equal(engine.canonical(0), np.asarray(g["words"], np.uint32))
    # what survives is the normal form plus garbage still referenced by
    # garbage the bounded cascade has not reached yet
    assert g["nodes"] <= c["live_terms"] <= 4 * g["nodes"]


@pytest.mark.parametrize("name", ["fibbatch64_s3", "mergesort50_s42", "transform6"])
def test_fetch_store_export(engine, name):
    """Device export in the reference TermStore layout: the live store only,
    refcounts = references from exported slots + root pins (the reference's
    ghost invariant, sweep_engine.cpp:335-359), every slot reachable, and the
    canonical words of every root unchanged."""
    g = CASES[name]
    s = api.System(g["text"])
    st = api.Store.load(s)
    v = st.view()
    engine.set_program(s)
    engine.load(st)
    engine.run()
    before = [engine.canonical(k) for k in range(v["num_roots"])]
    out = engine.fetch_store(v["maxarity"], v["num_roots"])
    n = out["n"]
    arity = np.zeros(n, np.int64)
    counted = np.zeros(n, np.int64)
    for r in out["roots"]:
        counted[r] += 1
    ar_of = [s.symbol_arity(f) for f in range(s.num_symbols)]
    for y in range(1, n):
        a = ar_of[out["hss"][y]]
        arity[y] = a
        for j in range(a):
            c = out["args"][j, y]
            assert 0 < c < n
            counted[c] += 1
        for j in range(a, v["maxarity"]):
            assert out["args"][j, y] == 0
    np.testing.assert_array_equal(out["refcounts"][1:], counted[1:])
    assert (counted[1:] > 0).all()  # nothing unreachable survives
    assert out["nf"][1:].all()      # a normal form
    # the export leaves the engine state alone
    after = [engine.canonical(k) for k in range(v["num_roots"])]
    for a, b in zip(before, after):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(before[0], np.asarray(g["words"], np.uint32))


@pytest.mark.parametrize("name", ["ackermann23", "fib12", "mergesort50_s42", "reverse64", "unit_two_waiters"])
@pytest.mark.parametrize("gc_interval", [0, 3])
def test_resident_mode_is_invisible(engine, name, gc_interval):
    """The shared-memory resident arena of the single-CTA mode (with its own
    compactions) gives the same widths, rewrites and normal form as sweeping
    the store in HBM."""
    g = CASES[name]
    modes = []
    for no_resident in (0, 1):
        o = api.make_options(gc_interval=gc_interval)
        o.reserved[1] = no_resident
        res = api.normalize_texts(g["text"], engine=engine, options=o)
        modes.append(int(engine.phys_trace()["mode"].max()))  # physical sweeps: which mode ran them
        assert res.total_rewrites == g["rewrites"]
        np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
        np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))
    assert modes[0] >= 1


@pytest.mark.parametrize("k", [3, 6, 10, 20])
@pytest.mark.parametrize("mode", ["default", "grid_only", "gc3"])
def test_wide_records_against_oracle(engine, k, mode):
    """Wide symbols (W = 16 and 32 word records) and a depth-3 pattern (the
    interpreted matcher) against the C oracle restatement of the reference."""
    from oracle import oracle as port

    text = W.wide(k)
    o = port.run_text(text)
    opts = {"default": {}, "grid_only": {"disable_small": 1}, "gc3": {"gc_interval": 3}}[mode]
    res = run(engine, text, **opts)
    assert res.total_rewrites == o.rewrites and res.sweeps == o.sweeps
    np.testing.assert_array_equal(res.widths, np.asarray(o.widths, np.uint64))
    np.testing.assert_array_equal(res.words[0], o.words[0])
    assert res.stats["record_words"] == (8 if k <= 4 else 16 if k <= 8 else 32)


@pytest.mark.parametrize("nrules", [8, 32, 40])
@pytest.mark.parametrize("interp", [0, 2])
def test_many_rules_against_oracle(engine, nrules, interp):
    """A symbol with up to 40 rules (beyond the 32-rule match tables: rule
    walk), with and without the per-program specialisation, against the C
    oracle restatement of the reference."""
    from oracle import oracle as port

    text = W.many_rules(nrules)
    o = port.run_text(text)
    opts = api.make_options()
    opts.reserved[1] = interp
    res = api.normalize_texts(text, engine=engine, options=opts)
    assert res.total_rewrites == o.rewrites and res.sweeps == o.sweeps
    np.testing.assert_array_equal(res.widths, np.asarray(o.widths, np.uint64))
    np.testing.assert_array_equal(res.words[0], o.words[0])


def test_trace_records(engine):
    # sweep_engine_tests.cpp:238-255
    res = run(engine, CASES["mergesort10_s3"]["text"])
    tr = res.trace
    assert list(tr["sweep"]) == list(range(1, len(tr) + 1))
    assert len(tr) == res.sweeps and tr["rewrites"].sum() == res.total_rewrites
    assert tr["rewrites"][-1] == 0  # the empty sweep that ends the run (sweep_engine.cpp:147)
    # physical step-loop iterations: no more than the logical sweeps, and
    # together they executed every rewrite
    ph = engine.phys_trace()
    assert 1 <= len(ph) <= len(tr)
    assert list(ph["sweep"]) == list(range(1, len(ph) + 1))
    assert (ph["n"] >= 2).all() and (ph["live_terms"] >= 1).all()
    assert ph["rewrites"].sum() == res.total_rewrites
    assert engine.live_count() >= 1


@pytest.mark.parametrize("name", ["mergesort64_s1", "fib12", "ackermann23", "buildsum8", "fibbatch64_s3"])
@pytest.mark.parametrize("gc_interval", [0, 2])
def test_refcounts_recounted_equal_tracked(engine, name, gc_interval):
    """The step loop keeps refcounts only when validating; collectors and
    live_count recount them from the store (gc.cuh recount_refs).
    Without in-loop collection the store is the same either way, so the live
    count (refcount > 0) is.  With a collection every other sweep the
    collection points depend on the physical schedule (run-ahead) and a
    collection's cascade cap leaves timing-dependent garbage, so there the
    untracked run must give the reference's normal form and rewrite count,
    and a validating run on top of it (ghost invariant after the recount)
    must pass."""
    g = CASES[name]
    s = api.System(g["text"])
    st = api.Store.load(s)
    engine.set_program(s)
    counts = []
    for validate in (1, 0):
        engine.load(st)
        stats = engine.run(api.make_options(validate=validate, gc_interval=gc_interval))
        assert stats["total_rewrites"] == g["rewrites"]
        assert list(engine.canonical(0)) == g["words"]
        counts.append(engine.live_count())
    if gc_interval == 0:
        assert counts[0] == counts[1]
    engine.run(api.make_options(validate=1))  # recounts the untracked run's store first


def _sha(widths):
    return hashlib.sha1(np.asarray(widths, "<u8").tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["fib18", "transform22", "reverse16k", "ackermann36", "buildsum22"])
def test_full_size_config_widths(engine, name):
    """Full BASELINE sizes: rewrites, sweeps and the per-sweep width vector
    (sha1) equal the reference-derived fixture."""
    c = COUNTS.get(name)
    if c is None:
        pytest.skip(f"{name} not in workload_counts.json")
    res = run(engine, W.CONFIGS[name][0](), )
    assert res.total_rewrites == c["rewrites"] and res.sweeps == c["sweeps"]
    assert _sha(res.widths) == c["widths_sha1"]


def test_full_size_normal_forms(engine):
    """Size-independent properties of the full configs' normal forms."""
    s = api.System(W.fib(18))
    res = run(engine, W.fib(18))
    assert s.print_words(res.words[0]) == W.peano(2584)  # Fib(18) = 2584
    res = run(engine, W.ackermann(3, 6))
    assert api.System(W.ackermann(3, 6)).print_words(res.words[0]) == W.peano(509)
    res = run(engine, W.buildsum(22))
    assert res.total_rewrites == 33_554_404 and res.sweeps == 689
    assert api.System(W.buildsum(22)).print_words(res.words[0]) == "B0(" * 22 + "B1(Z())" + ")" * 22
    res = run(engine, W.transform(22))
    assert res.total_rewrites == (2 ** 23 - 1) + 26 * 2 ** 22  # seq_engine_tests.cpp:39-43
    words = res.words[0]
    assert len(words) == 3 * (2 ** 22 - 1) + 2 ** 22  # full binary tree of End leaves, no sharing


def test_full_size_mergesort_sorts(engine):
    """mergesort(2^14): the normal form is the independently sorted list."""
    text = W.mergesort(16384, 1)
    s = api.System(text)
    res = run(engine, text)
    assert res.total_rewrites == 4_538_513 and res.sweeps == 818_968
    nums = sorted(W.generated_numerals("mergesort", 16384, seed=1))
    expect = "".join(f"Cons({W.peano(v)}, " for v in nums) + "Nil()" + ")" * len(nums)
    assert s.print_words(res.words[0]) == expect


def test_full_size_batch_shard(engine):
    c = COUNTS["fibbatch_s1"]
    res = run(engine, W.fib_batch(1))
    assert res.total_rewrites == c["rewrites"] and res.sweeps == c["sweeps"]
    assert _sha(res.widths) == c["widths_sha1"]
    c = COUNTS["sortbatch_s1"]
    res = run(engine, W.treemergesort_batch(1))
    assert res.total_rewrites == c["rewrites"] and res.sweeps == c["sweeps"]
    assert _sha(res.widths) == c["widths_sha1"]


def test_async_run_behind_stream_gate(engine):
    """run_async + run_wait (with the whole step enqueued behind a stream
    gate) gives the same result as run, and a second pending run is refused."""
    g = CASES["mergesort64_s1"]
    s = api.System(g["text"])
    st = api.Store.load(s)
    engine.set_program(s)
    engine.load(st)
    engine.run()  # warm: modules loaded, arena sized
    engine.load(st)
    engine.hold()
    engine.run_async()
    with pytest.raises(ValueError):
        engine.run_async()  # one pending run per engine
    engine.release()
    stats = engine.run_wait()
    assert stats["total_rewrites"] == g["rewrites"]
    np.testing.assert_array_equal(engine.trace()["rewrites"], np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(engine.canonical(0), np.asarray(g["words"], np.uint32))
    with pytest.raises(ValueError):
        engine.run_wait()  # nothing pending


def test_export_after_step_budget(engine):
    """A run stopped by the step budget leaves a partial store; the export
    still writes back a consistent one (every slot reachable, refcounts =
    references from exported slots + root pins) with non-normal subterms."""
    g = CASES["fib12"]
    s = api.System(g["text"])
    st = api.Store.load(s)
    v = st.view()
    engine.set_program(s)
    engine.load(st)
    with pytest.raises(api.EngineError) as ei:
        engine.run(api.make_options(step_budget=100))
    assert ei.value.fault == api.EngineFault.StepBudget
    out = engine.fetch_store(v["maxarity"], v["num_roots"])
    n = out["n"]
    counted = np.zeros(n, np.int64)
    for r in out["roots"]:
        counted[r] += 1
    for y in range(1, n):
        for j in range(s.symbol_arity(int(out["hss"][y]))):
            c = out["args"][j, y]
            assert 0 < c < n
            counted[c] += 1
    np.testing.assert_array_equal(out["refcounts"][1:], counted[1:])
    assert (counted[1:] > 0).all()
    assert not out["nf"][1:].all()  # stopped before the normal form


@pytest.mark.parametrize("mode", ["default", "no_warp", "no_resident", "interp", "grid_only"])
@pytest.mark.parametrize("budget", [1, 10, 100, 1000])
def test_step_budget_every_mode(engine, mode, budget):
    """The budget stop is uniform in every execution mode: whichever mode the
    run is in when the total passes the budget (warp, single-CTA, resident,
    grid), the launch ends with StepBudget and the stats report the total."""
    g = CASES["fib12"]
    o = api.make_options(step_budget=budget)
    if mode == "no_warp":
        o.disable_warp_mode = 1
    if mode == "no_resident":
        o.reserved[1] = 1
    if mode == "interp":
        o.reserved[1] = 2
    if mode == "grid_only":
        o.disable_small = 1
    assert g["rewrites"] > budget
    with pytest.raises(api.EngineError) as ei:
        api.normalize_texts(g["text"], engine=engine, options=o)
    assert ei.value.fault == api.EngineFault.StepBudget


@pytest.mark.parametrize("name", ["ackermann23", "fib12", "mergesort50_s42", "reverse64", "unit_two_waiters"])
def test_no_warp_mode_is_invisible(engine, name):
    """Without the one-warp mode tiny frontiers run on the whole CTA: same
    widths, rewrites and normal form."""
    g = CASES[name]
    res = run(engine, g["text"], disable_warp_mode=1)
    assert res.total_rewrites == g["rewrites"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.parametrize("slab", [1, 7, 64, 4096])
@pytest.mark.parametrize("name", ["treemergesort_4_5_s7", "fibbatch64_s3", "unit_two_waiters"])
def test_slab_size_does_not_change_results(engine, name, slab):
    """The per-warp slab of fresh slots (allocator granularity, including
    slabs smaller than one rewrite's template) changes slot numbering only."""
    g = CASES[name]
    o = api.make_options(validate=1)
    o.reserved[2] = slab
    res = api.normalize_texts(g["text"], engine=engine, options=o)
    assert res.total_rewrites == g["rewrites"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.parametrize("mode", ["default", "grid_only", "no_warp", "gc1", "interp", "no_runahead", "validate2"])
@pytest.mark.parametrize("seed", range(40))
def test_random_programs_against_oracle(engine, seed, mode):
    """Random terminating systems (workloads.random_program; the oracle
    agrees with the reference on the same seeds, test_oracle.py) in every
    execution mode: rewrites, sweeps, per-sweep widths and the normal form."""
    from oracle import oracle as port

    text = W.random_program(seed)
    o = port.run_text(text)
    opts = {"default": {}, "grid_only": {"disable_small": 1}, "no_warp": {"disable_warp_mode": 1},
            "gc1": {"gc_interval": 1, "validate": 1}, "interp": {}, "no_runahead": {"no_runahead": 1},
            "validate2": {"validate": 2, "gc_interval": 3}}[mode]
    opt = api.make_options(**opts)
    if mode == "interp":
        opt.reserved[1] = 2
    res = api.normalize_texts(text, engine=engine, options=opt)
    assert (res.total_rewrites, res.sweeps) == (o.rewrites, o.sweeps)
    np.testing.assert_array_equal(res.widths, np.asarray(o.widths, np.uint64))
    np.testing.assert_array_equal(res.words[0], o.words[0])


@pytest.mark.parametrize("mode", ["default", "grid_only", "gc1", "interp"])
@pytest.mark.parametrize("seed", range(30))
def test_random_wide_programs_against_oracle(engine, seed, mode):
    """Random systems with arities up to 7 (16-word records when any symbol
    takes more than 4 arguments) against the oracle in several modes."""
    from oracle import oracle as port

    text = W.random_program(seed, max_arity=7, nfun=5, call_depth=2, calls=32, input_depth=5)
    o = port.run_text(text)
    opts = {"default": {}, "grid_only": {"disable_small": 1}, "gc1": {"gc_interval": 1, "validate": 1},
            "interp": {}}[mode]
    opt = api.make_options(**opts)
    if mode == "interp":
        opt.reserved[1] = 2
    res = api.normalize_texts(text, engine=engine, options=opt)
    assert (res.total_rewrites, res.sweeps) == (o.rewrites, o.sweeps)
    np.testing.assert_array_equal(res.widths, np.asarray(o.widths, np.uint64))
    np.testing.assert_array_equal(res.words[0], o.words[0])


@pytest.mark.parametrize("mode", ["default", "grid_only", "grow", "fixed_gc"])
@pytest.mark.parametrize("seed", range(20))
def test_random_program_batches_against_oracle(engine, seed, mode):
    """One random system, four inputs as the roots of one store: batch widths
    and every root's normal form against the oracle; also from a store that
    starts nearly full (growth), and with a fixed capacity that only fits by
    collecting (or fails with Capacity exactly when the oracle's does)."""
    from oracle import oracle as port

    texts = [W.random_program(seed, input_seed=k) for k in range(1, 5)]
    o = port.run_text(texts)
    s = api.System(texts[0])
    st = api.Store.load([api.System(t) for t in texts])
    n = st.view()["n"]
    engine.set_program(s)
    opts = {"grid_only": {"disable_small": 1}, "fixed_gc": {"fixed_capacity": 1, "gc_interval": 2}}.get(mode, {})
    cap = {"grow": n + 8, "fixed_gc": 2 * n + 4096}.get(mode, 0)
    engine.load(st, capacity=cap)
    stats = engine.run(api.make_options(validate=1, **opts))
    assert (stats["total_rewrites"], stats["sweeps"]) == (o.rewrites, o.sweeps)
    widths = engine.trace()["rewrites"]
    np.testing.assert_array_equal(widths, np.asarray(o.widths, np.uint64))
    for k in range(len(texts)):
        np.testing.assert_array_equal(engine.canonical(k), o.words[k])
    if mode == "grow":
        assert stats["regrows"] >= 1


@pytest.mark.parametrize("gc_interval", [0, 2])
@pytest.mark.parametrize("seed", range(20))
def test_random_program_export(engine, seed, gc_interval):
    """Device export of random batches: the live store only, the reference's
    refcount invariant over it, zeros past every arity, all nf, and the
    engine's normal forms (= the oracle's) unchanged by the export."""
    from oracle import oracle as port

    texts = [W.random_program(seed, input_seed=k) for k in range(1, 4)]
    o = port.run_text(texts)
    s = api.System(texts[0])
    st = api.Store.load([api.System(t) for t in texts])
    v = st.view()
    engine.set_program(s)
    engine.load(st)
    engine.run(api.make_options(gc_interval=gc_interval))
    out = engine.fetch_store(v["maxarity"], v["num_roots"])
    n = out["n"]
    ar_of = np.asarray([s.symbol_arity(f) for f in range(s.num_symbols)], np.int64)
    ar = ar_of[out["hss"][:n].astype(np.int64)]
    ar[0] = 0
    counted = np.bincount(np.asarray(out["roots"], np.int64), minlength=n)
    for j in range(v["maxarity"]):
        col = out["args"][j, :n].astype(np.int64)
        used = ar > j
        assert ((col > 0) & (col < n))[used].all()
        assert (col[~used] == 0).all()
        counted += np.bincount(col[used], minlength=n)
    np.testing.assert_array_equal(out["refcounts"][1:n], counted[1:])
    assert (counted[1:] > 0).all() and out["nf"][1:n].all()
    for k in range(len(texts)):
        np.testing.assert_array_equal(engine.canonical(k), o.words[k])


def test_validate2_reports_a_corrupted_store(engine):
    """validate=2 scans the store before the first sweep: a live slot whose
    argument is slot 0 is a sweep invariant violation (sweep_engine.cpp:
    341-344), reported as DanglingReference before any rewriting."""
    s = api.System(W.mergesort(2).split("input ")[0] + "input Cons(Zero(), Cons(Zero(), Nil()));\n")
    st = api.Store.load(s)
    st.poke_arg(1, 1, 0)
    engine.set_program(s)
    engine.load(st)
    with pytest.raises(api.EngineError) as ei:
        engine.run(api.make_options(validate=2))
    assert ei.value.fault == api.EngineFault.DanglingReference
    assert "sweep invariant violation" in str(ei.value)


@pytest.mark.parametrize("name", ["fibbatch_s1", "sortbatch_s1"])
def test_validate2_full_size_shard(engine, name):
    """The per-sweep device scans on a full-size config 5 shard (1,293 /
    982 scans of a multi-million-slot store) find nothing, and the run's
    results are the reference's."""
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_ref.json")))[name]
    text = W.fib_batch(1) if name.startswith("fib") else W.treemergesort_batch(1)
    res = api.normalize_texts(text, engine=engine, options=api.make_options(validate=2))
    assert res.total_rewrites == fx["rewrites"] and res.sweeps == fx["sweeps"]
    assert hashlib.sha1(res.widths.astype("<u8").tobytes()).hexdigest() == fx["widths_sha1"]


@pytest.mark.parametrize("budget", [10, 100, 1000])
def test_widths_clean_after_a_stopped_run(engine, budget):
    """A run stopped by its step budget has counted rewrites in sweeps past
    its last nf epoch; the next run on the same engine must not inherit them
    (the width histogram is cleared over everything the stopped run may have
    written)."""
    g = CASES["fib12"]
    with pytest.raises(api.EngineError):
        api.normalize_texts(g["text"], engine=engine, options=api.make_options(step_budget=budget))
    res = api.normalize_texts(g["text"], engine=engine)
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))


@pytest.mark.parametrize("name", ["reverse64", "ackermann23", "fib12", "mergesort64_s1"])
def test_runahead_engages_on_chains(engine, name, monkeypatch):
    """A latency-bound run (narrow frontiers) hands over from the lean
    synchronous build to the run-ahead build: far fewer physical sweeps than
    the reference's sweeps, and the reference's widths all the same."""
    g = CASES[name]
    if name.startswith("mergesort"):
        # 16-word records keep the synchronous build unless asked
        monkeypatch.setenv("TRS_B200_RUNAHEAD", "1")
    res = api.normalize_texts(g["text"], engine=engine)
    assert res.total_rewrites == g["rewrites"] and res.sweeps == g["sweeps"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))
    # 64 narrow sweeps in the lean build, then few physical sweeps for the rest
    assert len(engine.phys_trace()) < 64 + (g["sweeps"] - 64) // 2
    assert res.stats["launches"] >= 2  # lean build, then the run-ahead build


@pytest.mark.parametrize("name", ["transform6", "unit_chain_nf", "unit_chain_into_build"])
def test_constant_chains_in_registers(engine, name):
    """A program with constant chains (A() -> B() -> ...: transform's leaves)
    starts in the run-ahead build, which takes each chain in registers: the
    widths stay the reference's while the physical sweeps drop."""
    g = CASES[name]
    res = api.normalize_texts(g["text"], engine=engine)
    assert res.total_rewrites == g["rewrites"] and res.sweeps == g["sweeps"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))
    assert res.stats["launches"] == 1  # the run-ahead build from the start
    if name == "transform6":
        assert len(engine.phys_trace()) < g["sweeps"]


@pytest.mark.parametrize("knobs", [{}, {"no_runahead": 1}])
def test_histogram_growth_keeps_the_sweeps(knobs):
    """A fresh engine starts with a 65,536-sweep width histogram and trace;
    Ackermann(3,6) needs 344,976 sweeps, so both grow mid-run (the step loop
    exits and is relaunched, in the synchronous and the run-ahead build), and
    the sweep count and every width stay the reference's."""
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_ref.json")))["ackermann36"]
    eng = api.Engine(0)
    try:
        res = api.normalize_texts(W.ackermann(3, 6), engine=eng, options=api.make_options(**knobs))
        assert res.total_rewrites == fx["rewrites"] and res.sweeps == fx["sweeps"]
        assert hashlib.sha1(res.widths.astype("<u8").tobytes()).hexdigest() == fx["widths_sha1"]
        assert res.stats["launches"] >= 3
    finally:
        eng.close()


@pytest.mark.parametrize("define", ["-DTRS_B200_LONE=0", "-DTRS_B200_NF_CARRY=0", "-DTRS_B200_PUB_FAST=0"])
@pytest.mark.parametrize("case", ["reverse64", "fib12", "fibbatch16_s1", "random:3", "random:11"])
def test_chain_step_switches_are_invisible(engine, case, define, monkeypatch):
    """The chain-step shortcuts (lone steps, carried nf arguments, unanswered
    publications) change path length only: with each one
    compiled out, the reference's rewrites, widths and normal form stay."""
    monkeypatch.setenv("TRS_B200_JIT_DEFINES", define)
    if case.startswith("random:"):
        from oracle import oracle as port

        text = W.random_program(int(case[7:]))
        o = port.run_text(text)
        want = (o.rewrites, list(o.widths), list(o.words[0]))
    else:
        g = CASES[case]
        text = g["text"]
        want = (g["rewrites"], g["widths"], g["words"])
    res = api.normalize_texts(text, engine=engine)
    assert res.total_rewrites == want[0]
    np.testing.assert_array_equal(res.widths, np.asarray(want[1], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(want[2], np.uint32))


@pytest.mark.parametrize("past", ["1", "8"])
@pytest.mark.parametrize("name", ["fibbatch16_s1", "fib12", "treemergesort_2_3_s5"])
def test_shrinking_phase_handover_is_invisible(engine, name, past, monkeypatch):
    """An early hand-over to the run-ahead build on a steady frontier past
    the run's widest sweep (TRS_B200_RA_WARM_PAST) keeps the reference's
    rewrites, sweeps, widths and normal form."""
    monkeypatch.setenv("TRS_B200_RA_WARM_PAST", past)
    g = CASES[name]
    res = api.normalize_texts(g["text"], engine=engine)
    assert res.total_rewrites == g["rewrites"] and res.sweeps == g["sweeps"]
    np.testing.assert_array_equal(res.widths, np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))


def test_fetch_store_after_capacity_error(engine):
    """After a Capacity fault the folded bump is clamped to the capacity, so
    the write-back reads only allocated slots: fetch_store either exports a
    store within the capacity or reports an error, and the engine stays
    usable (slab fallback and export after an abort)."""
    s = api.System(W.mergesort(20, 4))
    st = api.Store.load(s)
    v = st.view()
    engine.set_program(s)
    cap = v["n"] + 8
    engine.load(st, capacity=cap)
    with pytest.raises(api.EngineError) as ei:
        engine.run(api.make_options(fixed_capacity=1, disable_gc=1, disable_small=1))
    assert ei.value.fault == api.EngineFault.Capacity
    try:
        out = engine.fetch_store(v["maxarity"], v["num_roots"])
        assert 0 < out["n"] <= cap
    except api.EngineError:
        pass
    g = CASES["fib10"]
    res = api.normalize_texts(g["text"], engine=engine)
    assert res.total_rewrites == g["rewrites"]
    np.testing.assert_array_equal(res.words[0], np.asarray(g["words"], np.uint32))


@pytest.mark.parametrize("frac", [0.9, 0.7])
def test_grid_fixed_capacity_below_slab_room(engine, frac):
    """Grid sweeps under a fixed capacity that leaves less free room than a
    slab per active warp: claims are cut at the capacity instead of failing,
    collections reclaim garbage, and the result is the reference's (or the
    run stops with Capacity, never with a wrong store)."""
    g = CASES["fibbatch16_s1"]
    s = api.System(g["text"])
    st = api.Store.load(s)
    engine.set_program(s)
    engine.load(st)
    peak = engine.run(api.make_options(disable_gc=1, disable_small=1))["peak_slots"]
    engine.load(st, capacity=int(peak * frac))
    try:
        stats = engine.run(api.make_options(fixed_capacity=1, disable_small=1, validate=1))
    except api.EngineError as e:
        assert e.fault == api.EngineFault.Capacity
        return
    assert stats["total_rewrites"] == g["rewrites"]
    np.testing.assert_array_equal(engine.trace()["rewrites"], np.asarray(g["widths"], np.uint64))
    np.testing.assert_array_equal(engine.canonical(0), np.asarray(g["words"], np.uint32))
