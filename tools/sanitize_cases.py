"""Small normalisations for compute-sanitizer runs (tools/sanitize.sh): the
golden unit and family cases and random programs, in the default
(run-ahead), synchronous, grid-only, interpreted and collect-every-sweep
(refcounts kept, or recounted by the collector) modes, each checked against its fixture or the oracle so that a run that
the sanitizer lets through is also a correct one."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as port  # noqa: E402
from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

MODES = {"default": {}, "sync": {"no_runahead": 1}, "grid": {"disable_small": 1},
         "interp": {"interpreted": 1}, "gc1": {"gc_interval": 1, "validate": 1},
         "gc1u": {"gc_interval": 1},  # collect every sweep, refcounts recounted by the collector
         "validate2": {"validate": 2}}


def main():
    modes = sys.argv[1].split(",") if len(sys.argv) > 1 else list(MODES)
    nrand = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "small.json")))["cases"]
    names = ["unit_two_waiters", "unit_shared_fresh", "unit_dupvar", "transform3", "fib10", "mergesort10_s3",
             "treemergesort_2_3_s5", "ackermann22", "reverse8", "fibbatch16_s1"]
    if len(sys.argv) > 3:
        names = names[: int(sys.argv[3])]
    eng = api.Engine(0)
    bad = 0
    for mode in modes:
        for name in names:
            g = cases[name]
            res = api.normalize_texts(g["text"], engine=eng, options=api.make_options(**MODES[mode]))
            ok = (res.total_rewrites == g["rewrites"] and list(res.widths) == g["widths"]
                  and list(res.words[0]) == g["words"])
            bad += not ok
            print(f"{mode} {name} {'ok' if ok else 'MISMATCH'}", flush=True)
        for seed in range(nrand):
            text = W.random_program(seed) if seed % 2 == 0 else W.random_program(
                seed, max_arity=7, nfun=5, call_depth=2, calls=32, input_depth=5)
            o = port.run_text(text)
            res = api.normalize_texts(text, engine=eng, options=api.make_options(**MODES[mode]))
            ok = (res.total_rewrites, res.sweeps) == (o.rewrites, o.sweeps) and np.array_equal(
                res.widths, np.asarray(o.widths, np.uint64)) and np.array_equal(res.words[0], o.words[0])
            bad += not ok
            print(f"{mode} random{seed} {'ok' if ok else 'MISMATCH'}", flush=True)
    eng.close()
    print(f"cases done, {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
