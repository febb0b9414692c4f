"""Knob combinations x small cases against the golden widths: which
execution-mode combination (if any) breaks parity."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402

cases = json.load(open(os.path.join(ROOT, "tests", "golden", "small.json")))["cases"]
names = sys.argv[1:] or ["fib12", "fib10", "ackermann23", "mergesort50_s42", "treemergesort_4_5_s7", "fibbatch64_s3"]
eng = api.Engine(0)
knobs = ["disable_warp_mode", "no_runahead", "no_resident", "disable_small", "interpreted"]
for name in names:
    g = cases[name]
    for combo in itertools.product([0, 1], repeat=len(knobs)):
        kw = {k: v for k, v in zip(knobs, combo) if v}
        bad = 0
        for rep in range(3):
            res = api.normalize_texts(g["text"], engine=eng, options=api.make_options(**kw))
            w = res.widths
            ok = res.total_rewrites == g["rewrites"] and len(w) == len(g["widths"]) and np.array_equal(
                w, np.asarray(g["widths"], np.uint64)) and list(res.words[0]) == g["words"]
            bad += not ok
        if bad:
            diff = None
            if len(w) == len(g["widths"]):
                d = np.nonzero(w != np.asarray(g["widths"], np.uint64))[0]
                diff = [int(x) for x in d[:10]]
            print(json.dumps({"name": name, "knobs": kw, "bad_of_3": bad, "first_diff_sweeps": diff}), flush=True)
print("done", flush=True)
