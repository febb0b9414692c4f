"""Repeat small cases many times in one mode; count parity failures (races)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402

cases = json.load(open(os.path.join(ROOT, "tests", "golden", "small.json")))["cases"]
reps = int(sys.argv[1])
kw = json.loads(sys.argv[2])
names = sys.argv[3:]
eng = api.Engine(0)
for name in names:
    g = cases[name]
    bad = 0
    diffs = []
    for rep in range(reps):
        res = api.normalize_texts(g["text"], engine=eng, options=api.make_options(**kw))
        w = res.widths
        ok = res.total_rewrites == g["rewrites"] and len(w) == len(g["widths"]) and np.array_equal(
            w, np.asarray(g["widths"], np.uint64)) and list(res.words[0]) == g["words"]
        if not ok:
            bad += 1
            if len(w) == len(g["widths"]) and len(diffs) < 3:
                d = np.nonzero(w != np.asarray(g["widths"], np.uint64))[0]
                diffs.append([(int(x), int(w[x]), int(g["widths"][x])) for x in d[:6]])
    print(json.dumps({"name": name, "knobs": kw, "reps": reps, "bad": bad, "diffs": diffs}), flush=True)
