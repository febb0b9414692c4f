"""Latency configs under each execution-mode knob: device time and the
physical sweeps per mode (0 grid, 1 single-CTA, 2 warp/solo, 3 resident)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

eng = api.Engine(0)
for name in sys.argv[1:] or ["ackermann36", "fib18"]:
    s = api.System(W.CONFIGS[name][0]())
    st = api.Store.load(s)
    eng.set_program(s)
    for knobs in ({}, {"no_runahead": 1}, {"no_resident": 1}, {"no_runahead": 1, "no_resident": 1},
                  {"no_runahead": 1, "interpreted": 1}):
        best = None
        for _ in range(2):
            eng.load(st)
            r = eng.run(api.make_options(**knobs))
            best = r if best is None or r["kernel_ms"] < best["kernel_ms"] else best
        ph = eng.phys_trace()
        modes = {int(m): int(c) for m, c in zip(*np.unique(ph["mode"], return_counts=True))}
        print(json.dumps({"name": name, "knobs": knobs, "kernel_ms": round(best["kernel_ms"], 2),
                          "sweeps": best["sweeps"], "phys": len(ph), "modes": modes,
                          "gc_runs": best["gc_runs"]}), flush=True)
