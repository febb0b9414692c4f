"""Physical-sweep trace of one run (per step-loop iteration: frontier entries,
rewrites, duration, mode), condensed, to see where a run's time goes.

    python tools/tail_trace.py fibbatch1 [fibbatch ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402
from tools.run_config import texts_for  # noqa: E402

MODES = {0: "grid", 1: "cta", 2: "warp", 3: "resident"}

for name in sys.argv[1:] or ["fibbatch1"]:
    systems = [api.System(t) for t in texts_for(name)]
    store = api.Store.load(systems)
    eng = api.Engine(0)
    eng.set_program(systems[0])
    for rep in range(2):
        eng.load(store, capacity=128 << 20)
        st = eng.run()
    tr = eng.phys_trace()
    ns = tr["ns"].astype(np.float64)
    print(json.dumps({"name": name, "kernel_ms": st["kernel_ms"], "launches": st["launches"], "phys": len(tr),
                      "sum_sweep_ms": ns.sum() * 1e-6}))
    # buckets of 16 physical sweeps
    for b in range(0, len(tr), 16):
        t = tr[b:b + 16]
        print(f"{b:5d}-{b + len(t) - 1:5d} m {int(t['active'].min()):7d}..{int(t['active'].max()):7d} "
              f"rw {int(t['rewrites'].sum()):9d} ms {t["ns"].sum() * 1e-6:7.3f} "
              f"us/sweep {t["ns"].mean() * 1e-3:7.2f} modes {sorted(set(MODES.get(int(x), str(x)) for x in t['mode']))}")
