"""Profiling build: per grid sweep, the slowest warp's entry time (cycles, in
the trace's free_len) against the sweep's device time, bucketed by frontier."""
import os, sys, json
os.environ["TRS_B200_PROFILE_BUILD"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np
from paper_2009_07174_b200 import api
from run_config import texts_for
name = sys.argv[1]
systems = [api.System(t) for t in texts_for(name)]
store = api.Store.load(systems)
eng = api.Engine(0); eng.set_program(systems[0])
for _ in range(2):
    eng.load(store); eng.run()
tr = eng.trace()
g = tr[tr["mode"] == 0]
act = g["active"].astype(np.int64); ns = g["ns"].astype(float); mx = g["free_len"].astype(float) / 1.965
for lo, hi in ((4096, 32768), (32768, 262144), (262144, 1 << 40)):
    sel = (act > lo) & (act <= hi)
    if sel.any():
        print(json.dumps({"name": name, "active": f"({lo},{hi}]", "sweeps": int(sel.sum()), "sweep_us": round(ns[sel].mean() / 1e3, 2),
                          "slowest_warp_us": round(mx[sel].mean() / 1e3, 2)}))
