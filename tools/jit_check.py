"""Specialised vs interpreted step loop: compile info, parity and time per workload."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np
from paper_2009_07174_b200 import api
from run_config import texts_for
for name in sys.argv[1:]:
    systems = [api.System(t) for t in texts_for(name)]
    store = api.Store.load(systems)
    eng = api.Engine(0)
    eng.set_program(systems[0])
    info = eng.jit_info()
    out = {"name": name, "jit": info["active"], "compile_s": round(info["seconds"], 2)}
    if not info["active"]:
        out["log"] = info["log"][-2000:]
    for label, flag in (("jit", 0), ("interp", 2)):
        o = api.make_options()
        o.reserved[1] = flag
        best = None
        for _ in range(2):
            eng.load(store)
            st = eng.run(o)
            best = st
        tr = eng.trace()
        out[label] = {"ms": round(best["kernel_ms"], 3), "rw": best["total_rewrites"], "sweeps": best["sweeps"],
                      "wsum": int(tr["rewrites"].astype(np.int64).sum())}
    print(json.dumps(out), flush=True)
    eng.close()
