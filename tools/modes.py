import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2009_07174_b200 import api, workloads as W
for name in ("fib18", "ackermann36", "reverse16k"):
    s = api.System(W.CONFIGS[name][0]()); st = api.Store.load(s); e = api.Engine(0); e.set_program(s)
    for no_res in (0, 1):
        o = api.make_options(); o.reserved[1] = no_res
        e.load(st); r = e.run(o); e.load(st); r = e.run(o)
        tr = e.trace()
        modes = {int(m): int((tr["mode"] == m).sum()) for m in np.unique(tr["mode"])}
        print(name, "no_resident" if no_res else "resident", round(r["kernel_ms"], 2), "gc", r["gc_runs"], modes, "peak", r["peak_slots"])
