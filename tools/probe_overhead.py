"""Fixed per-sweep overhead: grid barrier alone and barrier + frontier staging."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07174_b200 import api, workloads as W
s = api.System(W.fib(10)); st = api.Store.load(s)
e = api.Engine(0)
for variant in (1, 2):
    e.set_program(s); e.load(st); e.run(api.make_options(variant=variant))
    for mb in (0, 74, 16):
        out = {"variant": variant, "max_blocks": mb}
        for mode in (0, 1):
            e.overhead_probe(500, mode, mb)
            out[f"mode{mode}_ns"] = e.overhead_probe(5000, mode, mb)
        print(json.dumps(out), flush=True)
