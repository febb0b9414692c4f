"""AoS-32B vs SoA A/B: the derive's probe pattern over the
store a BASELINE run leaves (config 5F: 80 M slots; build+sum(22)), visiting
the parents in slot order (children of fresh nodes sit near them: dense SoA
columns share sectors) and in a hashed order (no locality), timed
with CUDA events; run under ncu (-k regex:probe_) for DRAM bytes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

eng = api.Engine(0)
for name, texts in (("fibbatch", W.batch_shards("fib")), ("buildsum22", [W.buildsum(22)])):
    systems = [api.System(t) for t in texts]
    store = api.Store.load(systems)
    eng.set_program(systems[0])
    eng.load(store)
    eng.run()
    for order, base in (("slot", 0), ("random", 2)):
        aos = eng.layout_probe(base)
        soa = eng.layout_probe(base + 1)
        print(json.dumps({"name": name, "order": order, "slots": aos["slots"], "aos_ms": round(aos["ms"], 3),
                          "soa_ms": round(soa["ms"], 3), "soa_over_aos": round(soa["ms"] / aos["ms"], 2)}), flush=True)
