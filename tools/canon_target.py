"""ncu target: config 5F run, then its device canonical relabelling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

systems = [api.System(t) for t in W.batch_shards("fib")]
store = api.Store.load(systems)
eng = api.Engine(0)
eng.set_program(systems[0])
eng.load(store)
eng.run()
c = eng.canonical_all(8, words=False)
print([int(h) for h in c["hashes"]])
