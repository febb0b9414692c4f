"""Profiling build: the export's phase times (clear, mark, renumber, pack) on config 5F."""
import ctypes, os, sys, json
os.environ["TRS_B200_PROFILE_BUILD"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_07174_b200 import api, workloads as W
systems = [api.System(W.fib_batch(s)) for s in range(1, 9)]
store = api.Store.load(systems)
eng = api.Engine(0); eng.set_program(systems[0])
for rep in range(2):
    eng.load(store); eng.run()
    n = ctypes.c_uint32(0)
    api.lib().trs_gpu_fetch_store(eng._h, ctypes.byref(n), None, None, None, None, None, 0)
    pc = eng.profile_counters()
    print(json.dumps({"n": n.value, "clear_ms": pc["gc_claim_ns"] / 1e6, "mark_ms": pc["gc_count_ns"] / 1e6,
                      "renumber_ms": pc["gc_scatter_ns"] / 1e6, "pack_ms": pc["gc_remap_ns"] / 1e6}))
