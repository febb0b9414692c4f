"""Time the parts of the e2e path (H2D+load, run, compaction, pack+D2H) for config 5F."""
import ctypes, os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2009_07174_b200 import api, workloads as W
texts = [W.fib_batch(s) for s in range(1, 9)]
systems = [api.System(t) for t in texts]
store = api.Store.load(systems)
v = store.view()
eng = api.Engine(0)
eng.set_program(systems[0])
L = api.lib()
p = {k: torch.from_numpy(v[k].view(np.int32)).pin_memory() for k in ("hss", "args", "refcounts")}
roots = torch.from_numpy(v["roots"].copy().view(np.int32)).pin_memory()
out = None
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = L.trs_gpu_load(eng._h, v["n"], roots.data_ptr(), roots.numel(), p["hss"].data_ptr(),
                        p["args"].data_ptr(), v["maxarity"], p["refcounts"].data_ptr(), 0)
    assert rc == 0
    t1 = time.perf_counter()
    st = eng.run()
    t2 = time.perf_counter()
    sc = eng.compact(8) if os.environ.get("COMPACT") == "1" else {"gc_runs": 0, "gc_ms": 0, "live_terms": 0}
    t3 = time.perf_counter()
    n = ctypes.c_uint32(0)
    L.trs_gpu_fetch_store(eng._h, ctypes.byref(n), None, None, None, None, None, 0)
    N = n.value
    if out is None:
        out = [torch.empty(N * 2, dtype=torch.int32).pin_memory() for _ in range(4)]
    t4 = time.perf_counter()
    L.trs_gpu_fetch_store(eng._h, ctypes.byref(n), None, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
                          out[3].data_ptr(), N * 2)
    t5 = time.perf_counter()
    print(json.dumps({"load_ms": (t1 - t0) * 1e3, "run_ms": (t2 - t1) * 1e3, "kernel_ms": st["kernel_ms"],
                      "compact_ms": (t3 - t2) * 1e3, "compact": {k: sc[k] for k in ("gc_runs", "gc_ms", "live_terms")},
                      "query_ms": (t4 - t3) * 1e3, "pack_d2h_ms": (t5 - t4) * 1e3, "N": N}), flush=True)
if os.environ.get("TRS_B200_PROFILE_BUILD") == "1":
    print(json.dumps({k: v for k, v in eng.profile_counters().items() if k.startswith("gc")}))
