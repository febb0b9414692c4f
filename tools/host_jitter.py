"""Host-side timing of load / run_async / run_wait / export over repeated e2e steps (JIT on and off)."""
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
L = api.lib()
p = {k: torch.from_numpy(v[k].view(np.int32)).pin_memory() for k in ("hss", "args", "refcounts")}
roots = torch.from_numpy(v["roots"].copy().view(np.int32)).pin_memory()
for jit in (0, 2):
    eng = api.Engine(0)
    eng.set_program(systems[0])
    o = api.make_options(); o.reserved[1] = jit
    rows = []
    for rep in range(14):
        t0 = time.perf_counter()
        rc = L.trs_gpu_load(eng._h, v["n"], roots.data_ptr(), roots.numel(), p["hss"].data_ptr(), p["args"].data_ptr(), v["maxarity"], p["refcounts"].data_ptr(), 0)
        t1 = time.perf_counter()
        eng.run_async(o)
        t2 = time.perf_counter()
        st = eng.run_wait()
        t3 = time.perf_counter()
        n = ctypes.c_uint32(0)
        L.trs_gpu_fetch_store(eng._h, ctypes.byref(n), None, None, None, None, None, 0)
        t4 = time.perf_counter()
        rows.append([round(1e3 * x, 2) for x in (t1 - t0, t2 - t1, t3 - t2, st["kernel_ms"], t4 - t3)])
    print(json.dumps({"jit": jit == 0, "load/async/wait/kernel/export ms": rows[4:]}))
    eng.close()
