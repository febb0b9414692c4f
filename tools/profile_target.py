"""Profiling target: one warm run, then the profiled run of the same batch.

    ncu --profile-from-start off -k regex:step_loop ... python tools/profile_target.py fibbatch

The arena is pre-sized so no run regrows it; only the second, steady-state
run is inside the profiler range (cudaProfilerStart/Stop), so ncu captures
every step-loop launch of that run: the lean build and, when the run hands
over to run-ahead (kNeedRA), the run-ahead build.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_07174_b200 import api  # noqa: E402
from tools.run_config import texts_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "fibbatch"
capacity = int(sys.argv[2]) if len(sys.argv) > 2 else 128 << 20
systems = [api.System(t) for t in texts_for(name)]
store = api.Store.load(systems)
eng = api.Engine(0)
eng.set_program(systems[0])
import torch  # noqa: E402

for rep in range(2):
    eng.load(store, capacity=capacity)
    if rep == 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    st = eng.run()
    if rep == 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print(json.dumps({"rep": rep, "kernel_ms": st["kernel_ms"], "launches": st["launches"], "regrows": st["regrows"],
                      "sweeps": st["sweeps"], "rewrites": st["total_rewrites"]}), flush=True)
