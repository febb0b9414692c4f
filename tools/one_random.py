"""One random program (workloads.random_program) on the GPU: seed, mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07174_b200 import api, workloads as W  # noqa: E402

seed, mode = int(sys.argv[1]), sys.argv[2] if len(sys.argv) > 2 else "default"
opt = api.make_options(**{"grid_only": {"disable_small": 1}, "no_warp": {"disable_warp_mode": 1}}.get(mode, {}))
if mode == "interp":
    opt.reserved[1] = 2
res = api.normalize_texts(W.random_program(seed), options=opt)
print(res.total_rewrites, res.sweeps)
