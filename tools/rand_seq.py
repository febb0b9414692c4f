"""Random programs in sequence on ONE engine (state carried between
programs and modes), as the pytest session runs them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07174_b200 import api, workloads as W  # noqa: E402

seeds = range(int(sys.argv[1]), int(sys.argv[2]))
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["default", "grid_only", "no_warp", "gc1", "interp"]
eng = api.Engine(0)
for seed in seeds:
    for mode in modes:
        opts = {"grid_only": {"disable_small": 1}, "no_warp": {"disable_warp_mode": 1},
                "gc1": {"gc_interval": 1, "validate": 1}}.get(mode, {})
        opt = api.make_options(**opts)
        if mode == "interp":
            opt.reserved[1] = 2
        print(seed, mode, flush=True)
        res = api.normalize_texts(W.random_program(seed), engine=eng, options=opt)
        print("  ", res.total_rewrites, res.sweeps, flush=True)
