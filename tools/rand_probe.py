"""Random programs (workloads.random_program) against the oracle, one
process per run so that a device fault names its seed and mode."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys
sys.path.insert(0, %r)
import numpy as np
from paper_2009_07174_b200 import api, workloads as W
from oracle import oracle as port
seed, mode = int(sys.argv[1]), sys.argv[2]
text = W.random_program(seed)
o = port.run_text(text)
flags = set(mode.split("+"))
opt = api.make_options()
if "grid_only" in flags: opt.disable_small = 1
if "no_warp" in flags: opt.disable_warp_mode = 1
if "gc1" in flags: opt.gc_interval = 1
if "gc3" in flags: opt.gc_interval = 3
if "validate" in flags: opt.validate = 1
opt.reserved[1] = (2 if "interp" in flags else 0) | (1 if "no_resident" in flags else 0)
if "slab1" in flags: opt.reserved[2] = 1
if "enter4" in flags: opt.small_enter = 4; opt.small_exit = 4
res = api.normalize_texts(text, options=opt)
ok = (res.total_rewrites, res.sweeps) == (o.rewrites, o.sweeps) and np.array_equal(res.widths, o.widths) and np.array_equal(res.words[0], o.words[0])
print("OK" if ok else "MISMATCH")
'''


def main():
    seeds = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(40)
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["default", "interp"]
    src = CHILD % ROOT
    for seed in seeds:
        for mode in modes:
            try:
                r = subprocess.run([sys.executable, "-c", src, str(seed), mode], capture_output=True, text=True,
                                   timeout=60)
                out = (r.stdout.strip().splitlines() or [""])[-1] or r.stderr.strip().splitlines()[-1][-300:]
            except subprocess.TimeoutExpired:
                out = "HANG"
            print(json.dumps({"seed": seed, "mode": mode, "result": out}), flush=True)


if __name__ == "__main__":
    main()
