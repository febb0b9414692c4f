"""Step-budget stop across engine modes: each run in its own process with a
timeout, so a run that does not stop is reported instead of hanging."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CHILD = r'''
import json, sys
sys.path.insert(0, %r)
from paper_2009_07174_b200 import api
cases = json.load(open(%r))["cases"]
name, budget, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
o = api.make_options(step_budget=budget)
if mode == "no_resident": o.reserved[1] = 1
if mode == "interp": o.reserved[1] = 2
if mode == "no_warp": o.disable_warp_mode = 1
if mode == "grid_only": o.disable_small = 1
try:
    api.normalize_texts(cases[name]["text"], options=o)
    print("DONE")
except api.EngineError as e:
    print("FAULT", e.fault)
'''


def main():
    names = sys.argv[1:] or ["fib12"]
    src = CHILD % (ROOT, os.path.join(ROOT, "tests", "golden", "small.json"))
    for name in names:
        for mode in ["default", "no_resident", "interp", "no_warp", "grid_only"]:
            for budget in [1, 10, 100, 1000]:
                try:
                    r = subprocess.run([sys.executable, "-c", src, name, str(budget), mode], capture_output=True,
                                       text=True, timeout=20)
                    out = (r.stdout.strip().splitlines() or [r.stderr.strip()[-200:]])[-1]
                except subprocess.TimeoutExpired:
                    out = "HANG"
                print(json.dumps({"case": name, "mode": mode, "budget": budget, "result": out}), flush=True)


if __name__ == "__main__":
    main()
