"""Per-sweep timeline of one workload: frontier size, rewrites, mode and
device ns of every sweep (the engine's trace records), summarised into
buckets by frontier size so the time split between wide, medium and narrow
sweeps is visible.

    python tools/sweep_timeline.py fibbatch [--save out.npy]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402
from run_config import texts_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--save", default="")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--no-resident", action="store_true")
    ap.add_argument("--slab", type=int, default=0)
    args = ap.parse_args()
    texts = texts_for(args.name)
    systems = [api.System(t) for t in texts]
    store = api.Store.load(systems)
    eng = api.Engine(0)
    eng.set_program(systems[0])
    opts = api.make_options(variant=args.variant)
    opts.reserved[1] = 1 if args.no_resident else 0
    opts.reserved[2] = args.slab
    for _ in range(2):
        eng.load(store)
        st = eng.run(opts)
    tr = eng.phys_trace()  # physical step-loop iterations
    if args.save:
        np.save(args.save, tr)
    act = tr["active"].astype(np.int64)
    ns = tr["ns"].astype(np.float64)  # device globaltimer ns per sweep
    out = {"name": args.name, "kernel_ms": st["kernel_ms"], "sweeps": int(st["sweeps"]),
           "traced_ms": float(ns.sum() * 1e-6), "buckets": []}
    edges = [0, 32, 512, 4096, 32768, 262144, 1 << 21, 1 << 40]
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = (act > lo) & (act <= hi)
        if not sel.any():
            continue
        out["buckets"].append({"active": f"({lo},{hi}]", "sweeps": int(sel.sum()),
                               "ms": round(float(ns[sel].sum() * 1e-6), 3),
                               "us_per_sweep": round(float(ns[sel].mean() * 1e-3), 2),
                               "entries": int(act[sel].sum()), "rewrites": int(tr["rewrites"][sel].sum()),
                               "ns_per_entry": round(float(ns[sel].sum() / max(1, act[sel].sum())), 3),
                               "modes": sorted(set(int(m) for m in tr["mode"][sel]))})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
