"""Run-ahead on/off per BASELINE config: device time, logical and physical
sweeps, and parity (rewrites, width hash, normal-form hash) against the
reference fixture.  One JSON line per config and mode.

    python tools/ra_compare.py [names...]
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402

FX = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_ref.json")))


def texts(name):
    if name in W.CONFIGS:
        return [W.CONFIGS[name][0]()], [name]
    if name == "fibbatch":
        return W.batch_shards("fib"), [f"fibbatch_s{s}" for s in range(1, 9)]
    if name == "sortbatch":
        return W.batch_shards("sort"), [f"sortbatch_s{s}" for s in range(1, 9)]
    if name.startswith("fibbatch_s"):
        return [W.fib_batch(int(name[10:]))], [name]
    if name.startswith("sortbatch_s"):
        return [W.treemergesort_batch(int(name[11:]))], [name]
    raise KeyError(name)


def main():
    names = sys.argv[1:] or ["fib18", "ackermann36", "reverse16k", "transform22", "buildsum22", "fibbatch_s1",
                             "sortbatch_s1", "fibbatch", "sortbatch", "mergesort16k"]
    eng = api.Engine(0)
    for name in names:
        tx, keys = texts(name)
        systems = [api.System(t) for t in tx]
        store = api.Store.load(systems)
        eng.set_program(systems[0])
        ji = eng.jit_info()
        print(json.dumps({"name": name, "jit_active": ji["active"], "jit_seconds": round(ji["seconds"], 2),
                          "ptxas": [ln.strip() for ln in ji["log"].splitlines() if "registers" in ln or "spill" in ln]}),
              flush=True)
        for mode in ("runahead", "no_runahead"):
            o = api.make_options(no_runahead=(mode == "no_runahead"))
            best = None
            for _ in range(3):
                eng.load(store)
                st = eng.run(o)
                best = st if best is None or st["kernel_ms"] < best["kernel_ms"] else best
            widths = eng.trace()["rewrites"].astype("<u8")
            ph = eng.phys_trace()
            canon = eng.canonical_all(len(keys), words=False)
            fx = [FX[k] for k in keys]
            row = {"name": name, "mode": mode, "kernel_ms": round(best["kernel_ms"], 3),
                   "rewrites_ok": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                   "sweeps": st["sweeps"], "phys_sweeps": len(ph), "launches": st["launches"],
                   "small_sweeps": st["small_sweeps"], "regrows": st["regrows"],
                   "words_ok": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash") for k in range(len(keys))),
                   "rw_per_s": round(st["total_rewrites"] / (best["kernel_ms"] * 1e-3), 1)}
            if len(keys) == 1 and "widths_sha1" in fx[0]:
                row["widths_ok"] = hashlib.sha1(widths.tobytes()).hexdigest() == fx[0]["widths_sha1"]
                row["sweeps_ok"] = st["sweeps"] == fx[0]["sweeps"]
            else:
                row["sweeps_ok"] = st["sweeps"] == max(f.get("sweeps", 0) for f in fx)
            print(json.dumps(row), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
