"""Run-ahead tuning sweep: per config, device time (best of 3) and parity
(rewrites, per-root canonical hashes, width hash) under settings of the
TRS_B200_RA_* tuning hooks (read by trs_gpu_run on every run).

    python tools/ra_sweep.py [names...]
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_07174_b200 import api  # noqa: E402
from tools.ra_compare import FX, texts  # noqa: E402

WARPS = 148 * 16
# (ra_max per warp, ra_kill per warp, ra_steps, ra_warm)
SETTINGS = [(4, 8, 8, 64), (8, 16, 8, 64), (16, 32, 8, 64), (32, 64, 8, 64), (16, 32, 16, 64), (16, 32, 32, 64),
            (32, 64, 32, 64), (16, 32, 8, 16), (32, 64, 16, 16)]
if os.environ.get("RA_SWEEP_SETTINGS"):
    SETTINGS = [tuple(x) for x in json.loads(os.environ["RA_SWEEP_SETTINGS"])]


def main():
    names = sys.argv[1:] or ["fibbatch", "fibbatch_s1", "fib18", "buildsum22", "transform22", "reverse16k"]
    eng = api.Engine(0)
    for name in names:
        tx, keys = texts(name)
        systems = [api.System(t) for t in tx]
        store = api.Store.load(systems)
        eng.set_program(systems[0])
        fx = [FX[k] for k in keys]
        for (mx, kill, steps, warm) in SETTINGS:
            os.environ["TRS_B200_RA_MAX"] = str(mx * WARPS)
            os.environ["TRS_B200_RA_KILL"] = str(kill * WARPS)
            os.environ["TRS_B200_RA_STEPS"] = str(steps)
            os.environ["TRS_B200_RA_WARM"] = str(warm)
            best = None
            for _ in range(3):
                eng.load(store)
                st = eng.run()
                best = st if best is None or st["kernel_ms"] < best["kernel_ms"] else best
            canon = eng.canonical_all(len(keys), words=False)
            row = {"name": name, "ra_max_w": mx, "ra_kill_w": kill, "ra_steps": steps, "ra_warm": warm,
                   "kernel_ms": round(best["kernel_ms"], 3), "phys_sweeps": len(eng.phys_trace()),
                   "launches": st["launches"],
                   "rewrites_ok": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                   "words_ok": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash") for k in range(len(keys)))}
            if len(keys) == 1:
                widths = eng.trace()["rewrites"].astype("<u8")
                row["widths_ok"] = hashlib.sha1(widths.tobytes()).hexdigest() == fx[0]["widths_sha1"]
            print(json.dumps(row), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
