"""A/B of run options (api.make_options keywords) per config: device time
(best of 3, two rounds) and parity against the reference fixtures.

    OPTS='[{}, {"disable_warp_mode": 1}]' python tools/opts_ab.py fib18 reverse16k
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_07174_b200 import api  # noqa: E402
from tools.ra_compare import FX, texts  # noqa: E402

OPTS = json.loads(os.environ.get("OPTS", "[{}]"))


def main():
    eng = api.Engine(0)
    for name in sys.argv[1:]:
        tx, keys = texts(name)
        systems = [api.System(t) for t in tx]
        store = api.Store.load(systems)
        fx = [FX[k] for k in keys]
        eng.set_program(systems[0])
        for rnd in range(2):
            for o in OPTS:
                best = None
                for _ in range(3):
                    eng.load(store)
                    st = eng.run(api.make_options(**o))
                    best = st if best is None or st["kernel_ms"] < best["kernel_ms"] else best
                canon = eng.canonical_all(len(keys), words=False)
                row = {"name": name, "opts": o, "round": rnd, "kernel_ms": round(best["kernel_ms"], 3),
                       "phys_sweeps": len(eng.phys_trace()),
                       "rewrites_ok": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                       "words_ok": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash")
                                       for k in range(len(keys)))}
                if len(keys) == 1:
                    widths = eng.trace()["rewrites"].astype("<u8")
                    row["widths_ok"] = hashlib.sha1(widths.tobytes()).hexdigest() == fx[0]["widths_sha1"]
                print(json.dumps(row), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
