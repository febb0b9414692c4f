"""A/B of engine knobs given as environment settings (TRS_B200_* tuning hooks,
TRS_B200_JIT_DEFINES for compile-time ones): per config, device time (best of
3) and parity against the reference fixtures, alternating the settings twice.

    KNOBS='[{}, {"TRS_B200_JIT_DEFINES": "-DTRS_B200_RA_PREFETCH=0"}]' python tools/knob_ab.py fibbatch fib18
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_07174_b200 import api  # noqa: E402
from tools.ra_compare import FX, texts  # noqa: E402

KNOBS = json.loads(os.environ.get("KNOBS", "[{}]"))


def main():
    names = sys.argv[1:] or ["fibbatch", "fibbatch_s1", "fib18", "buildsum22", "transform22", "reverse16k"]
    eng = api.Engine(0)
    base = dict(os.environ)
    for name in names:
        tx, keys = texts(name)
        systems = [api.System(t) for t in tx]
        store = api.Store.load(systems)
        fx = [FX[k] for k in keys]
        for rnd in range(2):
            for knob in KNOBS:
                os.environ.clear()
                os.environ.update(base)
                os.environ.update(knob)
                eng.set_program(systems[0])  # compile-time knobs take effect here (cached per define set)
                best = None
                for _ in range(3):
                    eng.load(store)
                    st = eng.run()
                    best = st if best is None or st["kernel_ms"] < best["kernel_ms"] else best
                canon = eng.canonical_all(len(keys), words=False)
                row = {"name": name, "knob": knob, "round": rnd, "kernel_ms": round(best["kernel_ms"], 3),
                       "phys_sweeps": len(eng.phys_trace()),
                       "rewrites_ok": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                       "words_ok": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash")
                                       for k in range(len(keys)))}
                if len(keys) == 1:
                    widths = eng.trace()["rewrites"].astype("<u8")
                    row["widths_ok"] = hashlib.sha1(widths.tobytes()).hexdigest() == fx[0]["widths_sha1"]
                print(json.dumps(row), flush=True)
    os.environ.clear()
    os.environ.update(base)
    eng.close()


if __name__ == "__main__":
    main()
