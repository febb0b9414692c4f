"""A/B of refcount maintenance in the step loop (TRS_B200_TRACK_RC=1 keeps
them rewrite by rewrite, the default recounts them only for a collector):
device time best of 3 and parity per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_07174_b200 import api  # noqa: E402
from tools.ra_compare import FX, texts  # noqa: E402

names = sys.argv[1:] or ["fibbatch", "sortbatch", "buildsum22", "transform22", "fibbatch_s1"]
eng = api.Engine(0)
for name in names:
    tx, keys = texts(name)
    systems = [api.System(t) for t in tx]
    store = api.Store.load(systems)
    eng.set_program(systems[0])
    fx = [FX[k] for k in keys]
    for track in ("1", "0", "1", "0"):
        os.environ["TRS_B200_TRACK_RC"] = track
        ms = []
        for _ in range(3):
            eng.load(store)
            st = eng.run()
            ms.append(st["kernel_ms"])
        canon = eng.canonical_all(len(keys), words=False)
        print(json.dumps({"name": name, "track_rc": track, "kernel_ms": round(min(ms), 3), "gc_runs": st["gc_runs"],
                          "rewrites_ok": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                          "words_ok": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash")
                                          for k in range(len(keys)))}), flush=True)
eng.close()
