"""Raw arena consistency after a run (debugging aid): live records that
reference slot 0 or dead slots, and refcount mismatches, with reachability.
usage: arena_check.py SEED [gc_interval] [flags...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07174_b200 import api, workloads as W  # noqa: E402

seed = int(sys.argv[1])
gci = int(sys.argv[2]) if len(sys.argv) > 2 else 1
flags = set(sys.argv[3:])
text = W.random_program(seed)
s = api.System(text)
st = api.Store.load(s)
eng = api.Engine(0)
eng.set_program(s)
eng.load(st)
o = api.make_options(gc_interval=gci)
if "grid_only" in flags:
    o.disable_small = 1
if "no_resident" in flags:
    o.reserved[1] = 1
stats = eng.run(o)
nb, rw = eng.fetch_records()
buf = np.zeros(nb // 4, np.uint32)
roots = np.zeros(64, np.uint32)
eng.fetch_records(buf.ctypes.data, nb, roots.ctypes.data)
A = buf.reshape(-1, rw)
bump = stats["live_terms"] + 1
DEAD = 0xFFFFFFFF

print("stats", {k: stats[k] for k in ("sweeps", "gc_runs", "small_sweeps", "live_terms")}, "rw", rw)
mask = (1 << 24) - 1
def arity(h):
    return s.symbol_arity(int(h) & mask)
counted = np.zeros(bump, np.int64)
bad = []
for x in range(1, bump):
    h = A[x, 0]
    if h == DEAD:
        continue
    for j in range(arity(h)):
        c = A[x, 4 + j]
        if c == 0 or c >= bump or A[c, 0] == DEAD:
            bad.append((x, j, c))
        else:
            counted[c] += 1
r0 = roots[: st.view()["num_roots"]]
for r in r0:
    counted[r] += 1
reach = np.zeros(bump, bool)
stack = list(r0)
while stack:
    y = stack.pop()
    if reach[y]:
        continue
    reach[y] = True
    for j in range(arity(A[y, 0])):
        c = A[y, 4 + j]
        if 0 < c < bump and not reach[c]:
            stack.append(c)
print("bad refs", len(bad), bad[:10])
for x, j, c in bad[:5]:
    print("  rec", x, "words", A[x].tolist(), "sym", s.symbol_name(int(A[x, 0]) & mask) if hasattr(s, "symbol_name") else "",
          "reachable", bool(reach[x]), "parents", [int(y) for y in range(1, bump) if A[y, 0] != DEAD and x in A[y, 4:4 + arity(A[y, 0])]][:5])
mis = [(x, int(A[x, 2]), int(counted[x])) for x in range(1, bump) if A[x, 0] != DEAD and A[x, 2] != counted[x]]
print("rc mismatches", len(mis), mis[:10])
for x, rc, cnt in mis[:5]:
    print("  rec", x, "words", A[x].tolist(), "reachable", bool(reach[x]))
