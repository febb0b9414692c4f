"""Run one workload on the GPU, print stats and (optionally) parity vs the reference.

    python tools/run_config.py fib18 [--ref] [--disable-small] [--gc-interval N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if "--profile" in " ".join(sys.argv):
    os.environ.setdefault("TRS_B200_PROFILE_BUILD", "1")  # phase counters live in the profiling build

import numpy as np  # noqa: E402

from paper_2009_07174_b200 import api  # noqa: E402
from paper_2009_07174_b200 import workloads as W  # noqa: E402


def texts_for(name: str):
    if name in W.CONFIGS:
        return [W.CONFIGS[name][0]()]
    if name == "fibbatch":
        return W.batch_shards("fib")
    if name == "sortbatch":
        return W.batch_shards("sort")
    if name.startswith("fibbatchN"):
        return W.batch_shards("fib")[: int(name[len("fibbatchN"):])]
    if name.startswith("sortbatchN"):
        return W.batch_shards("sort")[: int(name[len("sortbatchN"):])]
    if name.startswith("fibbatch1"):
        return [W.fib_batch(1)]
    if name.startswith("sortbatch1"):
        return [W.treemergesort_batch(1)]
    fam, *args = name.split(":")
    return [getattr(W, fam)(*[int(a) for a in args])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--disable-small", action="store_true")
    ap.add_argument("--small-enter", type=int, default=0)
    ap.add_argument("--small-exit", type=int, default=0)
    ap.add_argument("--gc-interval", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--trace-out", default="")
    ap.add_argument("--max-blocks", type=int, default=0)
    ap.add_argument("--no-resident", action="store_true")
    ap.add_argument("--profile", type=int, nargs="?", const=1, default=0,
                    help="phase cycle accounting; N>1: only grid sweeps of <= N entries")
    args = ap.parse_args()
    texts = texts_for(args.name)
    t0 = time.time()
    systems = [api.System(t) for t in texts]
    store = api.Store.load(systems)
    t1 = time.time()
    eng = api.Engine(0)
    opts = api.make_options(disable_small=int(args.disable_small), small_enter=args.small_enter,
                            small_exit=args.small_exit, gc_interval=args.gc_interval, variant=args.variant,
                            blocks_per_sm=args.blocks_per_sm, max_blocks=args.max_blocks,
                            profile=args.profile)
    opts.reserved[1] = 1 if args.no_resident else 0
    for rep in range(args.reps):
        res = eng.normalize(systems[0], store, opts, words=(rep == args.reps - 1))
        st = res.stats
        rw = st["total_rewrites"]
        print(json.dumps({"name": args.name, "rep": rep, "rewrites": rw, "sweeps": st["sweeps"],
                          "kernel_ms": round(st["kernel_ms"], 3), "rw_per_s": rw / (st["kernel_ms"] * 1e-3),
                          "us_per_sweep": st["kernel_ms"] * 1e3 / max(1, st["sweeps"]),
                          "small_sweeps": st["small_sweeps"], "gc_runs": st["gc_runs"],
                          "gc_ms": round(st["gc_ms"], 3), "peak_slots": st["peak_slots"],
                          "grid": st["grid_blocks"], "regrows": st["regrows"], "load_ms": st["load_ms"]}),
              flush=True)
    print(f"parse+load host {t1 - t0:.2f}s", flush=True)
    if args.profile:
        pc = eng.profile_counters()
        n = max(1, pc["sweeps"])
        ns = max(1, pc["steps"])
        print(json.dumps({"cycles_per_sweep": {k: pc[k] / n for k in ("match", "claim", "apply", "push", "sweep")},
                          "cycles_per_warp_step": {k: round(pc[k] / ns) for k in ("match", "claim", "apply", "push", "m_record",
                                                                                  "m_children", "m_slots", "m_rules")},
                          "profiled_sweeps": pc["sweeps"], "warp_steps": pc["steps"],
                          "max_over_warps_per_sweep": {k[5:]: round(pc[k] / n) for k in pc if k.startswith("wmax_")}}),
              flush=True)
    if args.trace_out:
        np.save(args.trace_out, res.trace)
    if args.ref:
        from oracle import ref
        for k, t in enumerate(texts[:1]):
            r = ref.run(t, "sweep", workers=1)
            ok_w = len(r.widths) == len(res.widths) and bool((r.widths == res.widths).all()) if len(texts) == 1 else None
            ok_words = bool(np.array_equal(r.words, res.words[k]))
            print(json.dumps({"ref_rewrites": r.rewrites, "ref_sweeps": r.sweeps, "widths_equal": ok_w,
                              "words_equal": ok_words, "ref_sweep_s": r.micros * 1e-6}), flush=True)


if __name__ == "__main__":
    main()
