#!/usr/bin/env python
"""Benchmark: config 5 of BASELINE.json -- batches of 4096 independent fib
roots per shard (5F; `--workload sort` for the tree-merge-sort variant 5S),
normalised on the B200 engine, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong] [--workload fib|sort]

Scaling.  The path partitions into independent roots, so ranks share no
data: by default every rank normalises 8 shards x 4096 roots of its own
(rank r: seeds 8r+1..8r+8; "weak": the per-GPU work is config 5's 8 x 4096
at every N).  `--scaling strong` splits one 8-shard batch over the ranks.

One step = one full normalisation of this rank's shards, loaded as one
multi-root store.  `value` = rewrites of all ranks / max-over-ranks device
time, inputs already resident in HBM (device SoA -> load kernel -> step
loop), L2 flushed before every step.  `e2e` = the same through the host C
ABI with pinned host buffers: H2D of the SoA store, load, step loop, device
export of the normal forms (mark, recount, renumber, pack) and their D2H in
the reference TermStore layout.  DESIGN.md "Measurement" has the byte model.
"""
import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "rewrites/sec and achieved random-gather HBM GB/s (% of roofline) vs host CPU"
COUNTS = os.path.join(ROOT, "tests", "golden", "workload_counts.json")
FULLSIZE = os.path.join(ROOT, "tests", "golden", "fullsize_ref.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "traffic.json")
SHARDS_PER_RANK = 8


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["fib", "sort"], default="fib")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="backend of the two scalar reductions (gloo lets several ranks share one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config single-GPU table")
    ap.add_argument("--cpu-sweep", action="store_true",
                    help="also time the reference sweep engine (nproc workers) on the slow configs")
    ap.add_argument("--no-gate", action="store_true",
                    help="enqueue steps without the stream gate (needed under ncu, which serialises launches)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def my_seeds(rank: int, world: int, scaling: str):
    if scaling == "weak":
        return list(range(SHARDS_PER_RANK * rank + 1, SHARDS_PER_RANK * (rank + 1) + 1))
    lo = rank * SHARDS_PER_RANK // world
    hi = (rank + 1) * SHARDS_PER_RANK // world
    return list(range(lo + 1, hi + 1))


def load_json(path):
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    d = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if d:
        return d.get("hbm_gbs", 6544.3), "measured"
    return 6650.0, "fallback"


def workload_texts(kind: str, seeds):
    from paper_2009_07174_b200 import workloads as W

    mk = W.fib_batch if kind == "fib" else W.treemergesort_batch
    return [mk(s) for s in seeds]


def cpu_baseline_reference(texts):
    """The unmodified reference seq engine (oracle/_ref), one thread per shard,
    all shards concurrently (nproc concurrent seq processes)."""
    from oracle import ref

    if ref.available():
        wall, rewrites, status = ref.run_many(texts, "seq")
        assert all(s == 0 for s in status), status
        return {"value": sum(rewrites) / wall, "unit": "rewrites/s", "cores": len(texts), "kind": "reference",
                "sample": f"{len(texts)} shards x 4096 roots, reference seq engine (seq_engine.cpp), "
                          f"one thread per shard, {wall:.2f} s wall", "seconds": wall,
                "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
    from oracle import oracle as port

    t = time.time()
    total = 0
    for tx in texts[:2]:
        total += port.run_seq(tx, words=False).rewrites
    wall = time.time() - t
    return {"value": total / wall, "unit": "rewrites/s", "cores": 1, "kind": "port",
            "sample": "2 shards through the C oracle seq restatement, 1 thread", "seconds": wall,
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}


def workload_config(args, shards_per_rank, world):
    name = "fibbatch" if args.workload == "fib" else "treemergesort-batch"
    tag = "5F" if args.workload == "fib" else "5S"
    if args.scaling == "weak":
        desc = (f"config {tag}: {name}, {shards_per_rank} shards x 4096 independent roots per GPU "
                f"(rank r: seeds 8r+1..8r+8), {world} GPU(s)")
    else:
        desc = f"config {tag}: {name} 8 shards x 4096 independent roots (seeds 1..8) split over {world} GPU(s)"
    return {"workload": desc, "shards_per_gpu": shards_per_rank, "roots_per_shard": 4096,
            "parallelism": "shards (no inter-GPU traffic)",
            "l2": "flushed between timed steps (512 MiB write on the engine stream)"}


def run_reference(args):
    """--impl reference: the reference's own CPU rewriter (oracle/_ref, the
    unmodified reference compiled from its sources) on this host's cores,
    same metric.  Each step normalises a bounded sample of the workload: as
    many shards as there are host threads (at most all shards of all ranks),
    one thread per shard, concurrently; value = rewrites / wall of the engine
    calls (bench.cpp:56-61)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtrs_ref.so not built"}))
        return
    total_shards = SHARDS_PER_RANK * world if args.scaling == "weak" else SHARDS_PER_RANK
    k = max(1, min(total_shards, os.cpu_count() or 1))
    texts = workload_texts(args.workload, list(range(1, k + 1)))
    vals = []
    for step in range(args.warmup + args.steps):
        wall, rw, st = ref.run_many(texts, "seq")
        assert all(s == 0 for s in st)
        if step >= args.warmup:
            vals.append((sum(rw), wall))
    t = sum(w for _, w in vals)
    value = sum(r for r, _ in vals) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rewrites/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(vals),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args, SHARDS_PER_RANK, world),
        "cpu_baseline": {"value": value, "unit": "rewrites/s", "cores": k, "kind": "reference",
                         "sample": f"{k} shards (seeds 1..{k}) of the workload per step, unmodified reference seq "
                                   f"engine, one thread per shard, concurrently",
                         "host_cpus": os.cpu_count(), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "rewrites/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def gather_curve(device, api):
    """The random-gather roofline over footprint, access size and gathers in
    flight per thread (trs_gpu_gather_probe_ex)."""
    out = []
    for fp in (256 << 20, 1 << 30, 4 << 30, 16 << 30):
        for b in (4, 8, 32):
            for ilp in (4, 16):
                g = api.gather_probe(device, fp, b, 2, ilp=ilp)
                out.append({"footprint_mib": fp >> 20, "bytes": b, "ilp": ilp, "gbps": round(g, 1),
                            "g_accesses_per_s": round(g / b, 2)})
    return out


def engine_accesses(c: dict) -> int:
    """Random accesses per SURVEY.md 8(d) that this engine's step loop makes:
    the model's A without its refcount RMWs (the step loop keeps no
    refcounts; the collectors recount them, gc.cuh recount_refs)."""
    return int(c["A"]) - int(c["counts"]["rc_rmw"])


def per_config_table(eng, api, W, counts, fullsize, hbm_peak, gather_gbps, cpu_sweep):
    """Single-GPU timing + bit-exact parity of every BASELINE config (one
    warm-up, best of two timed runs), with the reference's CPU engines timed
    on this host: seq (1 core, every config) and sweep (nproc workers; the
    configs it finishes in seconds unless --cpu-sweep).  Rooflines:
    `gather_frac` is the SURVEY 8(d) model (4 B x A against the measured
    uniformly random 4-B gather, A without the refcount RMWs the step loop
    skips); it can exceed 1 where accesses hit L2, so
    `dram_frac` (ncu DRAM bytes of the same launch, profiles/traffic.json,
    over the run time against the measured HBM copy bandwidth) and the
    sector efficiency (4 A + S_min) / DRAM bytes sit beside it."""
    import hashlib

    import torch

    from oracle import ref

    traffic = load_json(PROFILE_SUMMARY)
    out = {}
    nproc = os.cpu_count() or 1
    names = ["fib18", "mergesort16k", "transform22", "buildsum22", "reverse16k", "ackermann36", "sortbatch"]
    # the reference sweep engine takes minutes on these at nproc workers
    slow_sweep = {"mergesort16k", "buildsum22", "sortbatch"}
    for name in names:
        if name == "sortbatch":
            texts = W.batch_shards("sort")
            keys = [f"sortbatch_s{s}" for s in range(1, 9)]
            tkey = "sortbatch_8shards"
        else:
            texts = [W.CONFIGS[name][0]()]
            keys = [name]
            tkey = name
        t0 = time.perf_counter()
        systems = [api.System(t) for t in texts]
        t1 = time.perf_counter()
        store = api.Store.load(systems)
        t2 = time.perf_counter()
        eng.set_program(systems[0])
        best = None
        for _ in range(3):
            eng.load(store)
            st = eng.run()
            if best is None or st["kernel_ms"] < best["kernel_ms"]:
                best = st
        widths = eng.trace()["rewrites"].astype("<u8")
        canon = eng.canonical_all(len(keys), words=False)
        fx = [fullsize.get(k) for k in keys]
        cs = [counts.get(k) for k in keys]
        t = best["kernel_ms"] * 1e-3
        row = {"rewrites": best["total_rewrites"], "sweeps": best["sweeps"], "kernel_ms": best["kernel_ms"],
               "rewrites_per_s": best["total_rewrites"] / t, "us_per_sweep": 1e6 * t / best["sweeps"],
               "small_sweeps": best["small_sweeps"], "gc_runs": best["gc_runs"],
               "phys_sweeps": int(len(eng.phys_trace())),
               "host_parse_ms": round(1e3 * (t1 - t0), 2), "host_flatten_ms": round(1e3 * (t2 - t1), 2)}
        if all(fx):
            row["parity"] = {
                "rewrites": sum(f["rewrites"] for f in fx) == best["total_rewrites"],
                "words": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash") for k in range(len(keys))),
                "sweeps": max(f.get("sweeps", 0) for f in fx) == best["sweeps"],
            }
            if len(keys) == 1 and "widths_sha1" in fx[0]:
                row["parity"]["widths"] = fx[0]["widths_sha1"] == hashlib.sha1(widths.tobytes()).hexdigest()
            row["parity"]["source"] = "tests/golden/fullsize_ref.json (unmodified reference, make_fullsize.py)"
        if all(cs):
            a = sum(engine_accesses(c) for c in cs)
            smin = sum(c["S_min"] for c in cs)
            row["gather_gbps"] = 4 * a / t / 1e9
            row["gather_frac"] = row["gather_gbps"] / gather_gbps if gather_gbps else None
            row["dram_model_gbps"] = (32 * a + smin) / t / 1e9
            row["dram_model_frac"] = row["dram_model_gbps"] / hbm_peak
            t_roof = max(4 * a / (gather_gbps * 1e9) if gather_gbps else 0, smin / (hbm_peak * 1e9))
            row["t_roof_frac"] = t_roof / t
            if tkey in traffic:
                row["sector_efficiency"] = (4 * a + smin) / traffic[tkey]
        if tkey in traffic:
            row["dram_gbps"] = traffic[tkey] / t / 1e9
            row["dram_frac"] = row["dram_gbps"] / hbm_peak
        # the reference's CPU engines on this host (engine time only, bench.cpp:56-61)
        if ref.available():
            if len(texts) == 1:
                sq = ref.run(texts[0], "seq", words=False)
                row["cpu_seq_s"] = sq.micros * 1e-6
                if name not in slow_sweep or cpu_sweep:
                    sw = ref.run(texts[0], "sweep", workers=nproc, words=False)
                    row["cpu_sweep_s"] = sw.micros * 1e-6
                    row["cpu_sweep_workers"] = nproc
            else:
                wall, rw, _ = ref.run_many(texts, "seq")
                row["cpu_seq_s"] = wall
                row["cpu_seq_note"] = f"{len(texts)} shards, one thread each, concurrently"
            if "cpu_seq_s" in row:
                row["gpu_vs_cpu_seq"] = row["cpu_seq_s"] / t
        out[name] = row
        del store, systems
        torch.cuda.synchronize()
    return out


def gc_at_scale(eng, api, W, fullsize):
    """Compacting GC on the large configs: a fixed capacity below the run's
    allocation forces in-loop collections (term_store.cpp:140-157's role);
    parity and the collection time are reported."""
    out = {}
    for name, texts, keys, cap in (("buildsum22", [W.buildsum(22)], ["buildsum22"], 36 << 20),
                                   ("fibbatch", W.batch_shards("fib"), [f"fibbatch_s{s}" for s in range(1, 9)],
                                    48 << 20)):
        systems = [api.System(t) for t in texts]
        store = api.Store.load(systems)
        eng.set_program(systems[0])
        eng.load(store, capacity=cap)
        try:
            st = eng.run(api.make_options(fixed_capacity=1))
        except api.EngineError as e:
            out[name] = {"capacity_slots": cap, "error": str(e)}
            continue
        canon = eng.canonical_all(len(keys), words=False)
        fx = [fullsize.get(k) for k in keys]
        out[name] = {"capacity_slots": cap, "kernel_ms": st["kernel_ms"], "gc_runs": st["gc_runs"],
                     "gc_ms": st["gc_ms"], "peak_slots": st["peak_slots"],
                     "rewrites_match": st["total_rewrites"] == sum(f["rewrites"] for f in fx),
                     "words_match": all(str(int(canon["hashes"][k])) == fx[k].get("words_hash")
                                        for k in range(len(keys)))}
        del store, systems
    return out


def main():
    args = parse_args()
    world, rank, local = dist_env()
    from paper_2009_07174_b200 import workloads as W

    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    from paper_2009_07174_b200 import api

    ndev = torch.cuda.device_count()
    dev_index = local % max(1, ndev)  # several ranks may share a GPU (gloo)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")

    def reduce(x, op):
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=op)
        return t.item()

    seeds = my_seeds(rank, world, args.scaling)
    t_in0 = time.perf_counter()
    texts = workload_texts(args.workload, seeds)
    systems = [api.System(t) for t in texts]
    t_in1 = time.perf_counter()
    store = api.Store.load(systems)
    t_in2 = time.perf_counter()
    v = store.view()
    eng = api.Engine(dev_index)
    eng.set_program(systems[0])
    jit = eng.jit_info()
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    # device-resident inputs (value path); the e2e path reads the host store
    # itself, which the front end flattened straight into page-locked memory
    # (host/trs_host.hpp PinnedAlloc)
    d_hss = torch.from_numpy(v["hss"].view(np.int32)).to(dev)
    d_args = torch.from_numpy(v["args"].view(np.int32)).to(dev)
    d_rc = torch.from_numpy(v["refcounts"].view(np.int32)).to(dev)
    roots = v["roots"].copy()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step_value(timed=None):
        # the whole step is enqueued behind a stream gate before the device
        # starts it, so host scheduling noise stays outside the event window
        # (warm-up steps run ungated: first launches may load modules)
        gate = not args.no_gate and timed is not None
        if gate:
            eng.hold()
        if timed is not None:
            timed[0].record(stream)
        eng.load_device(v["n"], roots, d_hss.data_ptr(), d_args.data_ptr(), v["maxarity"], d_rc.data_ptr())
        eng.run_async()
        if timed is not None:
            timed[1].record(stream)
        if gate:
            eng.release()
        st = eng.run_wait()
        if timed is not None and st["launches"] > 1:
            # a relaunch (arena growth) ran after the closing event: close the
            # window after it instead (conservative: includes host time)
            timed[1].record(stream)
        return st

    # ---- warm-up (also sizes the arena once so no growth happens inside timing)
    for _ in range(args.warmup):
        step_value()
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs
    evs = []
    stats = []
    with ClockSampler(dev_index) as clocks:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            stats.append(step_value(ev))
            evs.append(ev)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    max_ms = reduce(sum(step_ms), torch.distributed.ReduceOp.MAX if world > 1 else None)
    all_rw = reduce(sum(s["total_rewrites"] for s in stats), torch.distributed.ReduceOp.SUM if world > 1 else None)
    value = all_rw / (max_ms * 1e-3)
    # load_records + load_frontier + init_ctl, then prep_launch + step loop + finish_run per launch
    launches = sum(3 + 3 * s["launches"] for s in stats)

    # ---- e2e: pinned host buffers through the C ABI: H2D of the SoA store,
    # run, and the normal form written back in the reference TermStore layout
    # (trs_gpu_fetch_store: device export + D2H of hss, args, refcounts, nf, roots)
    import ctypes

    h2d = (v["hss"].size + v["args"].size + v["refcounts"].size + v["roots"].size) * 4
    d2h_bytes, e2e_ms, e2e_host = [], [], []
    out = None
    ma = int(v["maxarity"])
    L = api.lib()
    launches_e2e = 0
    e2e_clocks = ClockSampler(dev_index)
    e2e_clocks.__enter__()
    if world > 1:
        torch.distributed.barrier()
    for k in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        th0 = time.perf_counter()
        rc = L.trs_gpu_load(eng._h, v["n"], v["roots_ptr"], v["num_roots"], v["hss_ptr"], v["args_ptr"],
                            v["maxarity"], v["rc_ptr"], 0)
        assert rc == 0, eng._err()
        th1 = time.perf_counter()
        s_run = eng.run()
        th2 = time.perf_counter()
        n_out = ctypes.c_uint32(0)
        rc = L.trs_gpu_fetch_store(eng._h, ctypes.byref(n_out), None, None, None, None, None, 0)
        th3 = time.perf_counter()
        assert rc == 0, eng._err()
        N = n_out.value
        if out is None or out["hss"].numel() < N:
            cap = int(N * 1.25) + 1024
            out = {"hss": torch.empty(cap, dtype=torch.int32).pin_memory(),
                   "args": torch.empty(max(1, ma * cap), dtype=torch.int32).pin_memory(),
                   "rc": torch.empty(cap, dtype=torch.int32).pin_memory(),
                   "nf": torch.empty(cap, dtype=torch.uint8).pin_memory(),
                   "roots": torch.empty(len(roots), dtype=torch.int32).pin_memory()}
        rc = L.trs_gpu_fetch_store(eng._h, ctypes.byref(n_out), out["roots"].data_ptr(), out["hss"].data_ptr(),
                                   out["args"].data_ptr() if ma else None, out["rc"].data_ptr(),
                                   out["nf"].data_ptr(), out["hss"].numel())
        assert rc == 0, eng._err()
        th4 = time.perf_counter()
        e1.record(stream)
        e1.synchronize()
        if k >= args.warmup:
            e2e_host.append([round(1e3 * (b - a), 3) for a, b in ((th0, th1), (th1, th2), (th2, th3), (th3, th4))])
            e2e_ms.append(e0.elapsed_time(e1))
            d2h_bytes.append(N * (4 + 4 * ma + 4 + 1) + 4 * len(roots))
            # load (3); prep + step loop + finish per launch; export; pack, in 8 slot ranges
            launches_e2e = 3 + 3 * s_run["launches"] + 1 + 8
    e2e_clocks.__exit__(None, None, None)
    e2e_max = reduce(sum(e2e_ms), torch.distributed.ReduceOp.MAX if world > 1 else None)
    e2e_value = all_rw / (e2e_max * 1e-3)

    # ---- parity of this rank's shards against the reference fixture: every
    # shard's normal form (device relabelling + hash), rewrites, sweeps
    fullsize = load_json(FULLSIZE)
    key = "fibbatch" if args.workload == "fib" else "sortbatch"
    fx = [fullsize.get(f"{key}_s{s}") for s in seeds]
    canon = eng.canonical_all(len(seeds), words=False)
    parity = None
    if all(fx):
        words_ok = [str(int(canon["hashes"][k])) == fx[k].get("words_hash") for k in range(len(seeds))]
        parity = {"shards": seeds, "words_match": words_ok,
                  "rewrites_match": int(sum(f["rewrites"] for f in fx)) == int(stats[-1]["total_rewrites"]),
                  "reference_rewrites": int(sum(f["rewrites"] for f in fx))}
        if all("sweeps" in f for f in fx):
            parity["sweeps_match"] = max(f["sweeps"] for f in fx) == int(stats[-1]["sweeps"])
    ok = 1.0 if (parity and all(parity["words_match"]) and parity["rewrites_match"]) else 0.0
    all_ok = reduce(ok, torch.distributed.ReduceOp.MIN if world > 1 else None)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    counts = load_json(COUNTS)
    hbm_peak, peak_kind = measured_peaks()
    gather_gbps = api.gather_probe(dev_index, 4 << 30, 4, 5)
    kernel_ms = statistics.mean(s["kernel_ms"] for s in stats)
    cs = [counts.get(f"{key}_s{s}") for s in seeds]
    roofline = None
    if all(cs):
        A = sum(engine_accesses(c) for c in cs)
        A_survey = sum(c["A"] for c in cs)
        smin = sum(c["S_min"] for c in cs)
        t = kernel_ms * 1e-3
        alg_bytes = 32 * A + smin
        traffic = load_json(PROFILE_SUMMARY).get(f"{key}_{len(seeds)}shards")
        roofline = {
            "bound": "hbm", "achieved": alg_bytes / t / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": alg_bytes / t / 1e9 / hbm_peak, "traffic": traffic,
            "kernel": "step_loop<8> (persistent cooperative sweep loop)",
            "algorithmic_bytes_per_launch": alg_bytes,
            "byte_model": "32 B x A (one DRAM sector per random access) + S_min (frontier streaming), "
                          "SURVEY.md 8(d); A, S_min from the C oracle (tests/golden/workload_counts.json); A = the "
                          "survey's random accesses minus the refcount RMWs this step loop does not make (refcounts "
                          "are recounted by the collectors, gc.cuh recount_refs)",
            "accesses": A, "accesses_survey_model": A_survey,
            "peak_kind": peak_kind,
            "sector_efficiency": (4 * A + smin) / traffic if traffic else None,
            "gather": {"achieved_gbps": 4 * A / t / 1e9, "roofline_gbps": gather_gbps,
                       "frac": 4 * A / t / 1e9 / gather_gbps,
                       "definition": "4 B x A / step-loop time vs measured uniformly random 4-B gather over "
                                     "4 GiB (trs_gpu_gather_probe, 4 gathers in flight per thread)",
                       "accesses_per_s": A / t, "roofline_accesses_per_s": gather_gbps * 1e9 / 4},
            "t_roof_frac": max(4 * A / (gather_gbps * 1e9), smin / (hbm_peak * 1e9)) / t,
        }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_reference(workload_texts(args.workload, list(range(1, SHARDS_PER_RANK + 1))))
    configs = gc_rows = curve = None
    if world == 1 and not args.no_configs:
        curve = gather_curve(dev_index, api)
        configs = per_config_table(eng, api, W, counts, fullsize, hbm_peak, gather_gbps, args.cpu_sweep)
        gc_rows = gc_at_scale(eng, api, W, fullsize)
    line = {
        "metric": METRIC, "value": value, "unit": "rewrites/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, len(seeds), world),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "rewrites/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": int(statistics.mean(d2h_bytes)),
                "path": "trs_gpu_load (the host SoA store, flattened by the front end straight into page-locked "
                        "memory) + trs_gpu_run + trs_gpu_fetch_store (device export: mark from the roots, recount "
                        "references, renumber; pack in slot ranges, each range's D2H of the reference TermStore "
                        "columns into pinned host memory overlapping the next range's pack), CUDA events on the "
                        "engine stream",
                "ms_per_step": statistics.mean(e2e_ms), "gpu_launches_per_step": launches_e2e,
                "step_ms": [round(x, 3) for x in e2e_ms], "clocks": e2e_clocks.summary(),
                "host_ms_load_run_export_fetch": e2e_host[-1] if e2e_host else None,
                "input_side_host_ms": {"parse_resolve": round(1e3 * (t_in1 - t_in0), 1),
                                       "flatten_to_soa": round(1e3 * (t_in2 - t_in1), 1)}},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "parity": parity, "parity_all_ranks": bool(all_ok), "rewrites_all_ranks": int(all_rw / args.steps),
        "engine": {"sweeps": stats[-1]["sweeps"], "small_sweeps": stats[-1]["small_sweeps"],
                   "gc_runs": stats[-1]["gc_runs"], "grid_blocks": stats[-1]["grid_blocks"],
                   "block_threads": stats[-1]["block_threads"], "record_words": stats[-1]["record_words"],
                   "peak_slots": stats[-1]["peak_slots"], "kernel_ms": kernel_ms, "step_ms": step_ms,
                   "jit_active": jit["active"], "nvrtc_compile_s": round(jit["seconds"], 3),
                   "dist_backend": args.dist_backend if world > 1 else None},
        "gather_curve": curve,
        "per_config": configs,
        "gc_at_scale": gc_rows,
    }
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
