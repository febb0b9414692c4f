#!/usr/bin/env python
"""Benchmark: config 5 of BASELINE.json -- 8 shards x 4096 independent fib
roots (5F; `--workload sort` for the tree-merge-sort variant 5S), normalised
on the B200 engine, shards split across the ranks (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full normalisation of this rank's shards (all roots loaded as
one multi-root store).  `value` = rewrites of all ranks / max-over-ranks
device time, inputs already resident in HBM (device SoA -> engine load
kernel -> step loop), L2 flushed before every step.  `e2e` = the same
through the host C ABI with pinned host buffers: H2D of the SoA store, load,
step loop, device compaction, D2H of the normal-form arena.
"Measurement" for the roofline byte model.
"""
import argparse
import json
import os
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
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "traffic.json")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["fib", "sort"], default="fib")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config single-GPU table")
    ap.add_argument("--configs-only", action="store_true")
    ap.add_argument("--no-gate", action="store_true",
                    help="enqueue steps without the stream gate (needed under ncu, which serialises launches)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def my_shards(rank: int, world: int, total: int = 8):
    lo = rank * total // world
    hi = (rank + 1) * total // world
    return list(range(lo + 1, hi + 1))  # seeds


def load_counts():
    if os.path.exists(COUNTS):
        with open(COUNTS) as f:
            return json.load(f)
    return {}


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
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6544.3), "measured"
    return 6650.0, "fallback"


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
                "host_cpus": os.cpu_count()}
    from oracle import oracle as port

    t = time.time()
    total = 0
    for tx in texts[:2]:
        total += port.run_seq(tx, words=False).rewrites
    wall = time.time() - t
    return {"value": total / wall, "unit": "rewrites/s", "cores": 1, "kind": "port",
            "sample": "2 shards through the C oracle seq restatement, 1 thread", "seconds": wall,
            "host_cpus": os.cpu_count()}


def run_reference(args, texts_all):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtrs_ref.so not built"}))
        return
    vals = []
    total_rw = 0
    for k in range(args.warmup + args.steps):
        wall, rw, st = ref.run_many(texts_all, "seq")
        assert all(s == 0 for s in st)
        if k >= args.warmup:
            vals.append((sum(rw), wall))
            total_rw = sum(rw)
    t = sum(w for _, w in vals)
    value = sum(r for r, _ in vals) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rewrites/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(vals),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args, len(texts_all)),
        "cpu_baseline": {"value": value, "unit": "rewrites/s", "cores": len(texts_all), "kind": "reference",
                         "sample": f"{len(texts_all)} shards, unmodified reference seq engine, one thread per "
                                   f"shard, full workload per step ({total_rw} rewrites)",
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "rewrites/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(args, nshards):
    name = "fibbatch" if args.workload == "fib" else "treemergesort-batch"
    return {"workload": f"config 5{'F' if args.workload == 'fib' else 'S'}: {name} {nshards} shards x 4096 "
                        f"independent roots (seeds 1..{nshards})",
            "shards": nshards, "roots_per_shard": 4096, "parallelism": "shards (no inter-GPU traffic)",
            "l2": "flushed between timed steps (512 MiB write on the engine stream)"}


def per_config_table(eng, api, W, counts, hbm_peak, gather_gbps):
    """Single-GPU timing + parity of every BASELINE config (one warm-up, one
    timed run).  Rooflines: `gather_frac` is the SURVEY 8(d) model (4 B x A
    against the measured uniformly random 4-B gather); it can exceed 1 where
    part of the accesses hit L2 (build+sum: ~50 % L2 hit rate in ncu), so
    `dram_frac` -- the ncu-measured DRAM bytes of the same launch
    (profiles/traffic.json) over the run time, against the measured HBM copy
    bandwidth -- is given beside it where a capture exists."""
    import hashlib

    import torch

    traffic = {}
    if os.path.exists(PROFILE_SUMMARY):
        with open(PROFILE_SUMMARY) as f:
            traffic = json.load(f)
    out = {}
    names = ["fib18", "mergesort16k", "transform22", "buildsum22", "reverse16k", "ackermann36", "sortbatch"]
    for name in names:
        if name == "sortbatch":
            texts = [W.treemergesort_batch(s) for s in range(1, 9)]
            systems = [api.System(t) for t in texts]
            sysm = systems[0]
            store = api.Store.load(systems)
            keys = [f"sortbatch_s{s}" for s in range(1, 9)]
            tkey = "sortbatch_8shards"
        else:
            sysm = api.System(W.CONFIGS[name][0]())
            store = api.Store.load(sysm)
            keys = [name]
            tkey = name
        eng.set_program(sysm)
        best = None
        for rep in range(2):
            eng.load(store)
            st = eng.run()
            best = st
        tr = eng.trace()
        widths = tr["rewrites"].astype("<u8")
        cs = [counts.get(k) for k in keys]
        t = best["kernel_ms"] * 1e-3
        row = {"rewrites": best["total_rewrites"], "sweeps": best["sweeps"], "kernel_ms": best["kernel_ms"],
               "rewrites_per_s": best["total_rewrites"] / t, "us_per_sweep": 1e6 * t / best["sweeps"],
               "small_sweeps": best["small_sweeps"], "gc_runs": best["gc_runs"]}
        if all(cs):
            row["parity_rewrites"] = sum(c["rewrites"] for c in cs) == best["total_rewrites"]
            if len(cs) == 1:
                row["parity_widths"] = cs[0]["widths_sha1"] == hashlib.sha1(widths.tobytes()).hexdigest()
            else:
                row["parity_sweeps"] = max(c["sweeps"] for c in cs) == best["sweeps"]
            a = sum(c["A"] for c in cs)
            smin = sum(c["S_min"] for c in cs)
            row["gather_gbps"] = 4 * a / t / 1e9
            row["gather_frac"] = row["gather_gbps"] / gather_gbps if gather_gbps else None
            row["dram_model_gbps"] = (32 * a + smin) / t / 1e9
            row["dram_model_frac"] = row["dram_model_gbps"] / hbm_peak
            t_roof = max(4 * a / (gather_gbps * 1e9) if gather_gbps else 0, smin / (hbm_peak * 1e9))
            row["t_roof_frac"] = t_roof / t
        if tkey in traffic:
            row["dram_gbps"] = traffic[tkey] / t / 1e9
            row["dram_frac"] = row["dram_gbps"] / hbm_peak
        out[name] = row
        del store, sysm
        torch.cuda.synchronize()
    return out


def main():
    args = parse_args()
    world, rank, local = dist_env()
    from paper_2009_07174_b200 import workloads as W

    kind = args.workload
    seeds_all = list(range(1, 9))
    mk = W.fib_batch if kind == "fib" else W.treemergesort_batch
    if args.impl == "reference":
        run_reference(args, [mk(s) for s in seeds_all])
        return

    import torch

    from paper_2009_07174_b200 import api

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    seeds = my_shards(rank, world)
    texts = [mk(s) for s in seeds]
    systems = [api.System(t) for t in texts]
    store = api.Store.load(systems)
    v = store.view()
    eng = api.Engine(local)
    eng.set_program(systems[0])
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # device-resident inputs (value path) and pinned host inputs (e2e path)
    d_hss = torch.from_numpy(v["hss"].view(np.int32)).to(dev)
    d_args = torch.from_numpy(v["args"].view(np.int32)).to(dev)
    d_rc = torch.from_numpy(v["refcounts"].view(np.int32)).to(dev)
    roots = v["roots"].copy()
    p_hss = torch.from_numpy(v["hss"].view(np.int32)).pin_memory()
    p_args = torch.from_numpy(v["args"].view(np.int32)).pin_memory()
    p_rc = torch.from_numpy(v["refcounts"].view(np.int32)).pin_memory()
    p_roots = torch.from_numpy(roots.view(np.int32)).pin_memory()
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
        st = step_value()
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs
    evs = []
    stats = []
    with ClockSampler(local) as clocks:
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
    my_ms = sum(step_ms)
    my_rewrites = sum(s["total_rewrites"] for s in stats)
    tot = torch.tensor([my_ms], dtype=torch.float64, device=dev)
    rw = torch.tensor([my_rewrites], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(rw, op=torch.distributed.ReduceOp.SUM)
    max_ms = tot.item()
    all_rw = rw.item()
    value = all_rw / (max_ms * 1e-3)
    # load_records + load_frontier + init_ctl, then prep_launch + step loop per launch
    launches = sum(3 + 2 * s["launches"] for s in stats)

    # ---- e2e: pinned host buffers through the C ABI: H2D of the SoA store,
    # run, and the normal form written back in the reference TermStore layout
    # (trs_gpu_fetch_store: device compaction + pack + D2H of hss, args,
    # refcounts, nf and roots)
    h2d = (p_hss.numel() + p_args.numel() + p_rc.numel() + p_roots.numel()) * 4
    d2h_bytes = []
    e2e_ms = []
    e2e_host = []  # host ms of load, run, export, fetch per step (diagnostics)
    out = None
    ma = int(v["maxarity"])
    L = api.lib()
    import ctypes
    e2e_clocks = ClockSampler(local)
    e2e_clocks.__enter__()
    for k in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        th0 = time.perf_counter()
        rc = L.trs_gpu_load(eng._h, v["n"], p_roots.data_ptr(), len(roots), p_hss.data_ptr(),
                            p_args.data_ptr(), v["maxarity"], p_rc.data_ptr(), 0)
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
            launches_e2e = 3 + 2 * s_run["launches"] + 2  # load (3), prep + step loop(s), compaction, pack
    e2e_clocks.__exit__(None, None, None)
    e2e_tot = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_tot, op=torch.distributed.ReduceOp.MAX)
    e2e_value = all_rw / (e2e_tot.item() * 1e-3)

    # parity of this rank's shards against the reference-derived fixture
    counts = load_counts()
    key = "fibbatch" if kind == "fib" else "sortbatch"
    fx = [counts.get(f"{key}_s{s}") for s in seeds]
    parity = None
    if all(fx):
        parity = {"rewrites_match": int(sum(c["rewrites"] for c in fx)) == int(stats[-1]["total_rewrites"]),
                  "reference_rewrites": int(sum(c["rewrites"] for c in fx)),
                  "sweeps_match": max(c["sweeps"] for c in fx) == int(stats[-1]["sweeps"])}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    hbm_peak, peak_kind = measured_peaks()
    gather_gbps = api.gather_probe(local, 4 << 30, 4, 5)
    # the same probe at 8/16/32 bytes per access: the random-access rate is
    # the limit (flat up to 16 B), not bytes
    gather_wide = {f"{b}B_gbps": api.gather_probe(local, 4 << 30, b, 3) for b in (8, 16, 32)}
    kernel_ms = statistics.mean(s["kernel_ms"] for s in stats)
    roofline = None
    if all(fx):
        A = sum(c["A"] for c in fx)
        smin = sum(c["S_min"] for c in fx)
        t = kernel_ms * 1e-3
        alg_bytes = 32 * A + smin
        traffic = None
        if os.path.exists(PROFILE_SUMMARY):
            with open(PROFILE_SUMMARY) as f:
                traffic = json.load(f).get(f"{key}_{len(seeds)}shards")
        roofline = {
            "bound": "hbm", "achieved": alg_bytes / t / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": alg_bytes / t / 1e9 / hbm_peak, "traffic": traffic,
            "kernel": "step_loop<8> (persistent cooperative sweep loop)",
            "algorithmic_bytes_per_launch": alg_bytes,
            "byte_model": "32 B x A (one DRAM sector per random access) + S_min (frontier streaming), "
                          "SURVEY.md 8(d); A, S_min from the C oracle (tests/golden/workload_counts.json)",
            "peak_kind": peak_kind,
            "gather": {"achieved_gbps": 4 * A / t / 1e9, "roofline_gbps": gather_gbps,
                       "frac": 4 * A / t / 1e9 / gather_gbps,
                       "definition": "4 B x A / step-loop time vs measured uniformly random 4-B gather over "
                                     "4 GiB (trs_gpu_gather_probe)",
                       "accesses_per_s": A / t, "roofline_accesses_per_s": gather_gbps * 1e9 / 4,
                       "probe_wider": gather_wide},
            "t_roof_frac": max(4 * A / (gather_gbps * 1e9), smin / (hbm_peak * 1e9)) / t,
        }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_reference([mk(s) for s in seeds_all])
    configs = None
    if world == 1 and not args.no_configs:
        configs = per_config_table(eng, api, W, counts, hbm_peak, gather_gbps)
    line = {
        "metric": METRIC, "value": value, "unit": "rewrites/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, 8),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "rewrites/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": int(statistics.mean(d2h_bytes)),
                "path": "trs_gpu_load (pinned host SoA) + trs_gpu_run + trs_gpu_fetch_store (device export: "
                        "mark from the roots, recount references, renumber, pack; D2H of the reference TermStore "
                        "columns into pinned host memory), CUDA events on the engine stream", "ms_per_step": statistics.mean(e2e_ms),
                "gpu_launches_per_step": launches_e2e,
                "step_ms": [round(x, 3) for x in e2e_ms],
                "clocks": e2e_clocks.summary(),
                "host_ms_load_run_export_fetch": e2e_host[-1] if e2e_host else None},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "parity": parity,
        "engine": {"sweeps": stats[-1]["sweeps"], "small_sweeps": stats[-1]["small_sweeps"],
                   "gc_runs": stats[-1]["gc_runs"], "grid_blocks": stats[-1]["grid_blocks"],
                   "block_threads": stats[-1]["block_threads"], "record_words": stats[-1]["record_words"],
                   "peak_slots": stats[-1]["peak_slots"], "kernel_ms": kernel_ms,
                   "step_ms": step_ms},
        "per_config": configs,
    }
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
