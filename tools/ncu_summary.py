"""Summarise the ncu captures of tools/gpu_profiles.sh into profiles/r1_ncu_summary.txt and
profiles/traffic.json (DRAM bytes per launch, read by bench.py as roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'smsp__inst_executed.sum',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio']
NAMES = {"fibbatch": ("config 5F fib batch, 8 shards", "fibbatch_8shards"),
         "sortbatch": ("config 5S tree-merge-sort batch, 8 shards", "sortbatch_8shards"),
         "buildsum22": ("config 3b build+sum depth 22", "buildsum22"),
         "transform22": ("config 3a transform depth 22", "transform22"),
         "fib18": ("config 1 fib(18)", "fib18"),
         "fibbatch1": ("config 5F, one shard (the strong-scaling 8-GPU point)", "fibbatch_1shard"),
         "export": ("normal-form export of config 5F (trs_gpu_fetch_store)", "export_fibbatch_8shards"),
         "canon": ("device canonical relabelling of config 5F (canon_down)", "canon_fibbatch_8shards"),
         "probe": ("random 4-byte gather probe over 4 GiB (the roofline)", "gather_probe_4B_4GiB")}
SCALE = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    tag = sys.argv[2] if len(sys.argv) > 2 else "r1"
    out = [f"# {tag} ncu summaries (specialised step loop): ncu --set full --clock-control none --import-source on",
           "# one steady-state launch each; captured with tools/gpu_profiles*.sh, summarised by tools/ncu_summary.py",
           "#   step_loop: python tools/profile_target.py <workload>   (--profile-from-start off -k regex:step_loop: every launch of the 2nd run)",
           "#   export_store: python tools/e2e_parts.py                (-k regex:export_store -c 1)",
           "# ncu times are replayed/serialised: compare shares, not absolutes", ""]
    traffic = {}
    if os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)
    for c, (desc, key) in NAMES.items():
        rep = os.path.join(src, f"ncu_{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(r.splitlines()))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        launches = [v for v in rows[2:] if len(v) == len(h)]
        names = ", ".join(v[h.index('Kernel Name')] for v in launches)
        out.append(f"## {c}: {desc}  ({len(launches)} launch(es) of one run: {names})")
        total = 0.0
        for n, v in enumerate(launches):
            if len(launches) > 1:
                out.append(f"# launch {n}: {v[h.index('Kernel Name')]}")
            for w in WANT:
                i = h.index(w)
                out.append(f"{w:80s} {v[i]:>22s} {u[i]}")
            rd = float(v[h.index('dram__bytes_read.sum')]) * SCALE[u[h.index('dram__bytes_read.sum')]]
            wr = float(v[h.index('dram__bytes_write.sum')]) * SCALE[u[h.index('dram__bytes_write.sum')]]
            out.append(f"{'dram bytes of this launch (read+write)':80s} {rd + wr:22.4e} byte")
            total += rd + wr
        out.append(f"{'dram bytes per run (all launches, read+write)':80s} {total:22.4e} byte")
        out.append("")
        traffic[key] = total
    dest = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles")
    os.makedirs(dest, exist_ok=True)
    with open(os.path.join(dest, f"{tag}_ncu_summary.txt"), "w") as f:
        f.write("\n".join(out))
    with open(os.path.join(dest, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
