"""Full-size parity fixtures for every BASELINE config, from the UNMODIFIED
reference (oracle/_ref/libtrs_ref.so).  TEST INFRASTRUCTURE ONLY.

    python tests/golden/make_fullsize.py [--workers N] [names...]

For each config (and each of the 8 shards of config 5F / 5S, each of which
the reference normalises as one term: a balanced Node tree of 4096 roots)
it records

  * from the reference seq engine (`normalize`, seq_engine.cpp:136-192):
    total rewrites and the SHA-1 of the canonical DAG words of the normal
    form (pre-order, first-visit ids, (symbol, child ids)
    per node), their length and node count, and the position-keyed hash
    trs_gpu_canonical_all reports per root (api.canonical_hash);
  * from the reference sweep engine (`run`, sweep_engine.cpp:69-149): the
    per-sweep width vector's SHA-1, sweep count and max width, with its
    rewrite total and normal form asserted equal to the seq engine's
    (the reference's own divergence check, bench.cpp:147-159).

Widths are schedule-independent (sweep_engine_tests.cpp:162-186), so any
worker count gives the same vector.  Results are merged into
tests/golden/fullsize_ref.json as each config finishes; `-m gpu` tests and
bench.py's parity block compare the B200 engine against them.
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2009_07174_b200 import api  # noqa: E402  (canonical_hash: a pure numpy function)
from paper_2009_07174_b200 import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fullsize_ref.json")


def configs(max_seed: int = 8):
    """BASELINE configs; shards s1..s8 of config 5, and up to max_seed for
    the weak-scaling bench (rank r of N runs seeds 8r+1..8r+8)."""
    c = {k: v[0] for k, v in W.CONFIGS.items()}
    c.update({f"fibbatch_s{s}": (lambda s=s: W.fib_batch(s)) for s in range(1, max_seed + 1)})
    c.update({f"sortbatch_s{s}": (lambda s=s: W.treemergesort_batch(s)) for s in range(1, max_seed + 1)})
    return c


def sha1(a) -> str:
    return hashlib.sha1(a.tobytes()).hexdigest()


def record(name: str, text: str, workers: int, sweep: bool) -> dict:
    t = time.time()
    sq = ref.run(text, "seq")
    assert sq.status == 0, sq.message
    words = sq.words.astype("<u4")
    row = {"rewrites": int(sq.rewrites), "words_sha1": sha1(words), "n_words": int(words.size),
           "words_hash": str(api.canonical_hash(words)),
           "nodes": int(sq.n_nodes), "seq_seconds": round(sq.micros * 1e-6, 4),
           "generator": "oracle/_ref seq normalize"}
    print(f"{name}: seq {sq.rewrites} rewrites, {sq.n_nodes} nodes, {time.time() - t:.1f}s", flush=True)
    if sweep:
        t = time.time()
        sw = ref.run(text, "sweep", workers=workers, words=True)
        assert sw.status == 0, sw.message
        assert sw.rewrites == sq.rewrites, f"{name}: reference seq/sweep rewrite divergence"
        assert sha1(sw.words.astype("<u4")) == row["words_sha1"], f"{name}: reference seq/sweep DAG divergence"
        row.update({"sweeps": int(sw.sweeps), "max_width": int(sw.max_width),
                    "widths_sha1": sha1(sw.widths.astype("<u8")), "sweep_seconds": round(sw.micros * 1e-6, 3),
                    "sweep_workers": workers, "widths_generator": "oracle/_ref sweep run"})
        print(f"{name}: sweep {sw.sweeps} sweeps, max width {sw.max_width}, {time.time() - t:.1f}s", flush=True)
    return row


def merge(name: str, row: dict) -> None:
    # several generator processes may run at once: merge under a lock
    import fcntl

    with open(OUT + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        data = {}
        if os.path.exists(OUT):
            with open(OUT) as f:
                data = json.load(f)
        data.setdefault(name, {}).update(row)
        tmp = OUT + f".tmp{os.getpid()}"
        with open(tmp, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        os.replace(tmp, OUT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--no-sweep", action="store_true", help="seq words only")
    ap.add_argument("--max-seed", type=int, default=8, help="config 5 shards up to this seed")
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    for name, fn in configs(a.max_seed).items():
        if a.names and name not in a.names:
            continue
        merge(name, record(name, fn(), a.workers, not a.no_sweep))


if __name__ == "__main__":
    main()
