"""Multi-GPU host logic on CPU: world_size-2 `gloo` processes shard the
batched config exactly as bench.py does (no data-path collective; one
max-reduction of the timing and one sum of the rewrite counts), and the
per-rank results assemble to the single-process answer.  The oracle
stands in for the GPU run here (CPU test)."""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, roots, out):
    sys.path.insert(0, ROOT)
    import torch

    import bench
    from oracle import oracle as O
    from paper_2009_07174_b200 import workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = bench.my_seeds(rank, world, "strong")
    texts = [W.fib_batch(s, roots=roots) for s in seeds]
    res = O.run_text(texts, words=True)  # one multi-root store per rank, like the engine
    rw = torch.tensor([float(res.rewrites)])
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(rw, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"seeds": seeds, "words": [w.tolist() for w in res.words],
                                      "sweeps": int(res.sweeps)})
    if rank == 0:
        out.put({"rewrites": rw.item(), "tmax": t.item(), "parts": gathered})
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_batch_matches_single_process(world):
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    from paper_2009_07174_b200 import workloads as W

    shards, roots = 8, 4
    covered = sorted(s for r in range(world) for s in bench.my_seeds(r, world, "strong"))
    assert covered == list(range(1, shards + 1))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, roots, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = O.run_text([W.fib_batch(s, roots=roots) for s in range(1, shards + 1)])
    assert got["rewrites"] == whole.rewrites
    assert got["tmax"] == world
    words = [w for part in got["parts"] for w in part["words"]]
    assert len(words) == shards
    for a, b in zip(words, whole.words):
        assert a == b.tolist()
    # sweeps of a multi-root store = max over its independent roots
    assert max(p["sweeps"] for p in got["parts"]) == whole.sweeps


def test_partition_strong_uneven():
    """--scaling strong: one 8-shard batch split over the ranks."""
    sys.path.insert(0, ROOT)
    import bench

    for world in (1, 2, 3, 4, 8):
        seen = [s for r in range(world) for s in bench.my_seeds(r, world, "strong")]
        assert sorted(seen) == list(range(1, 9))


def test_partition_weak():
    """--scaling weak (the default): 8 shards of its own per rank, disjoint,
    seeds 8r+1..8r+8, so N ranks cover seeds 1..8N."""
    sys.path.insert(0, ROOT)
    import bench

    for world in (1, 2, 4, 8):
        per = [bench.my_seeds(r, world, "weak") for r in range(world)]
        assert all(len(p) == 8 for p in per)
        assert sorted(s for p in per for s in p) == list(range(1, 8 * world + 1))
