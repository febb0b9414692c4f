"""The multi-rank bench path on real hardware: two ranks (torchrun, one
process per rank) sharing the one metered B200, their scalar reductions over
gloo.  Each rank normalises its own shards through the engine and checks
every shard's normal form against the reference fixture (bench.py's parity
block, MIN-reduced over the ranks); the SUM of the rewrites over the ranks
is the batch's (67,968,202 for the 8 fib shards)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(scaling: str) -> dict:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--dist-backend", "gloo", "--no-configs",
           "--no-cpu-baseline", "--scaling", scaling]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_two_ranks_strong_scaling_sum_and_parity():
    d = _bench("strong")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["rewrites_all_ranks"] == 67_968_202
    assert d["parity_all_ranks"] is True
    assert d["parity"]["shards"] == [1, 2, 3, 4] and all(d["parity"]["words_match"])


def test_two_ranks_weak_scaling_parity():
    d = _bench("weak")
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["parity"]["shards"] == list(range(1, 9)) and all(d["parity"]["words_match"])
    assert d["parity_all_ranks"] is True  # rank 1's shards 9..16 against their reference fixtures
    assert d["value"] > 0 and d["e2e"]["value"] > 0
