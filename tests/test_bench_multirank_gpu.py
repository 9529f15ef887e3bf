"""GPU: bench.py's N > 1 paths with two torchrun ranks sharing the one visible GPU
(VATTN_BENCH_SHARED_GPU=1 -> gloo; a test hook, never a reported number).  Covers the
rendezvous, both partitions (--split batch = weak, --split bh = strong, the north_star
C5 layout), barrier + max-over-ranks timing, one JSON line from rank 0, and the
after-timing gather of every rank's slab to rank 0 with its bitwise check."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(*extra):
    env = dict(os.environ, VATTN_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_two_ranks_strong_split_gathers_and_verifies():
    line = _run("--config", "c1", "--split", "bh")
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["units_total"] == 2 and line["config"]["units_per_gpu"] == 1
    v = line["verify_gather"]
    assert v["bitwise_equal"] and v["units_checked"] == [0, 1]
    assert line["value"] > 0 and line["e2e"]["value"] > 0


def test_bench_two_ranks_weak_split():
    line = _run("--config", "c4")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["units_total"] == 2 * 8 * 16
