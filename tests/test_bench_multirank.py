"""bench.py's N > 1 code path (row shards + all-gather, k-split + all-reduce,
the reference arm under torchrun) exercised end to end on a one-GPU box:
both ranks share cuda:0 and the collectives run host-staged over gloo
(MSG_BENCH_SHARE_GPU=1).  A functional check of the plumbing the driver's
scaling run uses, never a measurement."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(*args):
    env = dict(os.environ, MSG_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 prints one JSON line
    return json.loads(lines[0])


@pytest.mark.parametrize("split", ["rows", "k"])
def test_bench_two_ranks(split):
    d = _torchrun("--config", "cfg4b4", "--steps", "3", "--warmup", "3", "--e2e-steps", "3",
                  "--no-cpu-baseline", "--split", split)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert ("k-split" in d["config"]["parallelism"]) == (split == "k")


def test_reference_arm_two_ranks():
    d = _torchrun("--config", "cfg2", "--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
