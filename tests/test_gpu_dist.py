"""Two ranks on one GPU through the real kernels (SWB_DIST_BACKEND=gloo: the
shards never wait on each other, so sharing the device is only slower, not
different). bench.py under torch.distributed.run must produce exactly the
single-rank results: config 2's merged top-100 (database sharded by target,
one all_gather of 100 records per rank) and config 3's scores (pairs sharded by
contiguous range, each rank generating only its own pairs, gathered after the
timed region)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(world: int, *args: str) -> dict:
    base = [sys.executable, os.path.join(REPO, "bench.py"), "--steps", "2", "--warmup", "3",
            "--no-cpu-baseline", *args]
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
               str(_port()), *base[1:]]
    else:
        cmd = base
    env = dict(os.environ, SWB_DIST_BACKEND="gloo")
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_config2_two_ranks_equal_one(cuda):
    one = _bench(1, "--config", "2", "--n-targets", "30000")
    two = _bench(2, "--config", "2", "--n-targets", "30000")
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "db-shard x2"
    assert two["topk_sha256"] == one["topk_sha256"] and two["top_hit"] == one["top_hit"]


def test_config3_two_ranks_equal_one_and_oracle(cuda, oracle):
    from paper_1909_00899_b200 import workloads as W

    n = 70_000  # not a multiple of the generator block: shard cuts inside a block
    one = _bench(1, "--config", "3", "--n-pairs", str(n))
    two = _bench(2, "--config", "3", "--n-pairs", str(n))
    assert two["config"]["parallelism"] == "pair-shard x2"
    assert two["scores_sha256"] == one["scores_sha256"]
    w = W.config3(n_pairs=n)
    s, _, _ = oracle.batch_scalar(w.flat_q, w.q_off, w.flat_r, w.r_off, sub=w.scheme.as_array(),
                                  go=6, ge=1)
    assert one["score_sum"] == int(s.sum())
    import hashlib

    assert one["scores_sha256"] == hashlib.sha256(s.astype(np.int32).tobytes()).hexdigest()


def test_runner_gpus2_identical_tsv(cuda, tmp_path):
    """runner --gpus 2 (pairs sharded over two worker processes; gloo when they share
    one device) writes the same TSV as one process, coordinates included."""
    from paper_1909_00899_b200 import runner

    def tsv(**kw):
        import io

        buf = io.StringIO()
        assert runner.run(runner.RunConfig(**kw), out=buf) == 0
        rows = []
        for line in buf.getvalue().splitlines():
            f = line.split("\t")
            if len(f) > 6 and f[0] != "query_id":
                f[6] = "T"
            rows.append(f)
        return rows

    for kern in ("scan", "lazyf"):
        kw = dict(kernel=kern, lanes=16, random_count=501, seed=5, len_max=300, coords=True)
        assert tsv(gpus=2, **kw) == tsv(**kw), kern
