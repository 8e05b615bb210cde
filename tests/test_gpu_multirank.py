"""The batch-sharded multi-rank path of bench.py, run for real on the GPU:
two ranks (torchrun, gloo process group for the host-side reductions) share
cuda:0, each runs its own shard of the global batch through the timed CUDA
graph, each checks its shard bit-exactly against the oracle (bench.py's
parity gate, per rank), and rank 0 reports the max over ranks.

Two ranks on one GPU is only a functional check of the sharding / gather /
max-over-ranks plumbing; the ranks never wait on each
other's kernels (no data-path collective exists)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_sharded_bench_two_ranks_on_one_gpu(cuda):
    port = 29500 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--batch", "16", "--steps", "3", "--warmup", "3", "--tune", "0",
           "--branch-search", "0", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["config"]["batch_per_gpu"] == 8 and res["config"]["global_batch"] == 16
    assert res["parity"]["bitexact"] is True and res["parity"]["layers"] == 23
    per = res["per_rank_ms_per_step"]
    assert len(per) == 2 and abs(res["ms_per_step"] - max(per)) <= 1e-3 * max(per) + 1e-4
    # whole-job throughput: both ranks' ops over the slowest rank's time
    ops = res["config"]["ops_per_step_per_gpu"]
    assert abs(res["value"] - ops * 2 / (res["ms_per_step"] * 1e-3) / 1e12) <= 0.01 * res["value"] + 0.01
