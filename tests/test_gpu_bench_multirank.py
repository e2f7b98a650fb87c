"""The multi-rank bench path (`bench.py --gpus 2`: spawned ranks, global sample
and fact ids, record all-gather, gradient all-reduce, max-over-ranks timing) on
a one-GPU box: both ranks share cuda:0 and talk over gloo (host-staged), so
this checks the plumbing the driver's scaling run uses, not a speed."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LOBSTER_BENCH_BACKEND="gloo", LOBSTER_BENCH_ONE_DEVICE="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True, env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 128
    # two ranks x two semiring fixpoints x (64 samples of 32^4 `path` tuples + one `endpoints_connected` row each)
    assert line["tuples_per_step"] == 4 * (64 * 32 ** 4 + 64)
    assert len(line["per_rank_ms_per_step"]) == 2
