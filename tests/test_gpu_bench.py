"""bench.py's multi-rank path (the driver's scaling run: torchrun, one
process per GPU) end to end on one GPU: two processes over gloo sharing
cuda:0 (DFNO_BENCH_SHARE_GPU), pipelined exchanges timed on the comm stream;
and the single-rank JSON line contract."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(cmd, env=None, timeout=600):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_bench_line():
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps", "1",
              "--warmup", "1", "--no-cpu-baseline", "--no-e2e", "--no-train"],
             env={"DFNO_BENCH_SHARE_GPU": "1", "DFNO_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    a2a = d["all_to_all"]
    assert a2a["exchanges_per_step"] == 32  # 4 blocks x 4 repartitions x 2 channel groups
    assert a2a["off_rank_bytes_per_step"] > 0
    assert "xdft.fwd" in d["kernels"] and "xmix_bwd" in d["kernels"]


def test_single_rank_bench_line():
    d = _run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-train"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["roofline"]["frac"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
