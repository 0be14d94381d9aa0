"""The multi-rank bench path the driver's SCALE run uses:
``bench.py --gpus 2`` re-launches itself under torch.distributed.run; with
SGAP_BENCH_SHARE_GPU=1 both ranks share cuda:0 over gloo (this pod has one
GPU), so shards, barriers and the max-over-ranks timing run for real while
the number itself is not a scaling result."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2209_02882_b200 import generators as G
from paper_2209_02882_b200.partition import shard_starts

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_strong_scaling_config2():
    env = dict(os.environ, SGAP_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "2",
                          "--steps", "5", "--warmup", "3", "--point", "nnz:256,col:4,r:1",
                          "--no-e2e", "--no-cpu"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong"
    cfg = rec["config"]
    g = G.rmat(20, 16, seed=1, device="cuda")
    want = shard_starts(g.row_ptr.cpu().numpy(), 2)
    assert cfg["shard_row_starts"] == [int(x) for x in want]
    assert cfg["nnz"] == g.nnz and cfg["shard_nnz"] > 0.49 * g.nnz
    # max over ranks: the step time is the slowest rank's
    assert len(cfg["rank_total_ms"]) == 2
    assert rec["ms_per_step"] == pytest.approx(max(cfg["rank_total_ms"]) / rec["steps"])
    assert rec["value"] == pytest.approx(2.0 * g.nnz * 128 / (rec["ms_per_step"] * 1e6))
    assert rec["gpu_launches"] >= rec["steps"]
