"""The tile kernel's launch buckets (train_planar.cu): tiles whose records fit a
full-residency shared-memory page run in a first launch, the rest in a second
with the page of the largest tile.  Per tile the arithmetic is the same, so an
epoch is bit-identical with and without buckets; the buckets are forced here
at a small page (GSVR_TILE_BUCKET_CAP) in a subprocess, since they only arise
by themselves at cfg4 sizes."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from bench import build_workload
from paper_2512_11624_b200 import _dev
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
cfg, stacks, batch, field, states, psf = build_workload("cfg1", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
losses = [eng.epoch(1.0, True, False, 0)["loss"] for _ in range(3)]
mu = _dev.to_host(eng.mu)
print(json.dumps({"losses": losses, "mu_sum": float(np.sum(mu)), "mu_bits": int(np.sum(mu.view(np.int64) % 1000003)),
                  "tiles": db.n_tiles}))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_tile_buckets_bit_identical():
    ref = _run({"GSVR_TILE_BUCKETS": "0"})
    got = _run({"GSVR_TILE_BUCKETS": "1", "GSVR_TILE_BUCKET_CAP": "96"})
    assert got["losses"] == ref["losses"]
    assert got["mu_bits"] == ref["mu_bits"] and got["mu_sum"] == ref["mu_sum"]
