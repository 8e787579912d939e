"""bench.py's multi-GPU path (BASELINE configs[2]: one cfg3 acquisition,
slices sharded over the ranks, field replicated, gradient all-reduced) run as
2 ranks with gloo on the one GPU this run has: it must emit the full JSON line
(headline, roofline, e2e, the sharded fit wall-clock).  NCCL on real NVLink is
the same code path with backend "nccl"."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(1200)
def test_bench_two_ranks_sharded_cfg3_gloo():
    env = dict(os.environ, GSVR_DIST_BACKEND="gloo", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--e2e-steps", "1", "--fit-epochs", "20",
           "--no-extras"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1100)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    print(json.dumps({k: out[k] for k in ("value", "ms_per_step", "scaling", "config")}, indent=1))
    assert out["n_gpus"] == 2 and out["scaling"] == "strong" and out["value"] > 0
    assert out["config"]["workload"].startswith("cfg3")
    assert out["config"]["points_total"] == 24_576_000
    assert out["config"]["points_per_gpu"] < out["config"]["points_total"]
    assert out["roofline"]["frac"] > 0 and out["gpu_launches"] > 0
    assert out["e2e"]["value"] > 0 and out["e2e_pinned"]["value"] > 0
    assert out["fit_cfg3"]["gpus"] == 2 and out["fit_cfg3"]["wall_s"] > 0
    assert out["nccl"]["world_size"] == 2
