import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
cfg, stacks, batch, field, states, psf = build_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
ts, tn, tsl, uoff, gid, perm = db.tile_info()
nu = np.diff(uoff)
print("tiles", len(tn), "points/tile mean", tn.mean(), "min", tn.min())
print("unique/tile percentiles 50/90/99/99.9/max:", np.percentile(nu, [50, 90, 99, 99.9]), nu.max())
print("pairs per unique gaussian (mean):", (tn * 50).sum() / nu.sum())
