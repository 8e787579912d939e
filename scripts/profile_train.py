"""Minimal driver for ncu: cfg2 workload, one refresh, 3 tile passes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig

cfg, stacks, batch, field, states, psf = build_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
for _ in range(3):
    eng.epoch(1.0, True, False, 0)
torch.cuda.synchronize()
print("ok")
