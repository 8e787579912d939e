"""One neighbour refresh at cfg2 (for ncu launch lists)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
cfg, stacks, batch, field, states, psf = build_workload("cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)  # unseeded; the profiled one below is seeded
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.refresh(50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
