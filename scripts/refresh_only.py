"""One neighbour refresh at a config for ncu captures: the unseeded first
refresh and 30 fit epochs run outside the profiler range; the profiled
refresh is a seeded one on moved points / means (as inside a fit)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg, stacks, batch, field, states, psf = build_workload(name, 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
for e in range(30):
    eng.epoch(1.0, e >= 10, True, 0, sync=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.refresh(50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
