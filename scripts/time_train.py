"""Time only the tile pass (CUDA events), for A/B of library variants (GSVR_B200_LIB)."""
import sys, os
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
    eng.train_pass()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    eng.train_pass()
e1.record()
torch.cuda.synchronize()
print(f"{os.environ.get('GSVR_B200_LIB', 'default')}: train pass {e0.elapsed_time(e1) / 20:.3f} ms, "
      f"tiles {db.n_tiles} unique {db.tile_gaussians}")
