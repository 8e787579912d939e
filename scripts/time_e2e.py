"""e2e drop-in timing at cfg2: pageable numpy vs pinned host buffers (bench._e2e)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig

cfg, stacks, batch, field, states, psf = build_workload("cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
for pinned in (False, True, False, True):
    r = bench._e2e(eng, db, batch, field, states, psf, 50, 3, None, pinned=pinned)
    print(f"pinned={pinned}: {r['ms_per_step']:.1f} ms/call, {r['value'] / 1e6:.1f} M px/s", flush=True)
