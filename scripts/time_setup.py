"""Breakdown of the fit's setup at a config (host init, batch build, device batch, engine)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import initialization as ini, synthetic
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
stacks, _ = synthetic.make_stacks(cfg, seed=0)
icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
torch.zeros(1).cuda()
for rep in range(2):
    T = {}
    t = time.perf_counter(); grads = [ini.gradient_magnitude(s) for s in stacks]; T["gradient(serial)"] = time.perf_counter() - t
    t = time.perf_counter(); pos = ini.sample_init_positions(stacks, icfg); T["sample_init_positions"] = time.perf_counter() - t
    t = time.perf_counter(); f = ini.init_field(pos, stacks, icfg); T["init_field"] = time.perf_counter() - t
    t = time.perf_counter(); b = g.build_point_batch(stacks); T["build_point_batch"] = time.perf_counter() - t
    t = time.perf_counter(); db = DeviceBatch(b, K=50); torch.cuda.synchronize(); T["DeviceBatch"] = time.perf_counter() - t
    psf = g.slice_psf_diags(b, stacks)
    t = time.perf_counter(); eng = FitEngine(db, f, g.init_states(stacks), psf, g.LossConfig(), g.OptimConfig()); torch.cuda.synchronize(); T["FitEngine"] = time.perf_counter() - t
    t = time.perf_counter(); eng.refresh(50); torch.cuda.synchronize(); T["first refresh"] = time.perf_counter() - t
    print({k: round(v, 3) for k, v in T.items()}, flush=True)
    del eng, db
