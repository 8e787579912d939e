"""Time refresh at the fit's initial state (init field from sampled stack voxels)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine, pick_tile_points
from paper_2512_11624_b200.motion import build_point_batch, init_states
from paper_2512_11624_b200.initialization import init_field, sample_init_positions
from paper_2512_11624_b200.train import LossConfig, OptimConfig, slice_psf_diags
cfg = synthetic.CONFIGS["cfg2"]
stacks, truth = synthetic.make_stacks(cfg, seed=0)
ic = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
batch = build_point_batch(stacks)
field = init_field(sample_init_positions(stacks, ic), stacks, ic)
states = init_states(stacks)
psf = slice_psf_diags(batch, stacks, True, None)
db = DeviceBatch(batch, K=50, tile_points=pick_tile_points(50))
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
mu = field.means
print("unique means", len(np.unique(mu, axis=0)), "of", len(mu))
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.refresh(50)
    torch.cuda.synchronize(); print("refresh", i, (time.perf_counter() - t0) * 1e3, "ms", flush=True)
from paper_2512_11624_b200.knn import _build_handle, NeighborIndex
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = _build_handle(eng.mu)
    torch.cuda.synchronize(); print("build", (time.perf_counter() - t0) * 1e3, "ms")
