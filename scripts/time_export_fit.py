"""HR export of a trained field: cfg3 fitted for a given number of epochs, then rasterize on the
cfg5 grid with stage timings (K-NN dominates for voxels far outside the object)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
from paper_2512_11624_b200.field import _voxel_centers_device
from paper_2512_11624_b200.knn import build_index, query_device

cfg = synthetic.CONFIGS["cfg3"]
stacks, _ = synthetic.make_stacks(cfg, seed=0)
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
field, _, _ = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None, g.OptimConfig(epochs=epochs))
n, sp = 410, 0.5
aff = np.diag([sp, sp, sp, 1.0])
aff[:3, 3] = -0.5 * sp * (n - 1)
grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
g.rasterize(field, g.VolumeGrid(np.zeros((128, 128, 128)), aff), 50)
for rep in range(2):
    c = _voxel_centers_device(grid.sizes, grid.affine)
    ix = build_index(field.means)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nb = query_device(ix, c, 50, out_i64=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    vol = g.rasterize(field, grid, 50)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"knn query {t1 - t0:.3f} s, rasterize {t2 - t1:.3f} s, checksum {float(np.sum(vol.data)):.10e} "
          f"nbr checksum {int(nb.long().sum())}", flush=True)
    del c, nb
