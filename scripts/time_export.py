"""HR export (cfg5: 410^3 voxels at 0.5 mm) stage timings on a cfg3-sized random field."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import _dev
from paper_2512_11624_b200.field import _voxel_centers_device, evaluate_field_device
from paper_2512_11624_b200.knn import build_index, query_device

rng = np.random.default_rng(0)
N = 500_000
field = g.GaussianField(rng.uniform(-100, 100, (N, 3)), np.full((N, 3), np.log(1.6)),
                        np.tile([1.0, 0, 0, 0], (N, 1)), rng.uniform(0.1, 0.9, N))
n, sp = 410, 0.5
aff = np.diag([sp, sp, sp, 1.0])
aff[:3, 3] = -0.5 * sp * (n - 1)
grid = g.VolumeGrid(np.zeros((n, n, n)), aff)


def clock(T, k, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    T[k] = round(time.perf_counter() - t, 4)
    return r


for rep in range(3):
    T = {}
    c = clock(T, "centres", lambda: _voxel_centers_device(grid.sizes, grid.affine))
    ix = clock(T, "index", lambda: build_index(field.means))
    nb = clock(T, "knn query", lambda: query_device(ix, c, 50, out_i64=False))
    fd = tuple(_dev.to_dev(a, np.float64) for a in (field.means, field.log_scales, field.quaternions, field.intensities))
    v = clock(T, "evaluate", lambda: evaluate_field_device(c, fd, nb))
    h = clock(T, "d2h", lambda: _dev.to_host(v))
    T["total rasterize"] = clock({}, "x", lambda: None) or None
    t0 = time.perf_counter()
    g.rasterize(field, grid, 50)
    torch.cuda.synchronize()
    T["total rasterize"] = round(time.perf_counter() - t0, 4)
    print(T, flush=True)
    del c, nb, v, h
