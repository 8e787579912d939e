"""cfg2 fit quality diagnostics: loss / PSNR / SSIM history, with and without motion."""
import sys, time, dataclasses
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic

def run(cfg, epochs, label, **ok):
    stacks, truth = synthetic.make_stacks(cfg, seed=0)
    n = 128
    aff = np.eye(4); aff[:3, 3] = -0.5 * (n - 1)
    grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
    gt = synthetic.phantom(grid.voxel_centers()).reshape(n, n, n)
    ref = g.VolumeGrid(gt, aff, mask=gt > 0)
    t0 = time.perf_counter()
    _, st, hist = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None,
                        g.OptimConfig(epochs=epochs, **ok), reference=ref, truth_states=truth, eval_every=25)
    print(f"== {label}: {time.perf_counter()-t0:.1f}s")
    for h in hist:
        if h["psnr"] is not None or h["reseeded"]:
            print(f"  ep {h['epoch']:4d} loss {h['loss']:.4e} data {h['data_term']:.4e} reg {h['reg_term']:.3e} "
                  f"psnr {h['psnr'] if h['psnr'] is None else round(h['psnr'],2)} "
                  f"ssim {h['ssim'] if h['ssim'] is None else round(h['ssim'],4)} reseeded {h['reseeded']}", flush=True)
    err = g.metrics.motion_error(st, truth) if hasattr(g, "metrics") else None
    from paper_2512_11624_b200.metrics import motion_error
    r, t = motion_error(st, truth)
    print(f"  motion error median {np.median(r):.2f} deg {np.median(t):.2f} mm")

cfg = synthetic.CONFIGS["cfg2"]
run(dataclasses.replace(cfg, rot_max_deg=0.0, trans_max_mm=0.0), 300, "cfg2 no motion")
run(cfg, 500, "cfg2 with motion")
