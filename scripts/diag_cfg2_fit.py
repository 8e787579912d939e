"""cfg2 fit quality diagnostics: loss / PSNR / SSIM history and final motion
error under variants (motion / no motion, noise / no noise, rotations frozen),
to locate the late-epoch quality drop of the synthetic cfg2 fit."""
import dataclasses
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
from paper_2512_11624_b200.metrics import motion_error


def run(cfg, epochs, label, mask_bg=False, **ok):
    stacks, truth = synthetic.make_stacks(cfg, seed=0)
    if mask_bg:
        stacks = [g.SliceStack(s.data, s.affine, s.inplane_spacing, s.thickness,
                               np.ones_like(s.data, bool) & (np.abs(s.data) > 0.05)) for s in stacks]
    n = 128
    aff = np.eye(4)
    aff[:3, 3] = -0.5 * (n - 1)
    grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
    gt = synthetic.phantom(grid.voxel_centers()).reshape(n, n, n)
    ref = g.VolumeGrid(gt, aff, mask=gt > 0)
    t0 = time.perf_counter()
    _, st, hist = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None,
                        g.OptimConfig(epochs=epochs, **ok), reference=ref, truth_states=truth,
                        eval_every=25)
    print(f"== {label}: {time.perf_counter() - t0:.1f}s", flush=True)
    for h in hist:
        if h["psnr"] is not None or h["reseeded"]:
            p = None if h["psnr"] is None else round(h["psnr"], 2)
            s = None if h["ssim"] is None else round(h["ssim"], 4)
            print(f"  ep {h['epoch']:4d} loss {h['loss']:.4e} data {h['data_term']:.4e} "
                  f"reg {h['reg_term']:.3e} psnr {p} ssim {s} reseeded {h['reseeded']}", flush=True)
    if len(st) == len(truth):
        r, t = motion_error(st, truth)
        print(f"  motion error median {np.median(r):.2f} deg {np.median(t):.2f} mm; "
              f"p90 {np.percentile(r, 90):.2f} deg {np.percentile(t, 90):.2f} mm", flush=True)


if __name__ == "__main__":
    cfg = synthetic.CONFIGS["cfg2"]
    which = sys.argv[1:] or ["motion", "nomotion", "frozenrot", "nonoise", "maskbg"]
    if "motion" in which:
        run(cfg, 500, "cfg2 with motion")
    if "nomotion" in which:
        run(dataclasses.replace(cfg, rot_max_deg=0.0, trans_max_mm=0.0), 500, "cfg2 no motion")
    if "frozenrot" in which:
        run(cfg, 500, "cfg2 motion, rotations frozen", rotation_warmup=10 ** 6)
    if "nonoise" in which:
        run(dataclasses.replace(cfg, noise_std=0.0), 500, "cfg2 motion, no noise")
    if "maskbg" in which:
        run(cfg, 500, "cfg2 motion, background masked", mask_bg=True)
