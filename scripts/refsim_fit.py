"""Fetal-scale acquisition from the reference's OWN simulator (package
simulate.py: reference phantom + CUDA PSF quadrature) fitted on the device:
GT make_phantom(size, spacing) (simulate.py:125-135), 3 orthogonal stacks at
the given in-plane spacing / thickness, 2 % noise, 6 deg / 4 mm motion, then a
500-epoch fit with the reference defaults, evaluated every 25 epochs (gauge
removed with the true states).

    python scripts/refsim_fit.py [size spacing inplane thickness n_gaussians noise]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import simulate
from paper_2512_11624_b200.metrics import motion_error


def main(size=128, spacing=0.8, inplane=0.8, thickness=3.5, n_gauss=200_000, noise=0.02, epochs=500):
    t0 = time.perf_counter()
    gt = simulate.make_phantom(size, seed=0, spacing=spacing)
    t_ph = time.perf_counter() - t0
    t0 = time.perf_counter()
    stacks, truths = simulate.simulate_protocol(
        gt, simulate.AcquisitionParams(inplane=inplane, thickness=thickness, noise_std=noise),
        simulate.MotionParams(6.0, 4.0, seed=0))
    t_sim = time.perf_counter() - t0
    truth = g.SliceStates(np.concatenate([t.quaternions for t in truths]),
                          np.concatenate([t.translations for t in truths]),
                          np.concatenate([t.log_sigma for t in truths]), np.concatenate([t.eta for t in truths]))
    px = sum(int(s.mask.sum()) for s in stacks)
    print(f"phantom {size}^3 @ {spacing} mm: {t_ph:.1f} s; simulate {[s.data.shape for s in stacks]} "
          f"({px} masked px): {t_sim:.2f} s", flush=True)
    t0 = time.perf_counter()
    g.fit(stacks, g.InitConfig(n_gaussians=n_gauss, seed=0), None, g.OptimConfig(epochs=epochs))
    wall = time.perf_counter() - t0
    _, st, hist = g.fit(stacks, g.InitConfig(n_gaussians=n_gauss, seed=0), None, g.OptimConfig(epochs=epochs),
                        reference=gt, truth_states=truth, eval_every=25)
    evals = [(h["epoch"], round(h["psnr"], 2), round(h["ssim"], 4)) for h in hist if h["psnr"] is not None]
    r, t = motion_error(st, truth)
    out = {"size": size, "spacing": spacing, "inplane": inplane, "thickness": thickness, "n_gaussians": n_gauss,
           "noise": noise, "pixels": px, "simulate_s": t_sim, "fit_wall_s": wall, "evals": evals,
           "motion_median_deg": float(np.median(r)), "motion_median_mm": float(np.median(t))}
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    a = [float(v) for v in sys.argv[1:]]
    kw = dict(zip(["size", "spacing", "inplane", "thickness", "n_gauss", "noise"], a))
    for k in ("size", "n_gauss"):
        if k in kw:
            kw[k] = int(kw[k])
    main(**kw)
