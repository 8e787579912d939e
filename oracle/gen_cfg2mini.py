"""The synthetic cfg2 generator at a CPU-feasible size, fitted by the REFERENCE
(this container only) -- the reference's behaviour on the same kind of data
as the fetal-scale bench fits.

    python oracle/gen_cfg2mini.py [noise]

cfg2 spacing (0.8 x 0.8 x 3.5 mm), 2 % noise and 6 deg / 4 mm slice motion
from paper_2512_11624_b200.synthetic (full-FOV stacks, no mask), but a
96 x 96 x 22 FOV (77 mm) per stack and 20,600 Gaussians -- the same ~29.5
pixels per Gaussian as cfg2 (5.9 M px / 200k).  Writes
tests/golden/cfg2mini{_clean}_data.npz (stacks as float32, true states) and
tests/golden/cfg2mini{_clean}_ref_fit.json: the reference's 500-epoch fit
(train.py:373-497) evaluated every 25 epochs against the analytic phantom on
a 64^3 1.2 mm grid over the same FOV, gauge removed with the true states.
Test infrastructure only.
"""
import dataclasses
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")


def make_case(noise):
    sys.path.insert(0, str(ROOT))
    from paper_2512_11624_b200 import synthetic
    cfg = dataclasses.replace(synthetic.CONFIGS["cfg2"], name="cfg2mini", nx=96, ny=96, n_slices=22,
                              n_gaussians=20_600, noise_std=noise)
    stacks, truth = synthetic.make_stacks(cfg, seed=0)
    n = 64
    aff = np.diag([1.2, 1.2, 1.2, 1.0])
    aff[:3, 3] = -0.5 * 1.2 * (n - 1)
    from paper_2512_11624_b200.volume import VolumeGrid
    grid = VolumeGrid(np.zeros((n, n, n)), aff)
    gt = synthetic.phantom(grid.voxel_centers()).reshape(n, n, n)
    return cfg, stacks, truth, gt, aff


def main():
    noise = float(sys.argv[1]) if len(sys.argv) > 1 else 0.02
    tag = "cfg2mini" if noise > 0 else "cfg2mini_clean"
    cfg, stacks, truth, gt, aff = make_case(noise)
    d = {"gt_data": gt, "gt_affine": aff, "truth_q": truth.quaternions, "truth_t": truth.translations,
         "n_gaussians": np.int64(cfg.n_gaussians)}
    for i, s in enumerate(stacks):
        d.update({f"s{i}_data": s.data.astype(np.float32), f"s{i}_affine": s.affine,
                  f"s{i}_spacing": s.inplane_spacing, f"s{i}_thickness": np.float64(s.thickness)})
    np.savez_compressed(OUT / f"{tag}_data.npz", **d)

    sys.path.insert(0, "/root/reference/pkg/src")
    import gsvr
    from gsvr.field import rasterize
    from gsvr.initialization import InitConfig
    from gsvr.metrics import motion_error, motion_gauge, psnr, ssim
    from gsvr.motion import SliceStack, SliceStates
    from gsvr.train import OptimConfig, fit
    from gsvr.volume import VolumeGrid
    rst = [SliceStack(d[f"s{i}_data"].astype(np.float64), d[f"s{i}_affine"], d[f"s{i}_spacing"],
                      float(d[f"s{i}_thickness"])) for i in range(3)]
    ref = VolumeGrid(gt, aff, mask=gt > 0)
    tr = SliceStates(truth.quaternions, truth.translations, truth.log_sigma, truth.eta)
    t0 = time.perf_counter()
    field, states, hist = fit(rst, InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None,
                              OptimConfig(epochs=500), reference=ref, truth_states=tr, eval_every=25)
    wall = time.perf_counter() - t0
    rot, trans = motion_error(states, tr)
    out = {"wall_s": wall, "epochs": 500, "n_gaussians": cfg.n_gaussians, "K": 50, "noise_std": noise,
           "pixels": int(sum(s.data.size for s in rst)),
           "evals": [{"epoch": h["epoch"], "loss": float(h["loss"]), "psnr": float(h["psnr"]),
                      "ssim": float(h["ssim"])} for h in hist if h["psnr"] is not None],
           "motion_rot_median": float(np.median(rot)), "motion_trans_median": float(np.median(trans)),
           "gsvr_version": getattr(gsvr, "__version__", "?"),
           "source": "gsvr.fit on paper_2512_11624_b200.synthetic stacks (cfg2 spacing/noise/motion, "
                     "96x96x22 FOV), build container, numba"}
    (OUT / f"{tag}_ref_fit.json").write_text(json.dumps(out, indent=1))
    print(tag, "reference fit", wall, "s", out["evals"][-1], rot.mean())


if __name__ == "__main__":
    main()
