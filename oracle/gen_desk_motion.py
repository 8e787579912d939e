"""Motion-bearing desk acquisition + the REFERENCE's fit of it (this container only).

    python oracle/gen_desk_motion.py

Reproduces the reference's own acceptance desk fixture
(/root/reference/pkg/tests/test_acceptance.py:35-101, `noisy_case` + `_desk`):
make_phantom(64, seed=0) (0.5 mm grid), simulate_protocol with
AcquisitionParams(inplane=0.5, thickness=3.0, noise_std=0.02) and
MotionParams(rot_max=6, trans_max=4, seed=0) (simulate.py:318-326), then
fit(InitConfig(n_gaussians=5000, seed=0), LossConfig(lambda_reg=2.5e-3),
OptimConfig(epochs=500, k_neighbors=50), reference=phantom, truth_states=truth,
eval_every=25) (train.py:373-497).

Writes tests/golden/desk_motion_data.npz (phantom, stacks, truth states) and
tests/golden/desk_motion_ref_fit.json: the gauge-removed PSNR/SSIM trajectory
every 25 epochs (train.py:361-370), the final aligned PSNR/SSIM the way
test_acceptance._desk computes them, and the final per-slice motion_error
(metrics.py:142-154) -- the slice-pose ("S" of SVR) trajectory pin for the
device fit (tests/test_gpu_fit.py::test_desk_motion_fit_tracks_reference).
Test infrastructure only.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

from gsvr.field import rasterize  # noqa: E402
from gsvr.initialization import InitConfig  # noqa: E402
from gsvr.metrics import motion_error, motion_gauge, psnr, ssim  # noqa: E402
from gsvr.motion import SliceStates  # noqa: E402
from gsvr.simulate import AcquisitionParams, MotionParams, make_phantom, simulate_protocol  # noqa: E402
from gsvr.train import LossConfig, OptimConfig, fit  # noqa: E402


def main():
    noise = float(os.environ.get("DESK_NOISE", "0.02"))
    tag = "desk_motion" if noise > 0 else "desk_motion_clean"
    gt = make_phantom(64, seed=0)
    stacks, truths = simulate_protocol(
        gt, AcquisitionParams(inplane=0.5, thickness=3.0, noise_std=noise),
        MotionParams(rot_max=6.0, trans_max=4.0, seed=0))
    truth = SliceStates.concatenate(truths)
    d = {"gt_data": gt.data, "gt_affine": gt.affine, "gt_mask": gt.mask,
         "truth_q": truth.quaternions, "truth_t": truth.translations,
         "truth_logsig": truth.log_sigma, "truth_eta": truth.eta}
    for i, s in enumerate(stacks):
        d.update({f"s{i}_data": s.data, f"s{i}_affine": s.affine, f"s{i}_mask": s.mask,
                  f"s{i}_spacing": s.inplane_spacing, f"s{i}_thickness": np.float64(s.thickness)})
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{tag}_data.npz", **d)
    t0 = time.perf_counter()
    field, states, hist = fit(stacks, InitConfig(n_gaussians=5000, seed=0),
                              LossConfig(lambda_reg=2.5e-3),
                              OptimConfig(epochs=500, k_neighbors=50),
                              reference=gt, truth_states=truth, eval_every=25)
    wall = time.perf_counter() - t0
    aligned = rasterize(field, gt, K=50, transform=motion_gauge(states, truth))
    rot, trans = motion_error(states, truth)
    out = {"wall_s": wall, "epochs": 500, "n_gaussians": 5000, "K": 50,
           "lambda_reg": 2.5e-3, "noise_std": noise, "rot_max": 6.0, "trans_max": 4.0,
           "threads": os.environ.get("NUMBA_NUM_THREADS", str(os.cpu_count())),
           "evals": [{"epoch": h["epoch"], "loss": float(h["loss"]), "psnr": float(h["psnr"]),
                      "ssim": float(h["ssim"])} for h in hist if h["psnr"] is not None],
           "loss": [float(h["loss"]) for h in hist],
           "final_psnr": float(psnr(aligned.data, gt.data, mask=gt.mask)),
           "final_ssim": float(ssim(aligned.data, gt.data, mask=gt.mask)),
           "motion_rot_deg": rot.tolist(), "motion_trans_mm": trans.tolist(),
           "motion_rot_median": float(np.median(rot)), "motion_trans_median": float(np.median(trans)),
           "states_q": states.quaternions.tolist(), "states_t": states.translations.tolist(),
           "source": "gsvr.fit on the reference acceptance desk fixture "
                     "(tests/test_acceptance.py:60-100), build container, numba"}
    (OUT / f"{tag}_ref_fit.json").write_text(json.dumps(out, indent=1))
    print("reference desk fit", wall, "s; final", out["final_psnr"], out["final_ssim"],
          "motion median", out["motion_rot_median"], out["motion_trans_median"])


if __name__ == "__main__":
    main()
