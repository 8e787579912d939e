"""Golden vectors for render.render_observed and the PSF helpers, made by
running the REFERENCE (this container only).

    python oracle/gen_render_golden.py   # writes tests/golden/render_observed_cases.npz

Cases follow the reference's own tests: rotated_psf_cov6 on five random
rotations (tests/test_psf.py:85-92), convolve_covariance on a random
primitive (tests/test_psf.py:61-70), and render_observed (render.py:22-65)
with a shared (3,3) rotation and with per-point (M,3,3) rotations + per-point
sigma, in float64 and float32 fields, on a conftest.make_field-style cloud
(tests/conftest.py:10-25).  Test infrastructure only.
"""
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

from conftest import make_field  # noqa: E402
from gsvr.geometry import build_covariance, quat_to_rotation  # noqa: E402
from gsvr.knn import build_index, query  # noqa: E402
from gsvr.psf import build_psf, convolve_covariance, rotated_psf_cov6  # noqa: E402
from gsvr.render import render_observed  # noqa: E402


def main():
    rng = np.random.default_rng(7)
    d = {}
    psf = build_psf(0.8, 2.5)
    R5 = quat_to_rotation(rng.normal(size=(5, 4)))
    d["psf_R5"] = R5
    d["psf_cov6_R5"] = rotated_psf_cov6(R5, psf)
    psf2 = build_psf(0.5, 3.0)
    Rq = quat_to_rotation(rng.normal(size=4))
    cov = build_covariance(np.log(rng.uniform(0.5, 1.5, 3)), rng.normal(size=4))
    d.update(conv_R=Rq, conv_cov=cov, conv_out=convolve_covariance(cov, Rq, psf2))

    field = make_field(300, seed=3, spread=12.0)
    M, K = 700, 24
    pts = rng.uniform(-12.0, 12.0, size=(M, 3))
    nbr = query(build_index(field.means), pts, K)
    Rshared = quat_to_rotation(np.array([0.9, 0.2, -0.3, 0.1]))
    Rper = quat_to_rotation(rng.normal(size=(M, 4)))
    sig = rng.uniform(0.5, 1.5, size=M)
    d.update(means=field.means, log_scales=field.log_scales, quaternions=field.quaternions,
             intensities=field.intensities, points=pts, nbr=nbr, R_shared=Rshared, R_per=Rper,
             sigma_per=sig, psf_inplane=np.float64(0.5), psf_thickness=np.float64(3.0))
    d["out_shared64"] = render_observed(pts, Rshared, field, psf2, nbr)
    d["out_per64"] = render_observed(pts, Rper, field, psf2, nbr, sigma_slice=sig)
    f32 = field.astype(np.float32)
    d["out_per32"] = render_observed(pts, Rper, f32, psf2, nbr, sigma_slice=sig)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "render_observed_cases.npz", **d)
    print("wrote render_observed_cases.npz")


if __name__ == "__main__":
    main()
