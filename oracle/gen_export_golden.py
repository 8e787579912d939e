"""Golden HR-export (rasterize) cases from the REFERENCE (this container only).

    python oracle/gen_export_golden.py

gsvr.field.rasterize (field.py:138-175: K-NN of the voxel centres + PSF-free
evaluate_field) on small rotated grids, with and without a mask and a rigid
transform, K below and above the primitive count -> tests/golden/export_cases.npz.
"""
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "export_cases.npz"


def main():
    from gsvr.field import GaussianField, rasterize
    from gsvr.geometry import quat_to_rotation
    from gsvr.volume import VolumeGrid
    rng = np.random.default_rng(5)
    d = {}
    cases = [("a", 600, 16, True, False), ("b", 600, 50, False, True), ("c", 12, 50, True, True)]
    for name, n, K, masked, transformed in cases:
        mu = rng.uniform(-12, 12, size=(n, 3))
        ls = np.log(rng.uniform(0.6, 2.0, size=(n, 3)))
        q = rng.normal(size=(n, 4))
        c = rng.uniform(0.1, 0.9, size=n)
        field = GaussianField(mu, ls, q, c)
        R = quat_to_rotation(np.array([1.0, 0.1, -0.2, 0.05]))
        aff = np.eye(4)
        aff[:3, :3] = R @ np.diag([1.3, 1.1, 1.7])
        aff[:3, 3] = [-11.0, -9.5, -12.0]
        shape = (18, 20, 14)
        mask = rng.random(shape) < 0.7 if masked else None
        grid = VolumeGrid(np.zeros(shape), aff, mask)
        tr = None
        if transformed:
            tr = (quat_to_rotation(np.array([1.0, -0.05, 0.02, 0.1])), np.array([0.4, -0.3, 0.2]))
        out = rasterize(field, grid, K, transform=tr)
        d.update({f"{name}_means": mu, f"{name}_log_scales": ls, f"{name}_quats": q, f"{name}_cvals": c,
                  f"{name}_affine": aff, f"{name}_K": np.int64(K), f"{name}_out": out.data})
        if mask is not None:
            d[f"{name}_mask"] = mask
        if tr is not None:
            d[f"{name}_R"], d[f"{name}_t"] = tr
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
