"""Golden hashes of the reference's host-side batch/initialisation logic (this container only).

    python oracle/gen_host_golden.py

On the reference's own cfg1 acquisitions (tests/golden/cfg1_data.npz and
cfg1_noisy_data.npz) it runs gsvr.motion.build_point_batch and
gsvr.initialization.sample_init_positions / init_field for a few configs and
stores SHA-256 digests of the output bytes in tests/golden/host_cases.json.
tests/test_host_golden.py recomputes them with this package: equal digests
mean bit-identical batches and starting fields (same numpy RNG stream).
"""
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "host_cases.json"

INIT_CASES = [  # (data file, n_gaussians, seed, lambda_init, initial_scale, intensity_policy)
    ("cfg1_data.npz", 10_000, 0, 0.0, 1.6, "source"),
    ("cfg1_data.npz", 3_000, 7, 0.3, 1.2, "mean"),
    ("cfg1_noisy_data.npz", 10_000, 3, 0.0, 1.6, "source"),
]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load_stacks(SliceStack, name):
    z = dict(np.load(ROOT / "tests" / "golden" / name))
    return [SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                       float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]


def main():
    from gsvr.initialization import InitConfig, init_field, sample_init_positions
    from gsvr.motion import SliceStack, build_point_batch
    out = {"batches": {}, "inits": []}
    for name in ("cfg1_data.npz", "cfg1_noisy_data.npz"):
        b = build_point_batch(load_stacks(SliceStack, name))
        out["batches"][name] = {"lifted": digest(b.lifted), "slice_ids": digest(b.slice_ids),
                                "intensities": digest(b.intensities), "n_points": int(b.lifted.shape[0])}
    for name, n, seed, lam, scale, pol in INIT_CASES:
        stacks = load_stacks(SliceStack, name)
        cfg = InitConfig(n_gaussians=n, lambda_init=lam, seed=seed, initial_scale=scale, intensity_policy=pol)
        pos = sample_init_positions(stacks, cfg)
        f = init_field(pos, stacks, cfg)
        out["inits"].append({"data": name, "n_gaussians": n, "seed": seed, "lambda_init": lam,
                             "initial_scale": scale, "intensity_policy": pol,
                             "positions": digest(pos), "intensities": digest(f.intensities),
                             "log_scales": digest(f.log_scales)})
    OUT.write_text(json.dumps(out, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
