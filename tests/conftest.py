"""Shared test plumbing: the `gpu` marker, golden-fixture loading, oracle access.

Tests marked ``gpu`` need a B200 and the built CUDA library; everything else
runs on CPU (oracle vs golden vectors, host logic, C-ABI symbol checks, gloo
multi-process tests).
"""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built library")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        d = {k: z[k] for k in z.files}
    if "nbr" in d:
        d["nbr"] = d["nbr"].astype(np.int64)
    return d


TRAIN_CASES = (["train_frozen"] + [f"train_grad_acc_s{s}" for s in range(5)]
               + [f"train_grad_unit_s{s}" for s in range(2)]
               + [f"train_medium_s{s}" for s in range(2)])


def loss_kwargs(d, prefix=""):
    """LossConfig fields a golden case was generated with."""
    if prefix == "outlier_":
        return dict(lambda_reg=2.5e-3, s_target=1.6, outlier_weighting=True)
    return dict(lambda_reg=float(d["cfg_lambda_reg"]), s_target=float(d["cfg_s_target"]),
                outlier_weighting=bool(d["cfg_outlier"]))


def output_prefix(name):
    return "plain_" if name == "train_frozen" else ""


@pytest.fixture(scope="session")
def oracle():
    from oracle import host
    host.lib()
    return host
