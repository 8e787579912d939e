"""Generate golden vectors by running the REFERENCE package (this container only).

    python oracle/gen_golden.py            # writes tests/golden/*.npz

Imports gsvr from /root/reference/pkg/src (read-only mount; numba cache goes
to /tmp).  Each fixture stores the instance inputs and the reference's own
outputs, so tests can check (1) the oracle restatement and (2) the CUDA path
against the reference without /root/reference being present (the GPU box has
no mount).  Instance builders follow the reference tests they cite.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, REF_SRC)

import gsvr  # noqa: E402
from gsvr import kernels  # noqa: E402
from gsvr.field import GaussianField, evaluate_field  # noqa: E402
from gsvr.knn import build_index, query  # noqa: E402
from gsvr.motion import PointBatch, SliceStack, SliceStates, build_point_batch  # noqa: E402
from gsvr.optim import AdamW, AdamWConfig  # noqa: E402
from gsvr.train import (LossConfig, _slice_inputs, backward, compute_loss,  # noqa: E402
                        corrected_points, render_batch, slice_psf_diags)


def _axis_angle_matrix(axis, degrees):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    a = np.deg2rad(degrees)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(a) * K + (1 - np.cos(a)) * (K @ K)


def _pack_instance(batch, field, states, psf_diags, nbr):
    return {
        "lifted": batch.lifted, "slice_ids": batch.slice_ids.astype(np.int32),
        "intensities_obs": np.asarray(batch.intensities, dtype=np.float64),
        "slice_to_stack": batch.slice_to_stack.astype(np.int32),
        "stack_rotations": batch.stack_rotations, "psf_diags": psf_diags,
        "nbr": np.asarray(nbr, dtype=np.int64),
        "means": field.means, "log_scales": field.log_scales,
        "quaternions": field.quaternions, "intensities": field.intensities,
        "slice_quaternions": states.quaternions,
        "slice_translations": states.translations,
        "log_sigma": states.log_sigma, "eta": states.eta,
    }


def _reference_outputs(batch, field, states, psf_diags, nbr, cfg, prefix=""):
    out = {}
    terms, grads, I_hat = backward(batch, field, states, psf_diags, cfg, nbr)
    out[prefix + "I_hat"] = I_hat
    for k, v in terms.items():
        out[prefix + "term_" + k] = np.float64(v)
    for k, v in grads.items():
        out[prefix + "grad_" + k] = v
    loss, _ = compute_loss(batch, field, states, psf_diags, cfg, nbr)
    out[prefix + "loss_fwd"] = np.float64(loss)
    out[prefix + "render"] = render_batch(batch, field, states, psf_diags, nbr)
    return out


def _raw_kernel_outputs(batch, field, states, psf_diags, nbr, cfg):
    """kernels.train_step_backward with train.py:235-269's own inputs, block-summed."""
    P, S, N = batch.n_points, batch.n_slices, field.count
    Rc, R_eff, psf6s, sigma_s = _slice_inputs(batch, states, psf_diags)
    wdata_s = np.exp(-states.eta) if cfg.outlier_weighting else np.ones(S)
    B = kernels.default_block_count(P)
    I_hat = np.empty(P)
    absres = np.empty(P)
    bufs = [np.zeros((B, N, 3)), np.zeros((B, N, 6)), np.zeros((B, N)),
            np.zeros((B, S, 3)), np.zeros((B, S, 3, 3)), np.zeros((B, S, 6)),
            np.zeros((B, S))]
    kernels.train_step_backward(
        np.ascontiguousarray(batch.lifted), batch.slice_ids.astype(np.int32), Rc,
        np.ascontiguousarray(states.translations), psf6s, sigma_s, wdata_s,
        np.ascontiguousarray(batch.intensities, dtype=np.float64),
        np.ascontiguousarray(nbr, dtype=np.int64), np.ascontiguousarray(field.means),
        np.ascontiguousarray(field.covariances6()), np.ascontiguousarray(field.intensities),
        gsvr.DELTA, B, I_hat, absres, *bufs)
    names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
    out = {"raw_I_hat": I_hat, "raw_absres": absres, "raw_Rc": Rc, "raw_psf6s": psf6s,
           "raw_sigma_s": sigma_s, "raw_wdata_s": wdata_s,
           "raw_cov6": field.covariances6()}
    for n, b in zip(names, bufs):
        out["raw_" + n] = b.sum(axis=0)
    return out


# ---------------------------------------------------------------------------
# instances

def frozen_oracle_instance():
    """tests/test_train.py:38-61 (IHAT/DATA/REG/TOTAL_ORACLE fixture)."""
    half = np.deg2rad(4.0) / 2.0
    axis = np.array([1.0, 2.0, -1.0]) / np.sqrt(6.0)
    q = np.concatenate([[np.cos(half)], np.sin(half) * axis])
    states = SliceStates([q], [[0.3, -0.2, 0.1]], [0.05], [0.3])
    batch = PointBatch(
        lifted=np.array([[1.2, 0.3, -0.9], [-0.8, 1.4, 0.6]]),
        slice_ids=np.array([0, 0], dtype=np.int32),
        stack_ids=np.array([0, 0], dtype=np.int32),
        intensities=np.array([0.55, 0.35]),
        slice_to_stack=np.array([0], dtype=np.int32),
        stack_rotations=np.eye(3)[None])
    si, st = 0.25479654008640573, 1.2739827004320285
    psf_diags = np.array([[si ** 2, si ** 2, st ** 2]])
    field = GaussianField(
        means=[[0.2, -0.1, 0.4], [1.5, 0.8, -0.6]],
        log_scales=np.log([[0.9, 1.1, 1.4], [1.3, 0.7, 1.0]]),
        quaternions=[[0.9, -0.1, 0.3, 0.2], [1.0, 0.0, 0.0, 0.0]],
        intensities=[0.8, 0.3])
    nbr = np.array([[0, 1], [0, 1]], dtype=np.int64)
    return batch, field, states, psf_diags, nbr


def grad_instance(seed, n, n_slices, K, nx, ny, scale_lo=0.8):
    """tests/test_acceptance.py:114-143 (n=20,S=3,K=10,5x4) and
    tests/test_train.py:119-147 (n=5,S=2,K=3,4x3)."""
    rng = np.random.default_rng(seed)
    affine = np.eye(4)
    affine[:3, :3] = _axis_angle_matrix([1.0, 1.0, 0.2], 25.0) @ np.diag([0.7, 0.7, 2.0])
    affine[:3, 3] = [-1.5, -1.5, -1.0]
    stack = SliceStack(data=rng.random((nx, ny, n_slices)), affine=affine,
                       inplane_spacing=0.7, thickness=2.0)
    batch = build_point_batch([stack])
    field = GaussianField(
        means=rng.normal(scale=1.5, size=(n, 3)),
        log_scales=np.log(rng.uniform(scale_lo, 2.0, size=(n, 3))),
        quaternions=rng.normal(size=(n, 4)) + np.array([3.0, 0, 0, 0]),
        intensities=rng.uniform(0.2, 0.9, size=n))
    states = SliceStates(
        rng.normal(scale=0.02, size=(n_slices, 4)) + np.array([1.0, 0, 0, 0]),
        rng.normal(scale=0.1, size=(n_slices, 3)),
        rng.normal(scale=0.05, size=n_slices),
        rng.normal(scale=0.2, size=n_slices))
    psf_diags = slice_psf_diags(batch, [stack])
    nbr = np.argsort(rng.random((batch.n_points, n)), axis=1)[:, :K].astype(np.int64)
    cfg = LossConfig(lambda_reg=1e-3, s_target=1.3, outlier_weighting=True)
    I_hat = render_batch(batch, field, states, psf_diags, nbr)
    shifts = np.where(rng.random(batch.n_points) < 0.5, -1.0, 1.0) \
        * rng.uniform(0.05, 0.2, batch.n_points)
    batch.intensities = I_hat + shifts
    return batch, field, states, psf_diags, nbr, cfg


def medium_instance(seed, n=400, K=50, nx=20, ny=18, n_slices=5):
    """Two oblique stacks, random well-conditioned field (conftest.make_field
    style, tests/conftest.py:10-20), perturbed slice motion, neighbours from the
    reference K-NN on the corrected points (train.py:457-465)."""
    rng = np.random.default_rng(100 + seed)
    stacks = []
    for axis, ang, origin in (([1.0, 0.3, 0.2], 20.0, [-6.0, -6.0, -4.0]),
                              ([0.1, 1.0, -0.4], 70.0, [-6.5, -5.0, -5.0])):
        affine = np.eye(4)
        affine[:3, :3] = _axis_angle_matrix(axis, ang) @ np.diag([0.65, 0.65, 2.2])
        affine[:3, 3] = origin
        stacks.append(SliceStack(data=rng.random((nx, ny, n_slices)), affine=affine,
                                 inplane_spacing=0.65, thickness=2.2))
    batch = build_point_batch(stacks)
    S = batch.n_slices
    quats = rng.normal(size=(n, 4))
    field = GaussianField(
        means=rng.uniform(-7.0, 7.0, size=(n, 3)),
        log_scales=np.log(rng.uniform(0.5, 1.8, size=(n, 3))),
        quaternions=quats,
        intensities=rng.uniform(0.1, 0.9, size=n))
    states = SliceStates(
        rng.normal(scale=0.02, size=(S, 4)) + np.array([1.0, 0, 0, 0]),
        rng.normal(scale=0.3, size=(S, 3)),
        rng.normal(scale=0.05, size=S),
        rng.normal(scale=0.2, size=S))
    psf_diags = slice_psf_diags(batch, stacks)
    nbr = query(build_index(field.means), corrected_points(batch, states), K)
    cfg = LossConfig(lambda_reg=2.5e-3, s_target=1.6, outlier_weighting=bool(seed % 2))
    I_hat = render_batch(batch, field, states, psf_diags, nbr)
    shifts = np.where(rng.random(batch.n_points) < 0.5, -1.0, 1.0) \
        * rng.uniform(0.02, 0.2, batch.n_points)
    batch.intensities = I_hat + shifts
    return batch, field, states, psf_diags, nbr, cfg


def save(name, d):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size} bytes)")


def gen_train_cases():
    # frozen fixture, both loss configs
    batch, field, states, psf_diags, nbr = frozen_oracle_instance()
    d = _pack_instance(batch, field, states, psf_diags, nbr)
    d.update(_reference_outputs(batch, field, states, psf_diags, nbr, LossConfig(), "plain_"))
    d.update(_reference_outputs(batch, field, states, psf_diags, nbr,
                                LossConfig(outlier_weighting=True), "outlier_"))
    d.update(_raw_kernel_outputs(batch, field, states, psf_diags, nbr, LossConfig()))
    d.update(cfg_lambda_reg=2.5e-3, cfg_s_target=1.6, cfg_outlier=False)
    save("train_frozen", d)

    cases = [("train_grad_acc_s%d" % s, dict(seed=s, n=20, n_slices=3, K=10, nx=5, ny=4))
             for s in range(5)]
    cases += [("train_grad_unit_s%d" % s, dict(seed=s, n=5, n_slices=2, K=3, nx=4, ny=3))
              for s in range(2)]
    for name, kw in cases:
        batch, field, states, psf_diags, nbr, cfg = grad_instance(**kw)
        d = _pack_instance(batch, field, states, psf_diags, nbr)
        d.update(_reference_outputs(batch, field, states, psf_diags, nbr, cfg))
        d.update(_raw_kernel_outputs(batch, field, states, psf_diags, nbr, cfg))
        d.update(cfg_lambda_reg=cfg.lambda_reg, cfg_s_target=cfg.s_target,
                 cfg_outlier=cfg.outlier_weighting)
        save(name, d)

    for s in range(2):
        batch, field, states, psf_diags, nbr, cfg = medium_instance(s)
        d = _pack_instance(batch, field, states, psf_diags, nbr)
        d["nbr"] = d["nbr"].astype(np.int32)  # stored compactly; widened on load
        d.update(_reference_outputs(batch, field, states, psf_diags, nbr, cfg))
        d.update(_raw_kernel_outputs(batch, field, states, psf_diags, nbr, cfg))
        d.update(cfg_lambda_reg=cfg.lambda_reg, cfg_s_target=cfg.s_target,
                 cfg_outlier=cfg.outlier_weighting)
        save("train_medium_s%d" % s, d)


def gen_knn_cases():
    rng = np.random.default_rng(0)
    d = {}
    # tests/test_knn.py:19-25
    means = rng.normal(size=(400, 3))
    points = rng.normal(size=(300, 3))
    d["random_means"], d["random_points"] = means, points
    for K in (1, 7, 50):
        d[f"random_K{K}"] = query(build_index(means), points, K)
    # tests/test_knn.py:28-35 (duplicated means)
    base = rng.normal(size=(40, 3))
    means = np.concatenate([base, base[:15], base[:5]])
    points = rng.normal(size=(60, 3)) * 0.5
    d["dup_means"], d["dup_points"] = means, points
    d["dup_K10"] = query(build_index(means), points, 10)
    # tests/test_knn.py:38-46 (lattice ties)
    g = np.stack(np.meshgrid(*[np.arange(3.0)] * 3, indexing="ij"), -1).reshape(-1, 3)
    center = np.array([[0.5, 0.5, 0.5]])
    d["lattice_means"], d["lattice_points"] = g, center
    for K in (4, 8):
        d[f"lattice_K{K}"] = query(build_index(g), center, K)
    # init-style: means sampled WITH replacement from pixel positions
    # (initialization.py:93), queried at every pixel -> many boundary ties.
    gx = np.stack(np.meshgrid(np.arange(24.0), np.arange(20.0), np.arange(4.0) * 3.0,
                              indexing="ij"), -1).reshape(-1, 3) * np.array([0.8, 0.8, 1.0])
    pick = rng.choice(gx.shape[0], size=900, replace=True)
    d["init_means"], d["init_points"] = gx[pick], gx
    d["init_K50"] = query(build_index(gx[pick]), gx, 50)
    # criterion 10 style (tests/test_acceptance.py:369-384), reduced
    rng2 = np.random.default_rng(11)
    pts = rng2.uniform(-50.0, 50.0, (4096, 3))
    q = rng2.uniform(-55.0, 55.0, (4000, 3))
    d["crit10_means"], d["crit10_points"] = pts, q
    d["crit10_K50"] = query(build_index(pts), q, 50)
    # N == K (k_eff == K, knn.py:54)
    m = rng.normal(size=(12, 3))
    p = rng.normal(size=(30, 3))
    d["nk_means"], d["nk_points"], d["nk_K12"] = m, p, query(build_index(m), p, 12)
    save("knn_cases", d)


def gen_misc_cases():
    d = {}
    # optim: tests/test_optim.py:12-20 trajectory + a multi-array run
    params = {"p": np.array([1.0])}
    opt = AdamW(params, {"p": 0.1}, AdamWConfig(weight_decay=0.01))
    traj = []
    for g in (0.5, -0.3, 0.2):
        opt.step({"p": np.array([g])}, 1.0)
        traj.append(params["p"][0])
    d["adamw_traj"] = np.array(traj)
    rng = np.random.default_rng(3)
    a0, b0 = rng.normal(size=(7, 3)), rng.normal(size=5)
    params = {"a": a0.copy(), "b": b0.copy()}
    opt = AdamW(params, {"a": 0.05, "b": 0.002}, AdamWConfig())
    gs = rng.normal(size=(6, 7, 3)), rng.normal(size=(6, 5))
    scales = [1.0, 1.0, 0.5, 0.5, 0.25, 1.0]
    for i in range(6):
        opt.step({"a": gs[0][i], "b": gs[1][i]}, scales[i])
    d.update(adamw_a0=a0, adamw_b0=b0, adamw_ga=gs[0], adamw_gb=gs[1],
             adamw_scales=np.array(scales), adamw_a=params["a"], adamw_b=params["b"])
    # evaluate_field (field.py:93-135)
    rng = np.random.default_rng(4)
    n = 60
    quats = rng.normal(size=(n, 4))
    f = GaussianField(means=rng.uniform(-4, 4, size=(n, 3)),
                      log_scales=np.log(rng.uniform(0.5, 1.8, size=(n, 3))),
                      quaternions=quats, intensities=rng.uniform(0.1, 0.9, size=n))
    pts = rng.uniform(-5, 5, size=(500, 3))
    pts[-1] = [1e3, 1e3, 1e3]  # far query: clamp + delta path
    nbr = query(build_index(f.means), pts, 12)
    d.update(ev_means=f.means, ev_log_scales=f.log_scales, ev_quats=f.quaternions,
             ev_cvals=f.intensities, ev_points=pts, ev_nbr=nbr,
             ev_out=evaluate_field(pts, f, nbr))
    save("misc_cases", d)


if __name__ == "__main__":
    gen_train_cases()
    gen_knn_cases()
    gen_misc_cases()
