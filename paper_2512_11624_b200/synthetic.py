"""Seeded synthetic acquisitions at the BASELINE.json configs.

The reference simulator (simulate.py) integrates a GT raster with 19^3-node PSF
quadrature per pixel -- hours at fetal scale -- and its FOV rule cannot produce
the cfg2-4 stack sizes.  For throughput runs this module builds the exact stack
geometry of a config (orthogonal stacks, simulate.py:26 orientation
permutations, centred), per-slice rigid motion drawn from per-slice
SeedSequence streams like simulate.py:278-284, and observations from an
analytic ellipsoidal "fetal brain" phantom integrated over the slice profile
(through-plane Gaussian quadrature at 1-sigma node spacing over +-3 sigma, as
simulate._axis_nodes; the in-plane PSF, sigma ~0.5 pixel, is not integrated)
at the moved pixel positions plus N(0, noise).

Configs (BASELINE.json "configs"):
  cfg1: 3 stacks 64x64x16 @ 1x1x4 mm, 10k Gaussians, no motion
  cfg2: 3 stacks 256x256x30 @ 0.8x0.8x3.5 mm, 200k Gaussians, motion
  cfg3: 6 stacks 320x320x40 @ 0.7x0.7x3 mm, 500k Gaussians, motion
  cfg4: 12 stacks 320x320x40 @ 0.7x0.7x3 mm, 2M Gaussians, heavy motion
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .motion import SliceStack, SliceStates

from .psf import FWHM_TO_SIGMA

ORIENTATIONS = ((0, 1, 2), (1, 2, 0), (2, 0, 1))
_NODE_OFF = np.arange(-3.0, 4.0)                 # through-plane nodes, units of sigma
_NODE_W = np.exp(-0.5 * _NODE_OFF ** 2) / np.exp(-0.5 * _NODE_OFF ** 2).sum()


@dataclass(frozen=True)
class SyntheticConfig:
    name: str
    n_stacks: int
    nx: int
    ny: int
    n_slices: int
    inplane: float
    thickness: float
    n_gaussians: int
    rot_max_deg: float
    trans_max_mm: float
    noise_std: float = 0.02


CONFIGS = {
    "cfg1": SyntheticConfig("cfg1", 3, 64, 64, 16, 1.0, 4.0, 10_000, 0.0, 0.0, 0.0),
    "cfg2": SyntheticConfig("cfg2", 3, 256, 256, 30, 0.8, 3.5, 200_000, 6.0, 4.0),
    "cfg3": SyntheticConfig("cfg3", 6, 320, 320, 40, 0.7, 3.0, 500_000, 6.0, 4.0),
    "cfg4": SyntheticConfig("cfg4", 12, 320, 320, 40, 0.7, 3.0, 2_000_000, 10.0, 6.0),
}


_ELLIPSES = (((-18, 5, 4), (9, 14, 12), 0.9), ((18, 5, 4), (9, 14, 12), 0.9),
             ((0, -20, -8), (16, 9, 10), 0.35), ((0, 22, 10), (6, 6, 18), 0.75))


def phantom(x):
    """Ellipsoidal head/brain phantom in [0, 1] (world mm, centred at 0).
    Accepts numpy arrays or torch tensors (evaluated where they live)."""
    xp = np
    if not isinstance(x, np.ndarray):
        import torch as xp  # noqa: N813  (same expression on the device)

    def ell(c, r):
        d = [(x[..., i] - c[i]) / r[i] for i in range(3)]
        return d[0] * d[0] + d[1] * d[1] + d[2] * d[2]
    v = xp.zeros_like(x[..., 0])
    v = xp.where(ell((0, 0, 0), (62, 52, 56)) <= 1.0, 0.25, v)
    v = xp.where(ell((0, 0, 0), (55, 45, 50)) <= 1.0,
                 0.55 + 0.15 * xp.cos(x[..., 0] / 7.0) * xp.sin(x[..., 1] / 9.0), v)
    for c, r, val in _ELLIPSES:
        v = xp.where(ell(c, r) <= 1.0, val, v)
    return v


def _euler(a: np.ndarray) -> np.ndarray:
    """simulate.py:218-227 (Rz Ry Rx)."""
    cx, sx, cy, sy, cz, sz = math.cos(a[0]), math.sin(a[0]), math.cos(a[1]), math.sin(a[1]), \
        math.cos(a[2]), math.sin(a[2])
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def _integrate(points: np.ndarray, step: np.ndarray) -> np.ndarray:
    """Through-plane quadrature of the phantom at points +- k * step (on the GPU
    when one is present -- data generation only, not the measured path)."""
    try:
        import torch
        if torch.cuda.is_available():
            x = torch.from_numpy(points).cuda()
            st = torch.from_numpy(np.asarray(step)).cuda()
            acc = torch.zeros(len(points), dtype=torch.float64, device="cuda")
            for off, wgt in zip(_NODE_OFF, _NODE_W):
                acc += float(wgt) * phantom(x + float(off) * st)
            return acc.cpu().numpy()
    except ImportError:
        pass
    acc = np.zeros(len(points))
    for off, wgt in zip(_NODE_OFF, _NODE_W):
        acc += wgt * phantom(points + off * step)
    return acc


def make_stacks(cfg: SyntheticConfig, seed: int = 0) -> Tuple[List[SliceStack], SliceStates]:
    """Stacks of the config and the true per-slice states (rotation about the
    volume centre, as simulate.py:286-288)."""
    stacks, quats, trans = [], [], []
    for t in range(cfg.n_stacks):
        o = ORIENTATIONS[t % 3]
        affine = np.eye(4)
        affine[:3, 0] = cfg.inplane * np.eye(3)[o[0]]
        affine[:3, 1] = cfg.inplane * np.eye(3)[o[1]]
        affine[:3, 2] = cfg.thickness * np.eye(3)[o[2]]
        half = 0.5 * np.array([cfg.nx - 1, cfg.ny - 1, cfg.n_slices - 1])
        affine[:3, 3] = -affine[:3, :3] @ half
        data = np.empty((cfg.nx, cfg.ny, cfg.n_slices))
        uu, vv = np.meshgrid(np.arange(cfg.nx), np.arange(cfg.ny), indexing="ij")
        pix = np.stack([uu, vv], -1).reshape(-1, 2).astype(np.float64)
        streams = np.random.SeedSequence([seed, t, *o]).spawn(cfg.n_slices)
        for k in range(cfg.n_slices):
            rng = np.random.default_rng(streams[k])
            ang = np.deg2rad(rng.uniform(-cfg.rot_max_deg, cfg.rot_max_deg, 3))
            shift = rng.uniform(-cfg.trans_max_mm, cfg.trans_max_mm, 3)
            Rp = _euler(ang)
            idx = np.concatenate([pix, np.full((len(pix), 1), float(k))], axis=1)
            moved = (idx @ affine[:3, :3].T + affine[:3, 3]) @ Rp.T + shift
            normal = Rp @ (affine[:3, 2] / np.linalg.norm(affine[:3, 2]))
            sz = cfg.thickness * FWHM_TO_SIGMA
            vals = _integrate(moved, normal * sz)
            if cfg.noise_std > 0:
                vals = vals + rng.normal(0.0, cfg.noise_std, size=vals.shape)
            data[:, :, k] = vals.reshape(cfg.nx, cfg.ny)
            w = math.sqrt(max(0.0, 1.0 + np.trace(Rp))) / 2.0
            q = np.array([w, (Rp[2, 1] - Rp[1, 2]) / (4 * w), (Rp[0, 2] - Rp[2, 0]) / (4 * w),
                          (Rp[1, 0] - Rp[0, 1]) / (4 * w)])
            quats.append(q)
            trans.append(shift)
        stacks.append(SliceStack(data=data, affine=affine,
                                 inplane_spacing=np.array([cfg.inplane, cfg.inplane]),
                                 thickness=cfg.thickness))
    S = len(quats)
    truth = SliceStates(np.array(quats), np.array(trans), np.zeros(S), np.zeros(S))
    return stacks, truth
