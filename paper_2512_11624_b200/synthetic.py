"""Seeded synthetic acquisitions at the BASELINE.json configs.

The reference simulator (simulate.py) integrates a GT raster with 19^3-node PSF
quadrature per pixel -- hours at fetal scale -- and its FOV rule cannot produce
the cfg2-4 stack sizes.  For throughput runs this module builds the exact stack
geometry of a config (orthogonal stacks, simulate.py:26 orientation
permutations, centred), per-slice rigid motion drawn from per-slice
SeedSequence streams like simulate.py:278-284, and observations from an
analytic ellipsoidal "fetal brain" phantom sampled at the moved pixel positions
plus N(0, noise) -- the shape of the data, not its clinical realism.

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

ORIENTATIONS = ((0, 1, 2), (1, 2, 0), (2, 0, 1))


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


def phantom(x: np.ndarray) -> np.ndarray:
    """Ellipsoidal head/brain phantom in [0, 1] (world mm, centred at 0)."""
    def ell(c, r):
        return np.sum(((x - np.asarray(c)) / np.asarray(r)) ** 2, axis=-1)
    v = np.zeros(x.shape[:-1])
    skull = ell((0, 0, 0), (62, 52, 56))
    brain = ell((0, 0, 0), (55, 45, 50))
    v = np.where(skull <= 1.0, 0.25, v)
    v = np.where(brain <= 1.0, 0.55 + 0.15 * np.cos(x[..., 0] / 7.0) * np.sin(x[..., 1] / 9.0), v)
    for c, r, val in (((-18, 5, 4), (9, 14, 12), 0.9), ((18, 5, 4), (9, 14, 12), 0.9),
                      ((0, -20, -8), (16, 9, 10), 0.35), ((0, 22, 10), (6, 6, 18), 0.75)):
        v = np.where(ell(c, r) <= 1.0, val, v)
    return v


def _euler(a: np.ndarray) -> np.ndarray:
    """simulate.py:218-227 (Rz Ry Rx)."""
    cx, sx, cy, sy, cz, sz = math.cos(a[0]), math.sin(a[0]), math.cos(a[1]), math.sin(a[1]), \
        math.cos(a[2]), math.sin(a[2])
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


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
            vals = phantom(moved)
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
