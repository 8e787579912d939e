"""Acquisition simulator (reference simulate.py) with the PSF quadrature on the GPU.

The reference integrates the ground-truth raster against each pixel's oriented
Gaussian PSF by dense tensor quadrature (19^3 nodes per pixel at the default
3 nodes per sigma, simulate.py:168-205) in numba on the CPU -- hours at fetal
scale.  Here that quadrature is ``gsvr_psf_quadrature`` (csrc/simulate.cu,
float64, the reference's rounding order), so the reference's OWN simulator
produces the cfg2-scale acquisitions used for quality comparisons.  Geometry,
per-slice motion streams, noise and masks are the reference's host arithmetic
(simulate.py:229-326), drawn from the same SeedSequence streams, so a stack
made here equals the reference's stack for the same arguments (tested against
the reference's 64^3 desk and cfg1 stacks, tests/test_gpu_simulate.py).

Data generation only: nothing here runs inside a fit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _dev
from ._native import check, lib
from .errors import InvalidParameterError
from .motion import SliceStack, SliceStates
from .psf import PsfModel, build_psf
from .volume import VolumeGrid

DEFAULT_ORIENTATIONS = ((0, 1, 2), (1, 2, 0), (2, 0, 1))  # simulate.py:26


@dataclass
class MotionParams:
    """simulate.py:29-37: per-slice Euler angles U(+-rot_max deg), shifts U(+-trans_max mm)."""
    rot_max: float = 6.0
    trans_max: float = 4.0
    seed: int = 0

    def __post_init__(self):
        if self.rot_max < 0 or self.trans_max < 0:
            raise InvalidParameterError("motion bounds must be non-negative")


@dataclass
class AcquisitionParams:
    """simulate.py:40-60."""
    inplane: float = 0.5
    thickness: float = 3.0
    noise_std: float = 0.02
    orientations: Sequence[Tuple[int, int, int]] = DEFAULT_ORIENTATIONS
    psf: Optional[PsfModel] = None
    nodes_per_sigma: int = 3
    background: bool = True

    def __post_init__(self):
        if self.inplane <= 0 or self.thickness <= 0:
            raise InvalidParameterError("spacings must be positive")
        if self.noise_std < 0:
            raise InvalidParameterError("noise_std must be non-negative")
        if self.nodes_per_sigma < 1:
            raise InvalidParameterError("nodes_per_sigma must be >= 1")
        for p in self.orientations:
            if sorted(p) != [0, 1, 2]:
                raise InvalidParameterError(f"orientation {p} is not an axis permutation")


# ---------------------------------------------------------------------------
# phantom (simulate.py:66-135): the same random draws in the same order, the
# same closed form; evaluated in chunks so a 256^3 raster stays in memory bounds

def _phantom_params(size_mm: float, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    p = {"axes": size_mm * np.array([0.44, 0.41, 0.38]),
         "ft": rng.integers(5, 8), "fp": rng.integers(4, 7),
         "phase": rng.uniform(0, 2 * np.pi, size=2)}
    p["dip_c"] = np.stack([rng.uniform([0.10, -0.25, -0.25], [0.40, 0.25, 0.25]),
                           rng.uniform([-0.40, -0.25, -0.25], [-0.10, 0.25, 0.25])])
    p["dip_s"] = rng.uniform(0.18, 0.28, size=(2, 3))
    p["blob_c"] = np.stack([rng.uniform([-0.30, 0.15, -0.45], [0.30, 0.50, 0.0]),
                            rng.uniform([-0.30, -0.50, 0.0], [0.30, -0.15, 0.45])])
    p["blob_s"] = rng.uniform(0.15, 0.22, size=(2, 3))
    p["tex_c"] = rng.uniform(-0.75, 0.75, size=(40, 3))
    p["tex_s"] = rng.uniform(0.06, 0.16, size=40)
    p["tex_a"] = rng.uniform(-0.12, 0.12, size=40)
    return p


def _phantom_chunk(x: np.ndarray, p: dict):
    xi = x / p["axes"]
    r = np.sqrt(np.sum(xi * xi, axis=-1))
    inside = r <= 1.0
    v = 0.72 - 0.35 * r * r
    theta = np.arccos(np.clip(xi[:, 2] / np.maximum(r, 1e-12), -1.0, 1.0))
    phi = np.arctan2(xi[:, 1], xi[:, 0])
    ripple = np.sin(p["ft"] * theta + p["phase"][0]) * np.sin(p["fp"] * phi + p["phase"][1])
    v = v + 0.28 * np.exp(-((r - 0.85) / 0.10) ** 2) * (0.55 + 0.45 * ripple)
    terms = [(c, s, -0.25) for c, s in zip(p["dip_c"], p["dip_s"])]
    terms += [(c, s, 0.15) for c, s in zip(p["blob_c"], p["blob_s"])]
    terms += list(zip(p["tex_c"], p["tex_s"], p["tex_a"]))
    for c, s, amp in terms:
        v = v + amp * np.exp(-np.sum(((xi - c) / s) ** 2, axis=-1))
    edge = np.clip((1.0 - r) / 0.08, 0.0, 1.0)
    return np.clip(v, 0.02, 1.0) * (edge * edge * (3.0 - 2.0 * edge)) * inside, inside


def phantom_intensity(points, size_mm: float, seed: int = 0, chunk: int = 1 << 20):
    """simulate.py:66-122: (value, inside) of the analytic brain phantom."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    p = _phantom_params(size_mm, seed)
    val, ins = np.empty(len(pts)), np.empty(len(pts), bool)
    for a in range(0, len(pts), chunk):
        val[a:a + chunk], ins[a:a + chunk] = _phantom_chunk(pts[a:a + chunk], p)
    return val, ins


def make_phantom(size: int, seed: int = 0, spacing: float = 0.5) -> VolumeGrid:
    """simulate.py:125-135: centred isotropic GT raster + support mask."""
    if size < 32:
        raise InvalidParameterError("phantom size must be >= 32")
    affine = np.diag([spacing, spacing, spacing, 1.0])
    affine[:3, 3] = -0.5 * (size - 1) * spacing
    grid = VolumeGrid(np.zeros((size, size, size)), affine)
    v, ins = phantom_intensity(grid.voxel_centers(), size_mm=size * spacing, seed=seed)
    return VolumeGrid(v.reshape(size, size, size), affine, mask=ins.reshape(size, size, size))


# ---------------------------------------------------------------------------
# geometry (simulate.py:208-242)

def _axis_nodes(sigma: float, nodes_per_sigma: int):
    """simulate.py:208-215: offsets over +-3 sigma and normalised Gaussian weights."""
    if sigma <= 0.0:
        return np.zeros(1), np.ones(1)
    m = 3 * nodes_per_sigma
    off = np.arange(-m, m + 1) * (sigma / nodes_per_sigma)
    w = np.exp(-0.5 * (off / sigma) ** 2)
    return off, w / w.sum()


def _euler_rotation(angles_rad: np.ndarray) -> np.ndarray:
    """simulate.py:218-227: Rz Ry Rx."""
    ax, ay, az = (float(a) for a in angles_rad)
    cx, sx, cy, sy, cz, sz = (math.cos(ax), math.sin(ax), math.cos(ay), math.sin(ay),
                              math.cos(az), math.sin(az))
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def _rotation_to_quat(R: np.ndarray) -> np.ndarray:
    """geometry.py:98-119 (scalar-first, w >= 0)."""
    t = np.trace(R)
    if t > 0:
        s = np.sqrt(t + 1.0) * 2
        q = np.array([0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s])
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = np.sqrt(max(R[i, i] - R[j, j] - R[k, k] + 1.0, 0.0)) * 2
        q = np.empty(4)
        q[0] = (R[k, j] - R[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (R[j, i] + R[i, j]) / s
        q[1 + k] = (R[k, i] + R[i, k]) / s
    if q[0] < 0:
        q = -q
    return q / np.linalg.norm(q)


def _stack_affine(gt: VolumeGrid, acq: AcquisitionParams, orientation):
    """simulate.py:229-242: stack covering the GT field of view, centred on it."""
    p0, p1, p2 = orientation
    extent = np.asarray(gt.sizes) * gt.spacing
    n = (int(np.ceil(extent[p0] / acq.inplane)), int(np.ceil(extent[p1] / acq.inplane)),
         int(np.ceil(extent[p2] / acq.thickness)))
    affine = np.eye(4)
    affine[:3, 0] = acq.inplane * np.eye(3)[p0]
    affine[:3, 1] = acq.inplane * np.eye(3)[p1]
    affine[:3, 2] = acq.thickness * np.eye(3)[p2]
    center = gt.index_to_world(0.5 * (np.asarray(gt.sizes) - 1))
    affine[:3, 3] = center - affine[:3, :3] @ (0.5 * np.array([n[0] - 1, n[1] - 1, n[2] - 1]))
    return affine, n


class _DeviceRaster:
    """GT raster + support uploaded once per protocol."""

    def __init__(self, gt: VolumeGrid):
        self.shape = tuple(int(v) for v in gt.sizes)
        self.vol = _dev.to_dev(np.ascontiguousarray(gt.data, dtype=np.float64), np.float64)
        sup = gt.mask if gt.mask is not None else np.ones(gt.sizes, bool)
        self.sup = _dev.to_dev(np.ascontiguousarray(sup, dtype=np.float64), np.float64)
        self.inv = np.ascontiguousarray(np.linalg.inv(gt.affine)[:3, :], dtype=np.float64)

    def quadrature(self, which, centers, sid, axes, nodes) -> np.ndarray:
        import ctypes
        M = len(centers)
        c_d = _dev.to_dev(centers, np.float64)
        s_d = _dev.to_dev(sid, np.int32)
        a_d = _dev.to_dev(axes, np.float64)
        n_d = _dev.to_dev(np.concatenate([np.concatenate(ax) for ax in nodes]), np.float64)
        out = _dev.empty((M,), np.float64)
        inv = (ctypes.c_double * 12)(*self.inv.ravel())
        nx, ny, nz = self.shape
        check(lib().gsvr_psf_quadrature(nx, ny, nz, _dev.ptr(which), ctypes.addressof(inv), M, _dev.ptr(c_d),
                                        _dev.ptr(s_d), _dev.ptr(a_d), len(nodes[0][0]), len(nodes[1][0]),
                                        len(nodes[2][0]), _dev.ptr(n_d), _dev.ptr(out), _dev.stream_ptr()),
              "psf quadrature")
        return _dev.to_host(out)


def simulate_stack(gt: VolumeGrid, acq: AcquisitionParams, motion: MotionParams,
                   orientation=(0, 1, 2), _raster: Optional[_DeviceRaster] = None
                   ) -> Tuple[SliceStack, SliceStates]:
    """simulate.py:245-315: one motion-corrupted stack and its true slice states.

    All slices' pixels go through ONE device quadrature launch per raster
    (intensity, then support); the per-slice RNG draws (motion, then noise)
    follow the reference's stream order exactly."""
    if np.max(gt.spacing) > acq.inplane + 1e-9:
        raise InvalidParameterError("GT spacing must be <= in-plane spacing")
    psf = acq.psf if acq.psf is not None else build_psf(acq.inplane, acq.thickness)
    affine, (nx, ny, ns) = _stack_affine(gt, acq, orientation)
    R_stack = affine[:3, :3] / np.linalg.norm(affine[:3, :3], axis=0)
    nodes = [_axis_nodes(s, acq.nodes_per_sigma) for s in psf.sigmas]
    center = gt.index_to_world(0.5 * (np.asarray(gt.sizes) - 1))
    uu, vv = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    pix = np.stack([uu, vv], axis=-1).reshape(-1, 2).astype(np.float64)
    streams = np.random.SeedSequence([motion.seed, *orientation]).spawn(ns)
    rngs, moved, axes = [], [], np.empty((ns, 3, 3))
    quats, trans = np.zeros((ns, 4)), np.zeros((ns, 3))
    for k in range(ns):
        rng = np.random.default_rng(streams[k])
        Rp = _euler_rotation(np.deg2rad(rng.uniform(-motion.rot_max, motion.rot_max, 3)))
        shift = rng.uniform(-motion.trans_max, motion.trans_max, 3)
        t_eff = center - Rp @ center + shift
        idx = np.concatenate([pix, np.full((len(pix), 1), float(k))], axis=1)
        nominal = idx @ affine[:3, :3].T + affine[:3, 3]
        moved.append(nominal @ Rp.T + t_eff)
        axes[k] = Rp @ R_stack
        quats[k], trans[k] = _rotation_to_quat(Rp), t_eff
        rngs.append(rng)
    raster = _raster or _DeviceRaster(gt)
    centers = np.ascontiguousarray(np.concatenate(moved))
    sid = np.repeat(np.arange(ns, dtype=np.int32), len(pix))
    vals = raster.quadrature(raster.vol, centers, sid, axes, nodes).reshape(ns, -1)
    cov = raster.quadrature(raster.sup, centers, sid, axes, nodes).reshape(ns, -1)
    data = np.zeros((nx, ny, ns))
    mask = np.zeros((nx, ny, ns), dtype=bool)
    for k in range(ns):
        v = vals[k]
        if acq.noise_std > 0:
            v = v + rngs[k].normal(0.0, acq.noise_std, size=v.shape)
        data[:, :, k] = v.reshape(nx, ny)
        anatomy = (cov[k] > 0.5).reshape(nx, ny)
        mask[:, :, k] = (anatomy.mean() >= 0.01) if acq.background else anatomy
    stack = SliceStack(data=data, affine=affine, inplane_spacing=np.array([acq.inplane, acq.inplane]),
                       thickness=acq.thickness, mask=mask)
    return stack, SliceStates(quats, trans, np.zeros(ns), np.zeros(ns))


def simulate_protocol(gt: VolumeGrid, acq: AcquisitionParams, motion: MotionParams
                      ) -> Tuple[List[SliceStack], List[SliceStates]]:
    """simulate.py:318-326: every stack of the protocol (raster uploaded once)."""
    raster = _DeviceRaster(gt)
    stacks, truths = [], []
    for o in acq.orientations:
        s, t = simulate_stack(gt, acq, motion, o, _raster=raster)
        stacks.append(s)
        truths.append(t)
    return stacks, truths
