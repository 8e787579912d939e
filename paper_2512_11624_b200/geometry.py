"""Small host-side rotation / covariance helpers (reference geometry.py).

These run on O(1)-sized host arrays (stack geometry, user-facing helpers).
Everything per primitive or per pixel runs in the CUDA library instead
(csrc/common.cuh restates the same maps on the device).
"""
from __future__ import annotations

import numpy as np

from .errors import InvalidParameterError

EIGENVALUE_FLOOR = 1e-6   # geometry.py:18
EXPONENT_CLAMP = -80.0    # geometry.py:22
_ROWS = np.array([0, 0, 0, 1, 1, 2])
_COLS = np.array([0, 1, 2, 1, 2, 2])


def quat_normalize(q):
    """geometry.py:28-34 (raises on zero / non-finite norm)."""
    q = np.asarray(q, dtype=np.float64)
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(n <= 1e-30) or not np.all(np.isfinite(n)):
        raise InvalidParameterError("quaternion with zero or non-finite norm")
    return q / n


def quat_to_rotation(q):
    """geometry.py:37-55: scalar-first quaternion(s) -> rotation matrices."""
    w, x, y, z = np.moveaxis(quat_normalize(q), -1, 0)
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def quat_from_axis_angle(axis, angle_rad):
    """geometry.py:88-96."""
    axis = np.asarray(axis, dtype=np.float64)
    n = np.linalg.norm(axis)
    if n == 0:
        raise InvalidParameterError("rotation axis must be nonzero")
    return np.concatenate([[np.cos(0.5 * angle_rad)], np.sin(0.5 * angle_rad) * axis / n])


def rotation_part(linear):
    """geometry.py:131-140: direction cosines of an affine's 3x3 block."""
    linear = np.asarray(linear, dtype=np.float64)
    norms = np.linalg.norm(linear, axis=0)
    if np.any(norms <= 0):
        raise InvalidParameterError("affine has a zero column")
    return linear / norms


def pack_sym6(A):
    """(..., 3, 3) -> (..., 6) in the order (00, 01, 02, 11, 12, 22)."""
    return np.asarray(A)[..., _ROWS, _COLS]


def unpack_sym6(v):
    v = np.asarray(v)
    A = np.empty(v.shape[:-1] + (3, 3), dtype=v.dtype)
    A[..., _ROWS, _COLS] = v
    A[..., _COLS, _ROWS] = v
    return A


def build_covariance(log_s, q):
    """geometry.py:143-150: R diag(exp(2 log_s)) R^T."""
    log_s = np.asarray(log_s)
    if not np.all(np.isfinite(log_s)):
        raise InvalidParameterError("non-finite log-scales")
    R = quat_to_rotation(q)
    return np.einsum("...ik,...k,...jk->...ij", R, np.exp(2.0 * log_s), R)
