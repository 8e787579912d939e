"""Observed-slice forward pass (reference render.py:22-65) on the device.

``render_observed`` validates like the reference (neighbour rows and id range,
rotation shapes) and evaluates Eq. 5 with clamp semantics through
``kernels.render_forward`` -> gsvr_render_forward (fp32 or fp64 as the field's
dtype).  The reference's Monte-Carlo oracle (render.py:68-100) is test-only and
not part of this package.
"""
from __future__ import annotations

import numpy as np

from . import kernels
from .errors import InvalidParameterError
from .field import DELTA, GaussianField
from .psf import PsfModel, rotated_psf_cov6


def render_observed(points_world, slice_rotations, field: GaussianField, psf: PsfModel,
                    neighbor_ids, sigma_slice=1.0, delta: float = DELTA) -> np.ndarray:
    """render.py:22-65: (M,) analytic observed intensities at corrected points.

    ``slice_rotations`` is (3, 3) for one rotation shared by all points or
    (M, 3, 3) per point; ``sigma_slice`` broadcasts to (M,)."""
    dtype = field.means.dtype
    points = np.ascontiguousarray(np.atleast_2d(points_world), dtype=dtype)
    M = points.shape[0]
    nbr = np.ascontiguousarray(np.atleast_2d(neighbor_ids), dtype=np.int64)
    if nbr.shape[0] != M:
        raise InvalidParameterError("neighbor_ids rows must match points")
    if nbr.size and (nbr.min() < 0 or nbr.max() >= field.count):
        raise InvalidParameterError("neighbor id out of range")
    R = np.asarray(slice_rotations)
    if R.shape == (3, 3):
        psf6 = np.broadcast_to(rotated_psf_cov6(R, psf), (M, 6))
    elif R.shape == (M, 3, 3):
        psf6 = rotated_psf_cov6(R, psf)
    else:
        raise InvalidParameterError("slice_rotations must be (3,3) or (M,3,3)")
    psf6 = np.ascontiguousarray(psf6, dtype=dtype)
    sigma = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma_slice, dtype=dtype), (M,)))
    out = np.empty(M, dtype=dtype)
    if M == 0 or nbr.shape[1] == 0:
        # the reference's kernel leaves den = delta, num = 0 -> 0 (kernels.py:57-75)
        out[:] = 0.0
        return out
    kernels.render_forward(points, psf6, sigma, nbr,
                           np.ascontiguousarray(field.means, dtype=dtype),
                           np.ascontiguousarray(field.covariances6(), dtype=dtype),
                           np.ascontiguousarray(field.intensities, dtype=dtype),
                           float(delta), out)
    return out
