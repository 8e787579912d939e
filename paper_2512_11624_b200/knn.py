"""Exact top-K nearest means on the device (reference knn.py:20-75).

``build_index`` snapshots the means into the device grid (gsvr_knn_build);
``query`` returns (M, K) int64 ids ordered by (distance, index) with the
reference's boundary-tie rule (gsvr_knn_query).  Same validation and errors.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _dev
from ._native import check, lib
from .errors import InvalidParameterError


class _Handle:
    def __init__(self, raw):
        self.raw = raw

    def __del__(self):
        try:
            if self.raw:
                lib().gsvr_knn_free(self.raw)
        except Exception:  # interpreter shutdown
            pass


@dataclass
class NeighborIndex:
    """Device grid over a snapshot of primitive means (knn.py:20-30)."""

    means: np.ndarray
    handle: _Handle = field(repr=False)
    epoch: int = 0

    @property
    def count(self) -> int:
        return self.means.shape[0]


def build_index(means, epoch: int = 0) -> NeighborIndex:
    """knn.py:33-40."""
    m = np.ascontiguousarray(np.atleast_2d(np.asarray(means if not hasattr(means, "cpu")
                                                       else means.cpu().numpy())), dtype=np.float64)
    if m.ndim != 2 or m.shape[1] != 3 or m.shape[0] < 1:
        raise InvalidParameterError("means must be a non-empty (N, 3) array")
    if not np.all(np.isfinite(m)):
        raise InvalidParameterError("non-finite means")
    return NeighborIndex(m.copy(), _build_handle(_dev.to_dev(m, np.float64)), epoch)


def _build_handle(means_dev) -> _Handle:
    raw = ctypes.c_void_p()
    check(lib().gsvr_knn_build(int(means_dev.shape[0]), _dev.ptr(means_dev), ctypes.byref(raw),
                               _dev.stream_ptr()), "build_index")
    return _Handle(raw)


def query(index: NeighborIndex, points, K: int) -> np.ndarray:
    """knn.py:43-75: (M, K) int64, rows sorted by distance, ties by index."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    n = index.count
    if K < 1 or K > n:
        raise InvalidParameterError(f"K must be in [1, {n}], got {K}")
    out = query_device(index, _dev.to_dev(pts, np.float64), K)
    return _dev.to_host(out)


def query_device(index: NeighborIndex, points_dev, K: int, out_i64: bool = True):
    M = int(points_dev.shape[0])
    out = _dev.empty((M, K), np.int64 if out_i64 else np.int32)
    check(lib().gsvr_knn_query(index.handle.raw, M, _dev.ptr(points_dev), int(K), _dev.ptr(out),
                               int(out_i64), _dev.stream_ptr()), "query")
    return out
