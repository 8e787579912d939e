"""The fit's setup on the device.

``DeviceStacks`` puts every stack raster (values + mask) in HBM once; from it
csrc/init.cu builds

* the point batch (``device_point_batch``; reference motion.py:183-237
  ``build_point_batch``), which stays on the device and feeds
  ``engine.DeviceBatch`` without a host round trip, and
* the content-adaptive initial field (``device_init_field``; reference
  initialization.py:44-152 ``sample_init_positions`` + ``init_field``): the
  gradient-weighted draw of numpy's ``Generator.choice`` with the host PCG64
  uniforms, the lifting of the drawn pixels and their source intensities.

Both are bit-identical to the reference's numpy on the same host (and to
``motion.build_point_batch`` / ``initialization.sample_init_positions`` /
``initialization.init_field``, which restate it on the host); init.cu's header
lists the numpy / glibc / OpenBLAS operation orders this relies on, and
tests/test_gpu_init.py pins them.
"""
from __future__ import annotations

import ctypes
import math
import warnings
from typing import Sequence

import numpy as np
import torch

from . import _dev
from ._native import check, lib
from .errors import InvalidParameterError
from .field import GaussianField
from .initialization import InitConfig
from .motion import PointBatch, SliceStack

f64, i32 = np.float64, np.int32


class _StackView(ctypes.Structure):
    """include/gsvr_b200.h gsvr_stack_view."""
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("ns", ctypes.c_int64),
                ("data", ctypes.c_void_p), ("mask", ctypes.c_void_p), ("affine", ctypes.c_double * 16)]


class DeviceStacks:
    """Stack rasters (float64 values, uint8 mask, C order) resident on the device."""

    def __init__(self, stacks: Sequence[SliceStack]):
        if len(stacks) == 0:
            raise InvalidParameterError("need at least one stack")
        self.stacks = list(stacks)
        self._keep = []
        self.views = (_StackView * len(stacks))()
        for i, st in enumerate(self.stacks):
            d = _dev.to_dev(st.data, f64)
            m = _dev.to_dev(np.ascontiguousarray(st.mask).view(np.uint8), np.uint8)
            self._keep += [d, m]
            v = self.views[i]
            v.nx, v.ny, v.ns = st.data.shape
            v.data, v.mask = _dev.ptr(d), _dev.ptr(m)
            v.affine[:] = [float(a) for a in np.asarray(st.affine, dtype=f64).ravel()]
        self.slice_to_stack = np.concatenate([np.full(s.n_slices, t, dtype=i32)
                                              for t, s in enumerate(self.stacks)])
        self.counts = np.zeros(len(self.slice_to_stack), dtype=np.int64)
        check(lib().gsvr_stack_slice_counts(len(self.stacks), self.views,
                                            self.counts.ctypes.data_as(ctypes.c_void_p),
                                            _dev.stream_ptr()), "stack slice counts")

    @property
    def n_slices(self) -> int:
        return len(self.slice_to_stack)


class DevicePointBatch:
    """motion.PointBatch whose per-point arrays live on the device (x0 (P, 3),
    slice ids, values); the host arrays are fetched on first access."""

    def __init__(self, x0: torch.Tensor, sid: torch.Tensor, values: torch.Tensor,
                 slice_to_stack: np.ndarray, stack_rotations: np.ndarray, counts: np.ndarray):
        self.x0, self.sid, self.values = x0, sid, values
        self.slice_to_stack = np.asarray(slice_to_stack, dtype=i32)
        self.stack_rotations = stack_rotations
        self._counts = np.asarray(counts, dtype=np.int64)
        self._host = None

    @property
    def n_points(self) -> int:
        return int(self.x0.shape[0])

    @property
    def n_slices(self) -> int:
        return len(self.slice_to_stack)

    def slice_counts(self) -> np.ndarray:
        return self._counts.copy()

    def host(self) -> PointBatch:
        if self._host is None:
            self._host = PointBatch(_dev.to_host(self.x0), _dev.to_host(self.sid),
                                    np.repeat(self.slice_to_stack, self._counts).astype(i32),
                                    _dev.to_host(self.values), self.slice_to_stack, self.stack_rotations)
        return self._host

    # PointBatch's host arrays, fetched once
    lifted = property(lambda self: self.host().lifted)
    slice_ids = property(lambda self: self.host().slice_ids)
    stack_ids = property(lambda self: self.host().stack_ids)
    intensities = property(lambda self: self.host().intensities)

    def shard(self, rank: int, world: int):
        """parallel.shard_batch on the device: this rank's slice range (slice
        ids renumbered from 0) and its global slice slice."""
        from .parallel import partition_slices
        b = partition_slices(self._counts, world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        off = np.concatenate([[0], np.cumsum(self._counts)])
        p0, p1 = int(off[lo]), int(off[hi])
        sub = DevicePointBatch(self.x0[p0:p1], self.sid[p0:p1] - lo, self.values[p0:p1],
                               self.slice_to_stack[lo:hi], self.stack_rotations, self._counts[lo:hi])
        return sub, slice(lo, hi)


def device_point_batch(ds: DeviceStacks) -> DevicePointBatch:
    """motion.py:210-237 on the device (csrc/init.cu k_build_points)."""
    P = int(ds.counts.sum())
    if P == 0:
        raise InvalidParameterError("no masked pixels in any stack")
    x0, sid, vals = _dev.empty((P, 3), f64), _dev.empty((P,), i32), _dev.empty((P,), f64)
    check(lib().gsvr_build_points(len(ds.stacks), ds.views, ds.counts.ctypes.data_as(ctypes.c_void_p),
                                  _dev.ptr(x0), _dev.ptr(sid), _dev.ptr(vals), _dev.stream_ptr()),
          "point batch")
    return DevicePointBatch(x0, sid, vals, ds.slice_to_stack, np.stack([s.rotation for s in ds.stacks]),
                            ds.counts)


def device_init_field(ds: DeviceStacks, cfg: InitConfig) -> GaussianField:
    """initialization.py:80-152 on the device: the N drawn positions (numpy's
    Generator.choice over the gradient weights, the host PCG64 uniforms) and
    the initial field around them."""
    n = cfg.n_gaussians
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    u = _dev.to_dev(rng.random(n), f64)  # Generator.choice's uniform draws (after its cdf)
    pos = _dev.empty((n, 3), f64)
    fallback = ctypes.c_int(0)
    msum = ctypes.c_double(0.0)
    want_mean = cfg.intensity_policy == "mean"
    f32 = False
    if want_mean:  # np.mean accumulates float32 data in float32, integers (exactly) in float64
        cat = np.result_type(*[s.data.dtype for s in ds.stacks])  # np.concatenate's dtype
        f32 = cat == np.float32
        if not (f32 or cat == np.float64 or cat.kind in "iub"):
            raise InvalidParameterError(f"intensity_policy='mean' on the device needs float64, float32 or "
                                        f"integer stack data, got {cat}")
    check(lib().gsvr_init_sample(len(ds.stacks), ds.views, ds.counts.ctypes.data_as(ctypes.c_void_p),
                                 float(cfg.lambda_init), n, _dev.ptr(u), _dev.ptr(pos), ctypes.byref(fallback),
                                 ctypes.byref(msum) if want_mean else None, int(f32), _dev.stream_ptr()),
          "init sampling")
    if fallback.value:
        warnings.warn("zero sampling mass (flat image with lambda_init=0); "
                      "falling back to uniform sampling")
    if want_mean:
        P = int(ds.counts.sum())
        mean = np.float32(msum.value) / P if f32 else np.float64(msum.value) / P  # _methods._mean
        c = torch.full((n,), float(mean), dtype=torch.float64, device=pos.device)
    else:
        inv = np.concatenate([np.linalg.inv(s.affine).ravel() for s in ds.stacks]).astype(f64)
        c = _dev.empty((n,), f64)
        left = ctypes.c_int64(0)
        check(lib().gsvr_init_source_intensity(len(ds.stacks), ds.views, inv.ctypes.data_as(ctypes.c_void_p), n,
                                               _dev.ptr(pos), _dev.ptr(c), ctypes.byref(left),
                                               _dev.stream_ptr()), "init intensities")
        if left.value:
            raise InvalidParameterError("position does not coincide with any stack pixel")
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    return GaussianField(_dev.to_host(pos), np.full((n, 3), math.log(cfg.initial_scale)), q, _dev.to_host(c))
