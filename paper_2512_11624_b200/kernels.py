"""Drop-in for the reference's ``gsvr.kernels`` (kernels.py:41-203).

Same entry points, same positional arguments, results written into the
caller's arrays.  Arrays may be numpy (copied to / from the device) or CUDA
torch tensors (used in place).  The work runs in libgsvr_b200.so:
``render_forward`` -> gsvr_render_forward, ``train_step_backward`` ->
gsvr_train_step_backward (tile binning + the fused tile kernel).

Difference by design: the reference accumulates into n_blocks private buffers
that the caller sums in order (train.py:263-269); the device reduces in one
pass, so the full gradient lands in block 0 and the other blocks stay zero --
the caller's ordered sum is unchanged.

Threading: calls may come from several Python threads (ctypes releases the
GIL).  The host-buffer path holds a per-device lock for the whole call, so
overlapping calls on one device run one after the other; calls on different
devices run concurrently.
"""
from __future__ import annotations

import numpy as np

from . import _dev
from ._native import F32, F64, check, lib
from .errors import InvalidParameterError

EXP_CLAMP = -80.0  # kernels.py:25


def default_block_count(n_points: int) -> int:
    """kernels.py:201-203 (kept for API compatibility)."""
    return max(1, min(16, int(n_points)))


def _nbr(nbr):
    is64 = (nbr.dtype == np.int64) if isinstance(nbr, np.ndarray) else (str(nbr.dtype) == "torch.int64")
    return _dev.to_dev(nbr, np.int64 if is64 else np.int32), int(is64)


def render_forward(points, psf6, sigma, nbr, mu, cov6, cvals, delta, out):
    """kernels.py:41-75: out[p] = sigma_p * sum_k c e_k / (sum_k e_k + delta), u clamped at -80."""
    odt = np.float32 if str(getattr(out, "dtype", "")) in ("float32", "torch.float32") else np.float64
    M, K = (int(nbr.shape[0]), int(nbr.shape[1])) if len(nbr.shape) == 2 else (0, 0)
    if M == 0:
        return
    N = int(mu.shape[0])
    t = [_dev.to_dev(a, odt) for a in (points, psf6, sigma, mu, cov6, cvals)]
    nb, is64 = _nbr(nbr)
    res = _dev.empty((M,), odt)
    check(lib().gsvr_render_forward(F64 if odt == np.float64 else F32, M, K, *map(_dev.ptr, t[:3]),
                                    _dev.ptr(nb), is64, N, *map(_dev.ptr, t[3:]), float(delta),
                                    _dev.ptr(res), _dev.stream_ptr()), "render_forward")
    _dev.write_back(out, res)


def _is_host(a) -> bool:
    return not (hasattr(a, "is_cuda") and a.is_cuda)


def _host(a, dtype):
    """C-contiguous host array of dtype -> (keep-alive object, address)."""
    if isinstance(a, np.ndarray) or not hasattr(a, "data_ptr"):
        arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
        return arr, arr.ctypes.data
    t = a.detach().to(dtype=_dev._TORCH[np.dtype(dtype)]).contiguous()
    return t, t.data_ptr()


def _host_out(a, dtype):
    """Writable contiguous host view of a caller output (or a temporary + copy-back)."""
    if isinstance(a, np.ndarray):
        if a.dtype == dtype and a.flags.c_contiguous and a.flags.writeable:
            return a, a.ctypes.data, None
        tmp = np.ascontiguousarray(a, dtype=dtype)
        return tmp, tmp.ctypes.data, lambda: np.copyto(a, tmp, casting="unsafe")
    tdt = _dev._TORCH[np.dtype(dtype)]
    if a.dtype == tdt and a.is_contiguous():
        return a, a.data_ptr(), None
    tmp = a.detach().to(tdt).contiguous()
    return tmp, tmp.data_ptr(), lambda: a.copy_(tmp)


def train_step_backward(x0pts, sid, Rc, tvec, psf6s, sigma_s, wdata_s, I_obs, nbr, mu, cov6,
                        cvals, delta, n_blocks, I_hat, absres, dmu, dcov6, dc, dt, dRc, dpsf6,
                        dsigraw):
    """kernels.py:78-198: forward + L1 + analytic gradients, accumulated into the
    caller-zeroed (n_blocks, ...) buffers (block 0 receives the reduced sum).

    Host (numpy / CPU tensor) inputs go through gsvr_train_step_backward_host,
    which overlaps the neighbour upload with planning and binning; CUDA tensors
    are used in place by gsvr_train_step_backward."""
    P, K = int(nbr.shape[0]), int(nbr.shape[1])
    if P == 0:
        return
    if int(x0pts.shape[0]) != P or int(sid.shape[0]) != P:
        raise InvalidParameterError("x0pts / sid rows must match nbr")
    S, N = int(Rc.shape[0]), int(mu.shape[0])
    f64 = np.float64
    if all(_is_host(a) for a in (x0pts, nbr, I_obs, mu)):
        is64 = (nbr.dtype == np.int64) if isinstance(nbr, np.ndarray) else (str(nbr.dtype) == "torch.int64")
        keep, ptrs = [], []
        for a, dt_ in ((x0pts, f64), (sid, np.int32), (Rc, f64), (tvec, f64), (psf6s, f64), (sigma_s, f64),
                       (wdata_s, f64), (I_obs, f64), (nbr, np.int64 if is64 else np.int32)):
            k, ptr = _host(a, dt_)
            keep.append(k)
            ptrs.append(ptr)
        fkeep = [_host(a, f64) for a in (mu, cov6, cvals)]
        outs = [_host_out(I_hat, f64), _host_out(absres, f64)]
        gouts = [_host_out(g[0], f64) for g in (dmu, dcov6, dc, dt, dRc, dpsf6, dsigraw)]
        check(lib().gsvr_train_step_backward_host(
            P, K, S, N, *ptrs[:8], ptrs[8], int(is64), *[f[1] for f in fkeep], float(delta),
            *[o[1] for o in outs], *[o[1] for o in gouts], _dev.stream_ptr()), "train_step_backward")
        for o in outs + gouts:
            if o[2] is not None:
                o[2]()
        del keep, fkeep
        return
    ins = [_dev.to_dev(x0pts, f64), _dev.to_dev(sid, np.int32)] + [
        _dev.to_dev(a, f64) for a in (Rc, tvec, psf6s, sigma_s, wdata_s, I_obs)]
    nb, is64 = _nbr(nbr)
    fld = [_dev.to_dev(a, f64) for a in (mu, cov6, cvals)]
    o_ihat, o_abs = _dev.empty((P,), f64), _dev.empty((P,), f64)
    shapes = [(N, 3), (N, 6), (N,), (S, 3), (S, 3, 3), (S, 6), (S,)]
    grads = [_dev.zeros(s, f64) for s in shapes]
    check(lib().gsvr_train_step_backward(P, K, S, N, *map(_dev.ptr, ins), _dev.ptr(nb), is64,
                                         *map(_dev.ptr, fld), float(delta), _dev.ptr(o_ihat),
                                         _dev.ptr(o_abs), *map(_dev.ptr, grads),
                                         _dev.stream_ptr()), "train_step_backward")
    _dev.write_back(I_hat, o_ihat)
    _dev.write_back(absres, o_abs)
    for dst, g in zip((dmu, dcov6, dc, dt, dRc, dpsf6, dsigraw), grads):
        blk = dst[0]
        if isinstance(dst, np.ndarray):
            blk += _dev.to_host(g).reshape(blk.shape)
        else:
            blk += g.reshape(blk.shape).to(blk.device)

