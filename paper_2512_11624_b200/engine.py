"""Device-resident reconstruction state and the per-epoch step (train.py:373-497).

Everything per pixel, per (tile, Gaussian) and per primitive stays in HBM
between epochs; one small pinned read-back per epoch carries the loss terms,
the staleness measure and the error flags (the reference's NaN / floor /
non-finite checks).  Kernel sequence per epoch:

    [refresh: device K-NN + (slice, tile) binning]      gsvr_batch_refresh
    fused tile forward + L1 + backward                  gsvr_train_tiles
    [multi-GPU: NCCL all-reduce of the field gradient]  parallel.Comm
    slice chain + masked AdamW + next slice inputs      gsvr_slice_adamw_step
    field chain + AdamW + next covariances / reg / floor gsvr_field_adamw_step
    staleness of the next epoch's points                gsvr_batch_displacement
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional

import numpy as np
import torch

from . import _dev
from ._native import check, lib
from .errors import InvalidParameterError, NumericalDegeneracyError, TrainingDivergedError
from .field import DELTA, GaussianField, evaluate_field_device
from .motion import PointBatch, SliceStates

f64, i32, i64 = np.float64, np.int32, np.int64
_NONE = (1 << 64) - 1  # "no index" marker of the device atomicMin flags


def pick_tile_points(K: int, want: int = 256) -> int:
    tp = want
    while tp > 1 and tp * K > 65535:
        tp //= 2
    return tp


class DeviceBatch:
    """A PointBatch in the tile layout of csrc/batch.cuh (created once per fit)."""

    def __init__(self, batch: PointBatch, K: int = 50, tile_points: Optional[int] = None,
                 I_obs=None):
        self.P, self.S = batch.n_points, batch.n_slices
        if hasattr(batch, "x0"):  # device_setup.DevicePointBatch: already resident
            self.x0, self.sid = batch.x0, batch.sid
            self.I_obs = batch.values if I_obs is None else _dev.to_dev(I_obs, f64)
        else:
            self.x0 = _dev.to_dev(batch.lifted, f64)
            self.sid = _dev.to_dev(batch.slice_ids, i32)
            self.I_obs = _dev.to_dev(batch.intensities if I_obs is None else I_obs, f64)
        self.stack_rots = _dev.to_dev(batch.stack_rotations, f64)
        self.s2t = _dev.to_dev(batch.slice_to_stack, i32)
        self.counts_host = batch.slice_counts().astype(f64)
        self.counts = _dev.to_dev(self.counts_host, f64)
        self.tile_points = tile_points or pick_tile_points(K)
        raw = ctypes.c_void_p()
        check(lib().gsvr_batch_create(self.P, self.S, _dev.ptr(self.x0), _dev.ptr(self.sid),
                                      _dev.ptr(self.I_obs), self.tile_points, ctypes.byref(raw),
                                      _dev.stream_ptr()), "point batch")
        self.raw = raw
        self.K = None

    def __del__(self):
        try:
            if getattr(self, "raw", None):
                lib().gsvr_batch_free(self.raw)
                self.raw = None
        except Exception:
            pass

    @property
    def n_tiles(self) -> int:
        return int(lib().gsvr_batch_tiles(self.raw))

    @property
    def tile_gaussians(self) -> int:
        return int(lib().gsvr_batch_tile_gaussians(self.raw))

    def bin(self, neighbor_ids, N: int) -> None:
        """(slice, tile) binning of caller-supplied (P, K) neighbour ids."""
        nbr = neighbor_ids if isinstance(neighbor_ids, torch.Tensor) else np.asarray(neighbor_ids)
        if len(nbr.shape) != 2 or nbr.shape[0] != self.P:
            raise InvalidParameterError("neighbor_ids must be (P, K) matching the batch")
        is64 = str(nbr.dtype) in ("int64", "torch.int64")
        nd = _dev.to_dev(nbr, i64 if is64 else i32)
        K = int(nbr.shape[1])
        check(lib().gsvr_batch_bin(self.raw, K, int(N), _dev.ptr(nd), int(is64), _dev.stream_ptr()),
              "binning")
        self.K = K

    def refresh(self, index, K: int, Rc, tvec) -> None:
        """Device K-NN of the corrected points against ``index`` + binning."""
        check(lib().gsvr_batch_refresh(self.raw, index.handle.raw, int(K), _dev.ptr(Rc),
                                       _dev.ptr(tvec), _dev.stream_ptr()), "neighbour refresh")
        self.K = int(K)

    def tile_info(self):
        """(tile_start, tile_n, tile_slice, uoff, gid, perm) as host arrays."""
        T, U = self.n_tiles, self.tile_gaussians
        ts, tn, tsl = _dev.empty((T,), i64), _dev.empty((T,), i32), _dev.empty((T,), i32)
        uoff, gid = _dev.empty((T + 1,), i32), _dev.empty((max(U, 1),), i32)
        perm = _dev.empty((self.P,), i32)
        check(lib().gsvr_batch_tile_info(self.raw, _dev.ptr(ts), _dev.ptr(tn), _dev.ptr(tsl),
                                         _dev.ptr(uoff), _dev.ptr(gid), _dev.ptr(perm),
                                         _dev.stream_ptr()))
        return tuple(_dev.to_host(x) for x in (ts, tn, tsl, uoff, gid[:U], perm))

    def tile_geometry(self):
        """(origin (T,3), basis (T,6), ab (P,2)) as host arrays."""
        T = self.n_tiles
        o, b, ab = _dev.empty((T, 3), f64), _dev.empty((T, 6), f64), _dev.empty((self.P, 2), np.float32)
        check(lib().gsvr_batch_tile_geometry(self.raw, _dev.ptr(o), _dev.ptr(b), _dev.ptr(ab),
                                             _dev.stream_ptr()))
        return _dev.to_host(o), _dev.to_host(b), _dev.to_host(ab)

    @property
    def planar(self) -> bool:
        return bool(lib().gsvr_batch_is_planar(self.raw))

    def neighbors(self) -> torch.Tensor:
        out = _dev.empty((self.P, self.K), i64)
        check(lib().gsvr_batch_neighbors(self.raw, _dev.ptr(out), _dev.stream_ptr()), "neighbors")
        return out

    def corrected_points(self, Rc, tvec) -> torch.Tensor:
        out = _dev.empty((self.P, 3), f64)
        check(lib().gsvr_corrected_points(self.P, _dev.ptr(self.x0), _dev.ptr(self.sid), _dev.ptr(Rc),
                                          _dev.ptr(tvec), _dev.ptr(out), _dev.stream_ptr()))
        return out


class FitEngine:
    """Field + slice parameters, AdamW moments and gradient buffers in HBM."""

    def __init__(self, dbatch: DeviceBatch, field: GaussianField, states: SliceStates,
                 psf_diags, loss_cfg, optim_cfg, comm=None, slice_offset: int = 0,
                 point_offset: int = 0, total_points: Optional[int] = None):
        self.b = dbatch
        # global point range of this rank's shard (reseed draws over all points)
        self.point_offset = point_offset
        self.total_points = dbatch.P if total_points is None else total_points
        self.loss_cfg, self.optim_cfg = loss_cfg, optim_cfg
        self.comm = comm
        self.S = dbatch.S
        self.slice_offset = slice_offset  # global id of local slice 0 (sharded runs)
        self.psf_diags = _dev.to_dev(np.asarray(psf_diags, dtype=f64), f64)
        self.set_field(field)
        st = np.concatenate([states.quaternions, states.translations, states.log_sigma[:, None],
                             states.eta[:, None]], axis=1)
        self.sstate = _dev.to_dev(st, f64)
        self.sm, self.sv = _dev.zeros((self.S, 9), f64), _dev.zeros((self.S, 9), f64)
        self.dslice = _dev.zeros((self.S, 20), f64)
        self.Rc, self.tv = _dev.empty((self.S, 9), f64), _dev.empty((self.S, 3), f64)
        self.p6, self.sig, self.w = (_dev.empty((self.S, 6), f64), _dev.empty((self.S,), f64),
                                     _dev.empty((self.S,), f64))
        self.Rc_ref, self.t_ref = None, None
        # per-epoch status read back with ONE copy: loss terms (4), staleness (1),
        # eigen-floor index and non-finite index (int64 views), pad
        self.status = _dev.zeros((8,), f64)
        self.loss = self.status[0:4]
        self.disp = self.status[4:5]
        self.floor = self.status[5:6].view(torch.int64)
        self.nonfinite = self.status[6:7].view(torch.int64)
        self.host = torch.empty(8, dtype=torch.float64, pin_memory=True)
        self.host_i = self.host.view(torch.int64)
        self.field_t = 0
        self.slice_t = 0
        self.floor_host = _NONE
        # the slice step and staleness pass run on a side stream beside the
        # field step (disjoint buffers); the epoch ends waiting for both.  High
        # priority: its single-block slice step must not queue behind the
        # field step's blocks, which fill every SM
        self._side = torch.cuda.Stream(priority=-1)
        self._ev_train, self._ev_slice = torch.cuda.Event(), torch.cuda.Event()
        self._slice_step(step_mask=0, lr_scale=1.0)  # slice inputs of the start state
        self._field_prep()
        self.sync_floor()

    def sync_floor(self) -> None:
        self.host.copy_(self.status)
        self.floor_host = int(self.host_i[5]) & _NONE

    # -- state -------------------------------------------------------------
    def set_field(self, field: GaussianField) -> None:
        self.N = field.count
        self.mu = _dev.to_dev(field.means, f64)
        self.ls = _dev.to_dev(field.log_scales, f64)
        self.q = _dev.to_dev(field.quaternions, f64)
        self.c = _dev.to_dev(field.intensities, f64)
        self._alloc_field_buffers()

    def _alloc_field_buffers(self):
        # a reseed keeps N: zero the existing buffers instead of allocating anew
        if getattr(self, "fm", None) is not None and self.fm.shape[0] == self.N:
            for t in (self.fm, self.fv, self.dfield, self.fstats):
                t.zero_()
        else:
            self.fm, self.fv = _dev.zeros((self.N, 11), f64), _dev.zeros((self.N, 11), f64)
            self.dfield = _dev.zeros((self.N, 10), np.float32)
            self.cov6 = _dev.empty((self.N, 6), f64)
            # the field step's private workspace (regulariser partials, flags)
            self.fstats = _dev.zeros((int(lib().gsvr_field_workspace_bytes()) // 8,), f64)
        self.field_t = 0

    def reset_optimizers(self):
        self.fm.zero_()
        self.fv.zero_()
        self.sm.zero_()
        self.sv.zero_()
        self.field_t = 0
        self.slice_t = 0

    def field_host(self) -> GaussianField:
        return GaussianField(_dev.to_host(self.mu), _dev.to_host(self.ls), _dev.to_host(self.q),
                             _dev.to_host(self.c))

    def states_host(self) -> SliceStates:
        st = _dev.to_host(self.sstate)
        return SliceStates(st[:, 0:4], st[:, 4:7], st[:, 7], st[:, 8])

    # -- kernels -----------------------------------------------------------
    def _adam(self):
        a = self.optim_cfg.adamw
        return a.betas[0], a.betas[1], a.eps, a.weight_decay

    def _field_prep(self):
        self._field_kernel(do_step=False, lr_scale=1.0)

    def _field_kernel(self, do_step: bool, lr_scale: float):
        o = self.optim_cfg
        lrs = (ctypes.c_double * 4)(o.lr_means, o.lr_log_scales, o.lr_quaternions, o.lr_intensities)
        b1, b2, eps, wd = self._adam()
        if do_step:
            self.field_t += 1
        t = max(self.field_t, 1)
        check(lib().gsvr_field_adamw_step(
            self.N, _dev.ptr(self.mu), _dev.ptr(self.ls), _dev.ptr(self.q), _dev.ptr(self.c),
            _dev.ptr(self.fm), _dev.ptr(self.fv), _dev.ptr(self.dfield), self.loss_cfg.lambda_reg,
            self.loss_cfg.s_target, lrs, lr_scale, b1, b2, eps, wd, 1.0 - b1 ** t, 1.0 - b2 ** t,
            int(do_step), _dev.ptr(self.cov6), _dev.ptr(self.fstats), _dev.ptr(self.floor),
            _dev.ptr(self.loss[3:4]) if do_step else None, _dev.stream_ptr()), "field step")

    def _slice_step(self, step_mask: int, lr_scale: float, anchor: int = -1):
        o = self.optim_cfg
        lrs = (ctypes.c_double * 4)(o.lr_slice_rotation, o.lr_slice_translation, o.lr_log_sigma,
                                    o.lr_eta)
        b1, b2, eps, wd = self._adam()
        if step_mask & 1:
            self.slice_t += 1
        t = max(self.slice_t, 1)
        check(lib().gsvr_slice_adamw_step(
            self.S, _dev.ptr(self.sstate), _dev.ptr(self.sm), _dev.ptr(self.sv), _dev.ptr(self.dslice),
            _dev.ptr(self.b.stack_rots), _dev.ptr(self.b.s2t), _dev.ptr(self.psf_diags),
            _dev.ptr(self.b.counts), int(self.loss_cfg.outlier_weighting), lrs, lr_scale, b1, b2, eps,
            wd, 1.0 - b1 ** t, 1.0 - b2 ** t, int(step_mask), int(anchor), _dev.ptr(self.loss),
            _dev.ptr(self.Rc), _dev.ptr(self.tv), _dev.ptr(self.p6), _dev.ptr(self.sig),
            _dev.ptr(self.w), _dev.stream_ptr()), "slice step")

    # -- epoch -------------------------------------------------------------
    def check_floor(self):
        """train.py:162-169, raised before the epoch like the reference."""
        if self.floor_host != _NONE:
            j = int(self.floor_host)
            smin = float(np.exp(_dev.to_host(self.ls[j]).min()))
            raise NumericalDegeneracyError(
                f"primitive {j} scale {smin:.3e} mm collapsed below the eigenvalue floor")

    def refresh(self, K: int) -> None:
        from .knn import NeighborIndex, _build_handle
        index = NeighborIndex(np.empty((self.N, 3)), _build_handle(self.mu))
        self.b.refresh(index, K, self.Rc, self.tv)
        self.Rc_ref, self.t_ref = self.Rc.clone(), self.tv.clone()

    def train_pass(self, I_hat=None, absres=None) -> None:
        self.nonfinite.fill_(-1)
        check(lib().gsvr_train_tiles(
            self.b.raw, self.S, self.N, _dev.ptr(self.Rc), _dev.ptr(self.tv), _dev.ptr(self.p6),
            _dev.ptr(self.sig), _dev.ptr(self.w), _dev.ptr(self.mu), _dev.ptr(self.cov6),
            _dev.ptr(self.c), DELTA, _dev.ptr(self.dfield), _dev.ptr(self.dslice), _dev.ptr(I_hat),
            _dev.ptr(absres), _dev.ptr(self.nonfinite), _dev.stream_ptr()), "train pass")

    def epoch(self, lr_scale: float, slice_step: bool, freeze_rotations: bool,
              anchor: Optional[int], sync: bool = True) -> Optional[dict]:
        """One fwd+bwd + both AdamW steps.  Returns the loss terms at the
        pre-step parameters (train.py:466-479) when sync=True."""
        self.check_floor()
        self.train_pass()
        # the field-gradient all-reduce overlaps the rank-local slice step and
        # staleness pass; the field step waits for it
        pending = self.comm.allreduce_sum_async(self.dfield) if self.comm is not None else None
        mask = (1 if slice_step else 0) | (2 if freeze_rotations else 0)
        local_anchor = -1
        if anchor is not None:
            local_anchor = anchor - self.slice_offset
            if not 0 <= local_anchor < self.S:
                local_anchor = -1
        main = torch.cuda.current_stream()
        self._ev_train.record(main)
        self._side.wait_event(self._ev_train)
        with torch.cuda.stream(self._side):
            self._slice_step(mask, lr_scale, local_anchor)
            if self.Rc_ref is not None:
                check(lib().gsvr_batch_displacement(self.b.raw, _dev.ptr(self.Rc), _dev.ptr(self.tv),
                                                    _dev.ptr(self.Rc_ref), _dev.ptr(self.t_ref),
                                                    _dev.ptr(self.disp), _dev.stream_ptr()))
            self._ev_slice.record(self._side)
        if pending is not None:
            pending.wait()
        # (also moves the regulariser of the parameters the loss was evaluated
        # at, fstats, into loss[3] before overwriting it)
        self._field_kernel(True, lr_scale)
        main.wait_event(self._ev_slice)
        if not sync:
            return None
        return self.read_terms()

    def read_terms(self) -> dict:
        if self.comm is not None:
            self.comm.allreduce_sum(self.loss[:3])
            self.comm.allreduce_max(self.disp)
            # the flag holds a rank-local point index: reduce the GLOBAL slice id
            # of each rank's first non-finite point instead (train.py:155-159)
            nf = self.nonfinite
            hit = nf != -1
            key = self.b.sid.index_select(0, nf.clamp(min=0)).to(torch.int64) + self.slice_offset
            nf.copy_(torch.where(hit, key, nf))
            self.comm.allreduce_min_u64(self.nonfinite)
        self.host.copy_(self.status, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = self.host.numpy()
        self.floor_host = int(self.host_i[5]) & _NONE
        nf = int(self.host_i[6]) & _NONE
        if nf != _NONE:
            # sharded runs already reduced the global slice id (above)
            s = nf if self.comm is not None else int(self.b.sid[nf])
            raise TrainingDivergedError(f"non-finite rendered intensity on slice {s}")
        reg = self.loss_cfg.lambda_reg * float(h[3])
        data, outlier = float(h[0]), float(h[1])
        if not self.loss_cfg.outlier_weighting:
            outlier = 0.0
        self.displacement = float(h[4])
        return {"loss": data + outlier + reg, "data_term": data, "reg_term": reg,
                "outlier_term": outlier}

    # -- reseed (train.py:312-358) ----------------------------------------
    def reseed(self, n_gaussians: int, initial_scale: float, seed: int,
               mode: str, k_neighbors: int, take=None) -> None:
        P = self.total_points
        pos = self.b.corrected_points(self.Rc, self.tv)
        if take is None:  # train.py:338-341 (fit() prepares it on a host thread)
            rng = np.random.Generator(np.random.PCG64(seed))
            take = rng.choice(P, size=n_gaussians, replace=n_gaussians > P)
        sharded = self.comm is not None and self.comm.world > 1
        if sharded:  # rows owned by this rank, assembled by a sum over ranks
            from .parallel import owned_draws
            rows, local = owned_draws(take, self.point_offset, self.b.P)
            rows_d, tk = _dev.to_dev(rows, i64), _dev.to_dev(local, i64)
            new_mu = torch.zeros((n_gaussians, 3), dtype=torch.float64, device=pos.device)
            new_mu.index_copy_(0, rows_d, pos.index_select(0, tk))
            self.comm.allreduce_sum(new_mu)
        else:
            tk = _dev.to_dev(take, i64)
            new_mu = pos.index_select(0, tk).contiguous()
        ls = torch.full((n_gaussians, 3), math.log(initial_scale), dtype=torch.float64,
                        device=new_mu.device)
        q = torch.zeros((n_gaussians, 4), dtype=torch.float64, device=new_mu.device)
        q[:, 0] = 1.0
        if mode == "observed":
            if sharded:
                c = torch.zeros((n_gaussians,), dtype=torch.float64, device=pos.device)
                c.index_copy_(0, rows_d, self.b.I_obs.index_select(0, tk))
                self.comm.allreduce_sum(c)
            else:
                c = self.b.I_obs.index_select(0, tk).contiguous()
        else:
            from .knn import NeighborIndex, _build_handle, query_device
            index = NeighborIndex(np.empty((self.N, 3)), _build_handle(self.mu))
            nbr = query_device(index, new_mu, min(k_neighbors, self.N), out_i64=False)
            c = evaluate_field_device(new_mu, (self.mu, self.ls, self.q, self.c), nbr)
            if mode == "resample":
                nearest = nbr[:, 0].long()
                ls = self.ls.index_select(0, nearest).contiguous()
                q = self.q.index_select(0, nearest).contiguous()
        self.N = n_gaussians
        self.mu, self.ls, self.q, self.c = new_mu, ls, q, c.contiguous()
        lib().gsvr_batch_invalidate_seeds(self.b.raw)  # old lists bound nothing in the new field
        self._alloc_field_buffers()
        self.reset_optimizers()
        self._field_prep()
        self.sync_floor()
