"""Loss, analytic gradients and the fit loop -- the reference's train.py API on B200.

Public functions keep the reference's names, arguments, return structures and
errors (train.py:46-497).  Arrays in and out are numpy like the reference;
all per-pixel and per-primitive work runs in libgsvr_b200.so:

* ``backward``      -> tile binning + fused tile kernel + device chains
                       (train.py:220-302), one call = one drop-in epoch.
* ``render_batch`` / ``compute_loss`` -> float64 device forward (clamp semantics).
* ``fit``           -> engine.FitEngine, the device-resident epoch loop with the
                       reference's refresh / reseed / warm-up / anchor policy.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field as _field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _dev
from ._native import check, lib, last_index, last_value
from .engine import DeviceBatch, FitEngine, pick_tile_points
from .errors import InvalidParameterError, NumericalDegeneracyError, TrainingDivergedError
from .field import DELTA, GaussianField, rasterize
from .initialization import InitConfig
from .motion import PointBatch, SliceStack, SliceStates, init_states
from .optim import AdamWConfig, SchedulerConfig, lr_at
from .psf import PsfModel, build_psf
from .volume import VolumeGrid

FIELD_PARAM_NAMES = ("means", "log_scales", "quaternions", "intensities")
SLICE_PARAM_NAMES = ("slice_quaternions", "slice_translations", "log_sigma", "eta")
f64, i32 = np.float64, np.int32


@dataclass
class LossConfig:
    """train.py:46-59."""
    lambda_reg: float = 2.5e-3
    s_target: float = 1.6
    outlier_weighting: bool = False
    point_budget: int = 10_000_000

    def __post_init__(self):
        if self.lambda_reg < 0:
            raise InvalidParameterError("lambda_reg must be >= 0")
        if self.s_target <= 0:
            raise InvalidParameterError("s_target must be positive")
        if self.point_budget < 1:
            raise InvalidParameterError("point_budget must be positive")


@dataclass
class OptimConfig:
    """train.py:62-115."""
    epochs: int = 500
    lr_means: float = 2.5e-2
    lr_log_scales: float = 2.5e-2
    lr_quaternions: float = 1e-2
    lr_intensities: float = 1e-2
    lr_slice_rotation: float = 2.5e-3
    lr_slice_translation: float = 1e-1
    lr_log_sigma: float = 1e-2
    lr_eta: float = 1e-2
    scheduler: SchedulerConfig = _field(default_factory=SchedulerConfig)
    adamw: AdamWConfig = _field(default_factory=AdamWConfig)
    knn_refresh_every: int = 50
    k_neighbors: int = 50
    knn_staleness_mm: float = 0.5
    motion_warmup: int = 10
    rotation_warmup: int = 100
    reseed_every: int = 100
    reseed_mode: str = "resample"
    anchor_slice: Optional[int] = 0

    def __post_init__(self):
        rates = [self.lr_means, self.lr_log_scales, self.lr_quaternions, self.lr_intensities,
                 self.lr_slice_rotation, self.lr_slice_translation, self.lr_log_sigma, self.lr_eta]
        if any(r <= 0 for r in rates):
            raise InvalidParameterError("all learning rates must be positive")
        if self.epochs < 1:
            raise InvalidParameterError("epochs must be positive")
        if self.knn_refresh_every < 1 or self.k_neighbors < 1:
            raise InvalidParameterError("knn settings must be positive")
        if self.motion_warmup < 0 or self.rotation_warmup < 0:
            raise InvalidParameterError("warmups must be >= 0")
        if self.reseed_every < 0:
            raise InvalidParameterError("reseed_every must be >= 0")
        if self.reseed_mode not in ("resample", "render", "observed"):
            raise InvalidParameterError("reseed_mode must be resample, render or observed")
        if self.knn_staleness_mm < 0:
            raise InvalidParameterError("knn_staleness_mm must be >= 0")

    def field_lrs(self) -> Dict[str, float]:
        return {"means": self.lr_means, "log_scales": self.lr_log_scales,
                "quaternions": self.lr_quaternions, "intensities": self.lr_intensities}

    def slice_lrs(self) -> Dict[str, float]:
        return {"slice_quaternions": self.lr_slice_rotation,
                "slice_translations": self.lr_slice_translation,
                "log_sigma": self.lr_log_sigma, "eta": self.lr_eta}


def slice_psf_diags(batch: PointBatch, stacks: Sequence[SliceStack], use_psf: bool = True,
                    psf_models: Optional[Sequence[PsfModel]] = None) -> np.ndarray:
    """train.py:129-142: (S, 3) slice-frame PSF variances."""
    if psf_models is None:
        psf_models = [build_psf(s.inplane_spacing, s.thickness) for s in stacks]
    if isinstance(psf_models, PsfModel):
        psf_models = [psf_models] * len(stacks)
    if len(psf_models) != len(stacks):
        raise InvalidParameterError("need one PSF model per stack")
    per_stack = np.stack([m.sigmas ** 2 for m in psf_models])
    if not use_psf:
        per_stack = np.zeros_like(per_stack)
    return per_stack[batch.slice_to_stack]


# ---------------------------------------------------------------------------
# device helpers for one-shot calls

class _SliceInputs:
    """train.py:145-152 on the device: Rc, psf6s, sigma_s (+ wdata_s)."""

    def __init__(self, batch: PointBatch, states: SliceStates, psf_diags, outlier: bool):
        S = batch.n_slices
        if len(states) != S:
            raise InvalidParameterError("slice state count does not match stacks")
        self.q = _dev.to_dev(states.quaternions, f64)
        self.ls = _dev.to_dev(states.log_sigma, f64)
        self.stack_rots = _dev.to_dev(batch.stack_rotations, f64)
        self.s2t = _dev.to_dev(batch.slice_to_stack, i32)
        self.psf_diags = _dev.to_dev(np.asarray(psf_diags, dtype=f64), f64)
        self.Rc, self.p6, self.sig = (_dev.empty((S, 3, 3), f64), _dev.empty((S, 6), f64),
                                      _dev.empty((S,), f64))
        self.tv = _dev.to_dev(states.translations, f64)
        self.wdata_host = np.exp(-states.eta) if outlier else np.ones(S)
        self.w = _dev.to_dev(self.wdata_host, f64)
        check(lib().gsvr_slice_inputs(S, _dev.ptr(self.q), _dev.ptr(self.stack_rots), _dev.ptr(self.s2t),
                                      _dev.ptr(self.ls), _dev.ptr(self.psf_diags), _dev.ptr(self.Rc), 0,
                                      _dev.ptr(self.p6), _dev.ptr(self.sig), _dev.stream_ptr()))


def _field_dev(field: GaussianField):
    return tuple(_dev.to_dev(a, f64) for a in (field.means, field.log_scales, field.quaternions,
                                               field.intensities))


def _check_scale_floor(field: GaussianField) -> None:
    """train.py:162-169 (same message)."""
    smin = np.min(field.scales(), axis=1)
    bad = smin * smin < 1e-6
    if bad.any():
        j = int(np.flatnonzero(bad)[0])
        raise NumericalDegeneracyError(
            f"primitive {j} scale {float(smin[j]):.3e} mm collapsed below the eigenvalue floor")


def _check_finite_render(I_hat: np.ndarray, slice_ids: np.ndarray) -> None:
    """train.py:155-159."""
    bad = ~np.isfinite(I_hat)
    if bad.any():
        s = int(slice_ids[int(np.flatnonzero(bad)[0])])
        raise TrainingDivergedError(f"non-finite rendered intensity on slice {s}")


def _loss_terms(l1_per_slice, counts, log_scales_sumsq, eta, wdata_s, cfg: LossConfig) -> dict:
    """train.py:172-186 from device-reduced per-slice L1 sums."""
    data = float(wdata_s @ l1_per_slice)
    outlier = float(counts @ eta) if cfg.outlier_weighting else 0.0
    reg = cfg.lambda_reg * float(log_scales_sumsq)
    return {"loss": data + outlier + reg, "data_term": data, "reg_term": reg,
            "outlier_term": outlier}


def _reg_sumsq(field: GaussianField, s_target: float) -> float:
    ds = field.scales() - s_target
    return float(np.sum(ds * ds))


# ---------------------------------------------------------------------------

def render_batch(batch: PointBatch, field: GaussianField, states: SliceStates, psf_diags,
                 neighbor_ids, delta: float = DELTA) -> np.ndarray:
    """train.py:189-206: observed intensities of every batch point (float64, clamp)."""
    si = _SliceInputs(batch, states, psf_diags, False)
    mu, ls, q, c = _field_dev(field)
    N = field.count
    cov6 = _dev.empty((N, 6), f64)
    check(lib().gsvr_field_covariances(N, _dev.ptr(ls), _dev.ptr(q), _dev.ptr(cov6), 0,
                                       _dev.stream_ptr()))
    nbr = np.asarray(neighbor_ids)
    is64 = nbr.dtype == np.int64
    nd = _dev.to_dev(nbr, np.int64 if is64 else np.int32)
    x0 = _dev.to_dev(batch.lifted, f64)
    sid = _dev.to_dev(batch.slice_ids, i32)
    out = _dev.empty((batch.n_points,), f64)
    check(lib().gsvr_render_batch(batch.n_points, int(nbr.shape[1]), _dev.ptr(x0), _dev.ptr(sid),
                                  _dev.ptr(si.Rc), _dev.ptr(si.tv), _dev.ptr(si.p6), _dev.ptr(si.sig),
                                  _dev.ptr(nd), int(is64), N, _dev.ptr(mu), _dev.ptr(cov6), _dev.ptr(c),
                                  float(delta), _dev.ptr(out), _dev.stream_ptr()), "render_batch")
    I_hat = _dev.to_host(out)
    _check_finite_render(I_hat, batch.slice_ids)
    return I_hat


def compute_loss(batch: PointBatch, field: GaussianField, states: SliceStates, psf_diags,
                 cfg: LossConfig, neighbor_ids) -> Tuple[float, dict]:
    """train.py:209-217."""
    I_hat = render_batch(batch, field, states, psf_diags, neighbor_ids)
    absres = np.abs(I_hat - batch.intensities)
    S = batch.n_slices
    wdata_s = np.exp(-states.eta) if cfg.outlier_weighting else np.ones(S)
    l1 = np.bincount(batch.slice_ids, weights=absres, minlength=S)
    terms = _loss_terms(l1, batch.slice_counts(), _reg_sumsq(field, cfg.s_target), states.eta,
                        wdata_s, cfg)
    return terms["loss"], terms


def backward(batch: PointBatch, field: GaussianField, states: SliceStates, psf_diags,
             cfg: LossConfig, neighbor_ids,
             delta: float = DELTA) -> Tuple[dict, Dict[str, np.ndarray], np.ndarray]:
    """train.py:220-302: (terms, grads, I_hat) for all parameter classes.

    One call = point planning + (slice, tile) binning of ``neighbor_ids`` + the
    fused tile kernel + the device gradient chains.  Primitives outside every
    neighbour set receive exactly zero data gradient."""
    _check_scale_floor(field)
    P, S, N = batch.n_points, batch.n_slices, field.count
    si = _SliceInputs(batch, states, psf_diags, cfg.outlier_weighting)
    mu, ls, q, c = _field_dev(field)
    cov6 = _dev.empty((N, 6), f64)
    check(lib().gsvr_field_covariances(N, _dev.ptr(ls), _dev.ptr(q), _dev.ptr(cov6), 0,
                                       _dev.stream_ptr()))
    nbr = np.asarray(neighbor_ids)
    db = DeviceBatch(batch, K=int(nbr.shape[1]))
    db.bin(nbr, N)
    dfield = _dev.zeros((N, 10), np.float32)
    dslice = _dev.zeros((S, 20), f64)
    I_hat = _dev.empty((P,), f64)
    nonfinite = _dev.empty((1,), np.int64)
    nonfinite.fill_(-1)
    check(lib().gsvr_train_tiles(db.raw, S, N, _dev.ptr(si.Rc), _dev.ptr(si.tv), _dev.ptr(si.p6),
                                 _dev.ptr(si.sig), _dev.ptr(si.w), _dev.ptr(mu), _dev.ptr(cov6),
                                 _dev.ptr(c), float(delta), _dev.ptr(dfield), _dev.ptr(dslice),
                                 _dev.ptr(I_hat), 0, _dev.ptr(nonfinite), _dev.stream_ptr()), "backward")
    # covariance chain (train.py:271-282) and slice chain (train.py:284-290)
    dcov6 = dfield[:, 3:9].double().contiguous()
    dls, dq = _dev.empty((N, 3), f64), _dev.empty((N, 4), f64)
    check(lib().gsvr_field_chain(N, _dev.ptr(ls), _dev.ptr(q), _dev.ptr(dcov6), cfg.lambda_reg,
                                 cfg.s_target, _dev.ptr(dls), _dev.ptr(dq), _dev.stream_ptr()))
    dRc = dslice[:, 3:12].contiguous()
    dp6 = dslice[:, 12:18].contiguous()
    dsg = dslice[:, 18].contiguous()
    dqi, dlsig = _dev.empty((S, 4), f64), _dev.empty((S,), f64)
    check(lib().gsvr_slice_chain(S, _dev.ptr(si.q), _dev.ptr(si.stack_rots), _dev.ptr(si.s2t),
                                 _dev.ptr(si.ls), _dev.ptr(si.psf_diags), _dev.ptr(dRc), _dev.ptr(dp6),
                                 _dev.ptr(dsg), _dev.ptr(dqi), _dev.ptr(dlsig), _dev.stream_ptr()))
    I_host = _dev.to_host(I_hat)
    _check_finite_render(I_host, batch.slice_ids)
    dslice_h = _dev.to_host(dslice)
    dfield_h = _dev.to_host(dfield).astype(f64)
    counts = batch.slice_counts()
    l1 = dslice_h[:, 19]
    if cfg.outlier_weighting:
        deta = -si.wdata_host * l1 + counts
    else:
        deta = np.zeros(S)
    terms = _loss_terms(l1, counts, _reg_sumsq(field, cfg.s_target), states.eta, si.wdata_host, cfg)
    grads = {"means": np.ascontiguousarray(dfield_h[:, 0:3]), "log_scales": _dev.to_host(dls),
             "quaternions": _dev.to_host(dq), "intensities": np.ascontiguousarray(dfield_h[:, 9]),
             "slice_quaternions": _dev.to_host(dqi),
             "slice_translations": np.ascontiguousarray(dslice_h[:, 0:3]),
             "log_sigma": _dev.to_host(dlsig), "eta": deta}
    return terms, grads, I_host


def corrected_points(batch: PointBatch, states: SliceStates) -> np.ndarray:
    """train.py:305-309 (device, einsum evaluation order)."""
    si = _SliceInputs(batch, states, np.zeros((batch.n_slices, 3)), False)
    x0 = _dev.to_dev(batch.lifted, f64)
    sid = _dev.to_dev(batch.slice_ids, i32)
    out = _dev.empty((batch.n_points, 3), f64)
    check(lib().gsvr_corrected_points(batch.n_points, _dev.ptr(x0), _dev.ptr(sid), _dev.ptr(si.Rc),
                                      _dev.ptr(si.tv), _dev.ptr(out), _dev.stream_ptr()))
    return _dev.to_host(out)


def reseed_draw(seed: int, n_points: int, n_gaussians: int) -> np.ndarray:
    """train.py:338-341: the reseed's point indices (reference RNG stream)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.choice(n_points, size=n_gaussians, replace=n_gaussians > n_points)


def reseed_field(batch: PointBatch, states: SliceStates, n_gaussians: int, initial_scale: float,
                 seed: int, source_field: Optional[GaussianField] = None, k_neighbors: int = 50,
                 mode: str = "resample") -> GaussianField:
    """train.py:312-358 (host RNG stream identical to the reference)."""
    from .field import evaluate_field
    from .knn import build_index, query

    if mode not in ("resample", "render", "observed"):
        raise InvalidParameterError(f"unknown reseed mode {mode!r}")
    if mode != "observed" and source_field is None:
        raise InvalidParameterError(f"reseed mode {mode!r} needs a source field")
    pos = corrected_points(batch, states)
    rng = np.random.Generator(np.random.PCG64(seed))
    take = rng.choice(batch.n_points, size=n_gaussians, replace=n_gaussians > batch.n_points)
    log_scales = np.full((n_gaussians, 3), np.log(initial_scale))
    quats = np.zeros((n_gaussians, 4))
    quats[:, 0] = 1.0
    if mode == "observed":
        intensities = batch.intensities[take].astype(np.float64)
    else:
        nbr = query(build_index(source_field.means), pos[take], min(k_neighbors, source_field.count))
        intensities = evaluate_field(pos[take], source_field, nbr)
        if mode == "resample":
            log_scales = source_field.log_scales[nbr[:, 0]].copy()
            quats = source_field.quaternions[nbr[:, 0]].copy()
    return GaussianField(pos[take].copy(), log_scales, quats, intensities)


@dataclass
class TrainState:
    """Run-time bookkeeping of ``fit`` (train.py:118-126); the optimiser moments
    and neighbour lists live on the device inside ``engine``."""
    engine: FitEngine
    epoch: int
    history: List[dict] = _field(default_factory=list)


def _evaluate(field: GaussianField, reference: VolumeGrid, K: int, states=None, truth_states=None):
    from .metrics import motion_gauge, psnr, ssim
    transform = None
    if states is not None and truth_states is not None:
        transform = motion_gauge(states, truth_states)
    recon = rasterize(field, reference, K=K, transform=transform)
    return (psnr(recon.data, reference.data, mask=reference.mask),
            ssim(recon.data, reference.data, mask=reference.mask))


def fit(stacks: Sequence[SliceStack], init_cfg: Optional[InitConfig] = None,
        loss_cfg: Optional[LossConfig] = None, optim_cfg: Optional[OptimConfig] = None, *,
        field: Optional[GaussianField] = None, states: Optional[SliceStates] = None,
        use_psf: bool = True, psf_models: Optional[Sequence[PsfModel]] = None,
        reference: Optional[VolumeGrid] = None, truth_states: Optional[SliceStates] = None,
        eval_every: int = 0, verbose: bool = False,
        comm=None) -> Tuple[GaussianField, SliceStates, List[dict]]:
    """train.py:373-497 with the state resident on the device.

    Same policy as the reference: refresh every ``knn_refresh_every`` epochs,
    on staleness > ``knn_staleness_mm`` and after every reseed; reseed every
    ``reseed_every`` epochs except in the last two segments; LR schedule per
    segment; slice states frozen for ``motion_warmup`` epochs of each segment,
    rotations until ``rotation_warmup``; anchor slice frozen.  ``comm`` (see
    parallel.py) shards the slices over ranks with the field replicated."""
    if len(stacks) == 0:
        raise InvalidParameterError("need at least one stack")
    init_cfg = init_cfg or InitConfig()
    loss_cfg = loss_cfg or LossConfig()
    optim_cfg = optim_cfg or OptimConfig()
    # the point batch and the content-adaptive initial field are built on the
    # device from the stack rasters (device_setup.py, csrc/init.cu), bit-identical
    # to build_point_batch / sample_init_positions / init_field
    from .device_setup import DeviceStacks, device_init_field, device_point_batch
    dstacks = DeviceStacks(stacks)
    batch = device_point_batch(dstacks)
    if field is None:
        field = device_init_field(dstacks, init_cfg)
    del dstacks
    field = field.astype(np.float64)
    states = states.copy() if states is not None else init_states(stacks)
    if len(states) != batch.n_slices:
        raise InvalidParameterError("slice state count does not match stacks")
    psf_diags = slice_psf_diags(batch, stacks, use_psf, psf_models)

    slice_offset, point_offset = 0, 0
    run_batch, run_states, run_psf = batch, states, psf_diags
    if comm is not None and comm.world > 1:
        run_batch, sl = batch.shard(comm.rank, comm.world)
        slice_offset = sl.start
        point_offset = int(batch.slice_counts()[:sl.start].sum())  # slice-contiguous
        run_states = SliceStates(states.quaternions[sl], states.translations[sl],
                                 states.log_sigma[sl], states.eta[sl])
        run_psf = psf_diags[sl]
    K = optim_cfg.k_neighbors
    dbatch = DeviceBatch(run_batch, K=K, tile_points=pick_tile_points(K))
    eng = FitEngine(dbatch, field, run_states, run_psf, loss_cfg, optim_cfg, comm=comm,
                    slice_offset=slice_offset, point_offset=point_offset, total_points=batch.n_points)
    state = TrainState(engine=eng, epoch=0)

    t_start = time.perf_counter()
    segment_start = 0
    refreshed = False
    # the reseed draws depend only on (seed + epoch, P, N): made on a host thread
    # while the GPU trains (the reference's RNG calls, train.py:338-341)
    reseed_epochs = [e for e in range(1, optim_cfg.epochs)
                     if optim_cfg.reseed_every > 0 and e % optim_cfg.reseed_every == 0
                     and e <= optim_cfg.epochs - 2 * optim_cfg.reseed_every]
    draws = {}
    pool = None
    if reseed_epochs:
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(max_workers=1)
        P_all = batch.n_points
        draws = {e: pool.submit(reseed_draw, init_cfg.seed + e, P_all, field.count) for e in reseed_epochs}
    for epoch in range(optim_cfg.epochs):
        state.epoch = epoch
        reseeded = False
        if epoch in draws:
            if optim_cfg.reseed_mode != "observed":
                # 'render' / 'resample' read the old field (evaluate_field's
                # floor check, field.py:114); 'observed' never looks at it
                eng.check_floor()
            eng.reseed(field.count, init_cfg.initial_scale,
                       init_cfg.seed + epoch, optim_cfg.reseed_mode, optim_cfg.k_neighbors,
                       take=draws.pop(epoch).result())
            segment_start = epoch
            reseeded = True
        seg_epoch = epoch - segment_start
        stale = (refreshed and optim_cfg.knn_staleness_mm > 0
                 and eng.displacement > optim_cfg.knn_staleness_mm ** 2)
        if reseeded or stale or epoch % optim_cfg.knn_refresh_every == 0:
            eng.refresh(K)
            refreshed = True
        scale = lr_at(seg_epoch, 1.0, optim_cfg.scheduler)
        step_slices = seg_epoch >= optim_cfg.motion_warmup and epoch >= optim_cfg.motion_warmup
        terms = eng.epoch(scale, step_slices, epoch < optim_cfg.rotation_warmup,
                          optim_cfg.anchor_slice)
        if not np.isfinite(terms["loss"]):
            raise TrainingDivergedError(f"loss diverged at epoch {epoch}")
        record = dict(terms)
        record.update(epoch=epoch, lr_scale=scale, reseeded=reseeded,
                      seconds=time.perf_counter() - t_start, psnr=None, ssim=None)
        if reference is not None and eval_every > 0 and (epoch + 1) % eval_every == 0:
            ev_states = eng.states_host()
            if comm is not None and comm.world > 1:  # truth_states covers every slice
                ev_states = comm.gather_states(ev_states, batch.n_slices, slice_offset)
            record["psnr"], record["ssim"] = _evaluate(eng.field_host(), reference, K,
                                                       ev_states, truth_states)
        state.history.append(record)
        if verbose and (epoch % 50 == 0 or epoch == optim_cfg.epochs - 1):
            extra = ""
            if record["psnr"] is not None:
                extra = f"  psnr={record['psnr']:.2f}  ssim={record['ssim']:.4f}"
            print(f"epoch {epoch:4d}  loss={terms['loss']:.6e}  lr_scale={scale:.4f}{extra}",
                  flush=True)
    if pool is not None:
        pool.shutdown(wait=False, cancel_futures=True)
    out_states = eng.states_host()
    if comm is not None and comm.world > 1:
        out_states = comm.gather_states(out_states, batch.n_slices, slice_offset)
    return eng.field_host(), out_states, state.history
