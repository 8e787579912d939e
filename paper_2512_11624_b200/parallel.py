"""Slice-sharded data parallelism, one process per GPU.

Pixels are independent given the field and the loss is a sum over pixels, so
the point batch is split into contiguous slice ranges balanced by pixel count
(points are slice-contiguous, motion.py:214-227).  Each rank owns its slices'
states and AdamW moments (no communication for them); the Gaussian field is
replicated, its fp32 (N, 10) gradient buffer is all-reduced once per epoch,
and every rank then runs the identical field chain + AdamW so the replicas
stay bit-identical.  Loss terms (sum), staleness (max) and the non-finite flag
(min) are reduced as scalars.  The backend is NCCL over NVLink on GPUs; the
host logic is exercised with gloo on CPU in tests/test_parallel.py.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np
import torch
import torch.distributed as dist

from .motion import PointBatch, SliceStates

_I64_MAX = (1 << 63) - 1


def partition_slices(counts: np.ndarray, world: int) -> np.ndarray:
    """Boundaries b[0..world] of contiguous slice ranges with ~equal pixel counts.

    Rank r owns slices [b[r], b[r+1]).  Greedy on the cumulative pixel count so
    every rank's share is within one slice of P / world."""
    counts = np.asarray(counts, dtype=np.int64)
    S = len(counts)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        # pick the closer of the two candidate cuts, keep ranges monotone
        if b > 0 and abs(cum[b - 1] - target) <= abs(cum[min(b, S)] - target):
            b -= 1
        bounds.append(min(max(b, bounds[-1]), S))
    bounds.append(S)
    return np.asarray(bounds, dtype=np.int64)


def shard_batch(batch: PointBatch, rank: int, world: int) -> Tuple[PointBatch, slice]:
    """This rank's sub-batch (slice ids renumbered from 0) and its global slice range."""
    b = partition_slices(batch.slice_counts(), world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    keep = (batch.slice_ids >= lo) & (batch.slice_ids < hi)
    sub = PointBatch(batch.lifted[keep], (batch.slice_ids[keep] - lo).astype(np.int32),
                     batch.stack_ids[keep], batch.intensities[keep],
                     batch.slice_to_stack[lo:hi], batch.stack_rotations)
    return sub, slice(lo, hi)


def owned_draws(take: np.ndarray, p_offset: int, p_local: int):
    """Reseed on a sharded run (train.py:338-358): every rank draws the same
    global point indices with the reference RNG; the rows whose point this rank
    owns (points are slice-contiguous, rank r holds [p_offset, p_offset+p_local))
    and their local indices.  Each row has exactly one owner, so a zero-filled
    buffer summed over ranks assembles the draw exactly (x + 0 = x)."""
    take = np.asarray(take, dtype=np.int64)
    rows = np.flatnonzero((take >= p_offset) & (take < p_offset + p_local))
    return rows, take[rows] - p_offset


class Comm:
    """Thin torch.distributed wrapper used by engine.FitEngine (any backend)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def _run(self, t: torch.Tensor, op) -> None:
        # NCCL reduces device tensors in place; gloo (CPU tests, single-GPU
        # multi-rank smoke runs) stages CUDA tensors through the host
        if t.is_cuda and dist.get_backend(self.group) != "nccl":
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)

    def allreduce_sum(self, t: torch.Tensor) -> None:
        if self.world > 1:
            self._run(t, dist.ReduceOp.SUM)

    def allreduce_sum_async(self, t: torch.Tensor):
        """Start a sum all-reduce; returns an object whose wait() orders the
        current stream after it.  NCCL runs it on its own stream, so work
        issued in between (the slice step) overlaps the transfer; other
        backends complete it here."""
        class _Done:
            def wait(self):
                return None
        if self.world > 1 and t.is_cuda and dist.get_backend(self.group) == "nccl":
            return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.allreduce_sum(t)
        return _Done()

    def allreduce_max(self, t: torch.Tensor) -> None:
        if self.world > 1:
            self._run(t, dist.ReduceOp.MAX)

    def allreduce_min_u64(self, t: torch.Tensor) -> None:
        """Min of device atomicMin flags whose 'none' value is all-ones (-1 as int64)."""
        if self.world > 1:
            t.masked_fill_(t == -1, _I64_MAX)
            self._run(t, dist.ReduceOp.MIN)
            t.masked_fill_(t == _I64_MAX, -1)

    def broadcast(self, t: torch.Tensor, src: int = 0) -> None:
        if self.world > 1:
            if t.is_cuda and dist.get_backend(self.group) != "nccl":
                h = t.cpu()
                dist.broadcast(h, src=src, group=self.group)
                t.copy_(h)
            else:
                dist.broadcast(t, src=src, group=self.group)

    def barrier(self) -> None:
        if self.world > 1:
            dist.barrier(group=self.group)

    def gather_states(self, local: SliceStates, n_slices: int, offset: int) -> SliceStates:
        """All ranks' slice states assembled in global slice order."""
        st = np.concatenate([local.quaternions, local.translations, local.log_sigma[:, None],
                             local.eta[:, None]], axis=1)
        full = np.zeros((n_slices, 9))
        full[offset:offset + len(st)] = st
        if self.world > 1:
            dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
            t = torch.from_numpy(full).to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            full = t.cpu().numpy()
        return SliceStates(full[:, 0:4], full[:, 4:7], full[:, 7], full[:, 8])
