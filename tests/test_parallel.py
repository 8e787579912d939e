"""Slice-sharded data parallelism (paper_2512_11624_b200/parallel.py) on CPU.

world_size 2 over gloo (127.0.0.1): every rank computes the reference gradient
of its own slice shard with the oracle (the checker), the field gradient is
summed with Comm.allreduce_sum exactly as FitEngine does on NCCL, and the
result must equal the full-batch gradient; slice gradients stay rank-local.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden, loss_kwargs


def test_partition_balances_pixels():
    from paper_2512_11624_b200.parallel import partition_slices
    counts = np.array([10, 400, 400, 10, 300, 300, 5, 5, 500, 70])
    for world in (1, 2, 3, 4, 8):
        b = partition_slices(counts, world)
        assert b[0] == 0 and b[-1] == len(counts) and np.all(np.diff(b) >= 0)
        loads = [counts[b[r]:b[r + 1]].sum() for r in range(world)]
        assert sum(loads) == counts.sum()
        if world <= len(counts):
            assert max(loads) - counts.sum() / world <= counts.max()


def test_shard_batch_is_a_partition():
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200.parallel import shard_batch
    d = load_golden("train_medium_s0")
    batch = g.PointBatch(d["lifted"], d["slice_ids"].astype(np.int32), d["slice_ids"] * 0,
                         d["intensities_obs"], d["slice_to_stack"], d["stack_rotations"])
    seen = 0
    for r in range(3):
        sub, sl = shard_batch(batch, r, 3)
        keep = (batch.slice_ids >= sl.start) & (batch.slice_ids < sl.stop)
        np.testing.assert_array_equal(sub.lifted, batch.lifted[keep])
        np.testing.assert_array_equal(sub.slice_ids + sl.start, batch.slice_ids[keep])
        seen += sub.n_points
    assert seen == batch.n_points


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import host as oracle
        from paper_2512_11624_b200.parallel import Comm, partition_slices
        comm = Comm()
        d = load_golden("train_medium_s1")
        kw = loss_kwargs(d)
        counts = np.bincount(d["slice_ids"], minlength=len(d["slice_to_stack"]))
        b = partition_slices(counts, world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        keep = (d["slice_ids"] >= lo) & (d["slice_ids"] < hi)
        shard = dict(d)
        for k in ("lifted", "intensities_obs", "nbr"):
            shard[k] = d[k][keep]
        shard["slice_ids"] = (d["slice_ids"][keep] - lo).astype(np.int32)
        for k in ("slice_to_stack", "slice_quaternions", "slice_translations", "log_sigma", "eta",
                  "psf_diags"):
            shard[k] = d[k][lo:hi]
        # per-shard data gradient (no regulariser: it is added once, not per rank)
        terms, grads, _ = oracle.backward(shard, **dict(kw, lambda_reg=0.0))
        field = torch.from_numpy(np.concatenate([grads["means"], grads["intensities"][:, None]], 1))
        comm.allreduce_sum(field)
        loss = torch.tensor([terms["data_term"], terms["outlier_term"]], dtype=torch.float64)
        comm.allreduce_sum(loss)
        flag = torch.tensor([-1 if rank == 0 else 7], dtype=torch.int64)
        comm.allreduce_min_u64(flag)
        disp = torch.tensor([float(rank + 1)], dtype=torch.float64)
        comm.allreduce_max(disp)
        from paper_2512_11624_b200.motion import SliceStates
        local = SliceStates(d["slice_quaternions"][lo:hi] * (1 + rank), d["slice_translations"][lo:hi],
                            d["log_sigma"][lo:hi], d["eta"][lo:hi])
        full = comm.gather_states(local, len(d["slice_to_stack"]), lo)
        q.put((rank, field.numpy(), loss.numpy(), int(flag.item()), float(disp.item()),
               grads["slice_translations"], (lo, hi), full.quaternions))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gradient_allreduce_matches_full_batch(oracle):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    d = load_golden("train_medium_s1")
    kw = loss_kwargs(d)
    terms, grads, _ = oracle.backward(d, **dict(kw, lambda_reg=0.0))
    want = np.concatenate([grads["means"], grads["intensities"][:, None]], 1)
    for r in res:
        np.testing.assert_allclose(r[1], want, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(r[2], [terms["data_term"], terms["outlier_term"]], rtol=1e-12)
        assert r[3] == 7 and r[4] == 2.0
        lo, hi = r[6]
        np.testing.assert_allclose(r[5], grads["slice_translations"][lo:hi], rtol=1e-10, atol=1e-13)
        # gathered states: each rank's slice range filled by its owner
        np.testing.assert_allclose(r[7][:res[1][6][0]], d["slice_quaternions"][:res[1][6][0]])
        np.testing.assert_allclose(r[7][res[1][6][0]:], 2 * d["slice_quaternions"][res[1][6][0]:])


def _reseed_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_11624_b200.parallel import Comm, owned_draws, partition_slices
        comm = Comm()
        rng = np.random.default_rng(4)
        counts = rng.integers(0, 40, size=13)
        sid = np.repeat(np.arange(13), counts)
        pts = rng.normal(size=(len(sid), 3))
        b = partition_slices(counts, world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        p_off = int(np.count_nonzero(sid < lo))
        local = pts[(sid >= lo) & (sid < hi)]
        take = np.random.Generator(np.random.PCG64(9)).choice(len(pts), size=300, replace=True)
        rows, idx = owned_draws(take, p_off, len(local))
        out = torch.zeros((300, 3), dtype=torch.float64)
        out[torch.from_numpy(rows)] = torch.from_numpy(local[idx])
        comm.allreduce_sum(out)
        q.put((rank, out.numpy(), pts[take]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_reseed_assembly_is_exact():
    """Sharded reseed (train.py:338-358): the global draw assembled from the
    owners' rows by a sum over ranks equals the single-rank gather bit for bit."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reseed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for _, got, want in res:
        np.testing.assert_array_equal(got, want)
