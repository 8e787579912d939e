"""Host-side logic of device_setup.DevicePointBatch (CPU): the slice-sharded
view a multi-rank fit takes (parallel.shard_batch on the device arrays) and the
lazily fetched host arrays, checked against motion.build_point_batch /
parallel.shard_batch on the same acquisition with CPU tensors standing in for
the device ones."""
import numpy as np
import pytest
import torch


def _stacks(g):
    rng = np.random.default_rng(0)
    out = []
    for t, shape in enumerate([(9, 7, 4), (6, 8, 5)]):
        A = np.eye(4)
        A[:3, :3] = np.diag([0.8, 0.9, 2.5]) @ np.eye(3)[[t, (t + 1) % 3, (t + 2) % 3]]
        A[:3, 3] = rng.normal(size=3)
        mask = rng.random(shape) < 0.7
        mask[:, :, 1] = False  # an empty slice
        out.append(g.SliceStack(rng.random(shape), A, 0.8, 2.5, mask))
    return out


def _device_like(g, hb):
    from paper_2512_11624_b200.device_setup import DevicePointBatch
    return DevicePointBatch(torch.from_numpy(hb.lifted.copy()), torch.from_numpy(hb.slice_ids.copy()),
                            torch.from_numpy(hb.intensities.copy()), hb.slice_to_stack, hb.stack_rotations,
                            hb.slice_counts())


def test_host_arrays_match_point_batch():
    import paper_2512_11624_b200 as g
    hb = g.build_point_batch(_stacks(g))
    db = _device_like(g, hb)
    assert db.n_points == hb.n_points and db.n_slices == hb.n_slices
    assert np.array_equal(db.slice_counts(), hb.slice_counts())
    for name in ("lifted", "slice_ids", "stack_ids", "intensities"):
        assert np.array_equal(getattr(db, name), getattr(hb, name)), name


@pytest.mark.parametrize("world", [2, 3, 4])
def test_shard_matches_parallel_shard_batch(world):
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200.parallel import shard_batch
    hb = g.build_point_batch(_stacks(g))
    db = _device_like(g, hb)
    total = 0
    for rank in range(world):
        hs, hsl = shard_batch(hb, rank, world)
        ds, dsl = db.shard(rank, world)
        assert hsl == dsl
        assert ds.n_points == hs.n_points and ds.n_slices == hs.n_slices
        assert np.array_equal(ds.lifted, hs.lifted)
        assert np.array_equal(ds.slice_ids, hs.slice_ids)
        assert np.array_equal(ds.intensities, hs.intensities)
        assert np.array_equal(ds.slice_counts(), hs.slice_counts())
        total += ds.n_points
    assert total == hb.n_points
