"""The fit's setup on the device (csrc/init.cu via device_setup.py) against the
reference and against numpy on this host, bit for bit:

* the point batch and the initial field reproduce the reference's SHA-256
  goldens (tests/golden/host_cases.json, the reference's own
  build_point_batch / sample_init_positions / init_field);
* on other acquisitions -- the reference simulator's desk stacks (oblique
  affines), random masks with single-pixel slices and empty slices, 2-pixel
  edges, float32 data, tiny and huge intensities, draws small enough that most
  (stack, slice) groups hold one pixel (OpenBLAS's gemv order), the 'mean'
  policy, lambda_init > 0, the zero-mass fallback -- device == host numpy;
* the building blocks alone: the weights (np.gradient + glibc hypot), numpy's
  pairwise sum and cumsum over sizes around every block boundary;
* cfg3 at full size (24.6 M pixels, 500k draws), with the setup times printed.
"""
import ctypes
import time
import warnings

import numpy as np
import pytest

from conftest import GOLDEN
from test_host_golden import CASES, digest, load_stacks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    assert torch.cuda.is_available()
    import paper_2512_11624_b200 as pkg
    return pkg


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint8)


def _same(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(_bits(a), _bits(b))


def _device_batch(g, stacks):
    from paper_2512_11624_b200.device_setup import DeviceStacks, device_point_batch
    return device_point_batch(DeviceStacks(stacks))


def _device_field(g, stacks, cfg):
    from paper_2512_11624_b200.device_setup import DeviceStacks, device_init_field
    return device_init_field(DeviceStacks(stacks), cfg)


@pytest.mark.parametrize("name", sorted(CASES["batches"]))
def test_device_batch_reproduces_reference_sha(g, name):
    ref = CASES["batches"][name]
    b = _device_batch(g, load_stacks(g, name))
    assert b.n_points == ref["n_points"]
    assert digest(b.lifted) == ref["lifted"]
    assert digest(b.slice_ids) == ref["slice_ids"]
    assert digest(b.intensities) == ref["intensities"]


@pytest.mark.parametrize("case", CASES["inits"], ids=lambda c: f"{c['data']}-n{c['n_gaussians']}-s{c['seed']}")
def test_device_init_reproduces_reference_sha(g, case):
    stacks = load_stacks(g, case["data"])
    cfg = g.InitConfig(n_gaussians=case["n_gaussians"], lambda_init=case["lambda_init"], seed=case["seed"],
                       initial_scale=case["initial_scale"], intensity_policy=case["intensity_policy"])
    f = _device_field(g, stacks, cfg)
    assert digest(f.means) == case["positions"]
    assert digest(f.intensities) == case["intensities"]
    assert digest(f.log_scales) == case["log_scales"]


def _desk_stacks(g, tag="desk_motion"):
    z = dict(np.load(GOLDEN / f"{tag}_data.npz"))
    n = sum(1 for k in z if k.endswith("_affine") and k.startswith("s"))
    return [g.SliceStack(z[f"s{i}_data"], z[f"s{i}_affine"], z[f"s{i}_spacing"], float(z[f"s{i}_thickness"]),
                         z[f"s{i}_mask"]) for i in range(n)]


def _odd_stacks(g, seed=0, dtype=np.float64, scale=1.0):
    """Random oblique affines, sparse masks with a single-pixel slice and an
    empty slice, a 2-pixel axis, wide value ranges."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(seed)
    out = []
    for t, shape in enumerate([(37, 29, 7), (2, 41, 5), (23, 2, 4), (31, 33, 9)]):
        A = np.eye(4)
        A[:3, :3] = Rotation.random(random_state=seed * 10 + t).as_matrix() @ np.diag(
            rng.uniform(0.4, 1.3, 3)) * np.array([1.0, 1.0, 2.5])
        A[:3, 3] = rng.normal(size=3) * 40
        data = (rng.normal(size=shape) * scale * 10.0 ** rng.integers(-3, 3, size=shape)).astype(dtype)
        mask = rng.random(shape) < 0.6
        mask[:, :, 0] = False                       # empty slice
        mask[:, :, 1] = False
        mask[rng.integers(shape[0]), rng.integers(shape[1]), 1] = True  # single-pixel slice
        out.append(g.SliceStack(data, A, np.array([0.8, 0.9]), 2.0, mask))
    return out


CASES_EXTRA = [("desk", 5000, 0.0, "source", 0), ("desk", 37, 0.0, "source", 4), ("desk", 20000, 0.25, "mean", 1),
               ("odd", 300, 0.0, "source", 0), ("odd", 5, 0.5, "source", 2), ("odd32", 800, 0.1, "mean", 3),
               ("tiny", 400, 0.0, "source", 5), ("huge", 400, 0.0, "source", 6)]


def _extra_stacks(g, kind):
    if kind == "desk":
        return _desk_stacks(g)
    if kind == "odd":
        return _odd_stacks(g, 0)
    if kind == "odd32":
        return _odd_stacks(g, 1, np.float32)
    if kind == "tiny":
        return _odd_stacks(g, 2, scale=1e-160)   # glibc hypot's tiny-input scaling
    return _odd_stacks(g, 3, scale=1e200)        # ... and its large-input scaling


@pytest.mark.parametrize("case", CASES_EXTRA, ids=lambda c: f"{c[0]}-n{c[1]}-l{c[2]}-{c[3]}-s{c[4]}")
def test_device_setup_matches_host_numpy(g, case):
    kind, n, lam, policy, seed = case
    stacks = _extra_stacks(g, kind)
    hb, db = g.build_point_batch(stacks), _device_batch(g, stacks)
    assert _same(db.lifted, hb.lifted)
    assert _same(db.slice_ids, hb.slice_ids)
    assert _same(db.stack_ids, hb.stack_ids)
    assert _same(db.intensities, hb.intensities)
    assert np.array_equal(db.slice_counts(), hb.slice_counts())
    cfg = g.InitConfig(n_gaussians=n, lambda_init=lam, seed=seed, intensity_policy=policy)
    pos = g.sample_init_positions(stacks, cfg)
    hf = g.init_field(pos, stacks, cfg)
    df = _device_field(g, stacks, cfg)
    assert _same(df.means, hf.means)
    assert _same(df.intensities, hf.intensities)
    assert _same(df.log_scales, hf.log_scales)
    assert _same(df.quaternions, hf.quaternions)


def test_weights_match_numpy(g):
    """np.gradient + glibc hypot per pixel, including the tiny / huge scaling
    branches and exact zeros."""
    from paper_2512_11624_b200 import _dev, initialization as ini
    from paper_2512_11624_b200._native import check, lib
    from paper_2512_11624_b200.device_setup import DeviceStacks
    for stacks, lam in [(_desk_stacks(g), 0.0), (_odd_stacks(g, 0), 0.3), (_odd_stacks(g, 2, scale=1e-160), 0.0),
                        (_odd_stacks(g, 3, scale=1e200), 0.0), (load_stacks(g, "cfg1_noisy_data.npz"), 0.0)]:
        want = (1.0 - lam) * np.concatenate([ini.gradient_magnitude(s)[s.mask] for s in stacks]) + lam
        ds = DeviceStacks(stacks)
        w = _dev.empty((want.size,), np.float64)
        check(lib().gsvr_init_weights(len(stacks), ds.views, ds.counts.ctypes.data_as(ctypes.c_void_p), lam,
                                      _dev.ptr(w), _dev.stream_ptr()))
        got = _dev.to_host(w)
        bad = np.flatnonzero(_bits(got) != _bits(want))
        assert bad.size == 0, (bad.size, got[bad[:3]], want[bad[:3]])


def _randn_wide(rng, n):
    return np.abs(rng.normal(size=n)) * 10.0 ** rng.integers(-8, 8, size=n)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 127, 128, 129, 136, 143, 144, 1000, 8192, 8193, 65537, 1_000_003,
                               24_576_000])
def test_pairwise_sum_matches_numpy(g, n):
    from paper_2512_11624_b200 import _dev
    from paper_2512_11624_b200._native import check, lib
    rng = np.random.default_rng(n)
    for x in (rng.random(n), _randn_wide(rng, n), rng.normal(size=n)):
        out = ctypes.c_double(0.0)
        t = _dev.to_dev(x, np.float64)
        check(lib().gsvr_pairwise_sum(n, _dev.ptr(t), ctypes.byref(out), _dev.stream_ptr()))
        assert _bits(np.array([out.value]))[0] == _bits(np.array([x.sum()]))[0], (n, out.value, x.sum())


@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2048, 2049, 4097, 16383, 16384, 16385, 1_000_001, 24_576_000])
def test_cumsum_matches_numpy(g, n):
    import torch
    from paper_2512_11624_b200 import _dev
    from paper_2512_11624_b200._native import check, lib
    rng = np.random.default_rng(n + 1)
    x = _randn_wide(rng, n) if n % 2 else rng.random(n) / n
    t = _dev.to_dev(x, np.float64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(lib().gsvr_cumsum(n, _dev.ptr(t), _dev.stream_ptr()))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    got, want = _dev.to_host(t), np.cumsum(x)
    bad = np.flatnonzero(_bits(got) != _bits(want))
    if n >= 1_000_000:
        print(f"cumsum chain n={n}: {dt * 1e3:.1f} ms on the device ({dt / n * 1e9:.2f} ns / element)")
    assert bad.size == 0, (bad.size, bad[:5])


def test_zero_mass_falls_back_to_uniform(g):
    stacks = [g.SliceStack(np.full((9, 8, 3), 2.5), np.diag([0.8, 0.8, 3.0, 1.0]), 0.8, 3.0)]
    cfg = g.InitConfig(n_gaussians=50, seed=3)
    with pytest.warns(UserWarning, match="zero sampling mass"):
        pos = g.sample_init_positions(stacks, cfg)
    with pytest.warns(UserWarning, match="zero sampling mass"):
        df = _device_field(g, stacks, cfg)
    assert _same(df.means, pos)


def test_setup_errors_match_host(g):
    st = g.SliceStack(np.ones((5, 5, 2)), np.eye(4), 1.0, 1.0, np.zeros((5, 5, 2), bool))
    with pytest.raises(g.InvalidParameterError, match="no masked pixels"):
        _device_batch(g, [st])
    with pytest.raises(g.InvalidParameterError, match="no masked pixels to sample from"):
        _device_field(g, [st], g.InitConfig(n_gaussians=4))
    thin = g.SliceStack(np.random.default_rng(0).random((1, 6, 3)), np.eye(4), 1.0, 1.0)
    with pytest.raises(ValueError, match="too small to calculate a numerical gradient"):
        g.sample_init_positions([thin], g.InitConfig(n_gaussians=4))
    with pytest.raises(ValueError, match="too small to calculate a numerical gradient"):
        _device_field(g, [thin], g.InitConfig(n_gaussians=4))


@pytest.mark.timeout(900)
def test_cfg3_setup_full_size(g):
    """cfg3 (6 stacks 320x320x40, 500k draws): device batch + initial field ==
    host numpy, and the setup times."""
    import torch
    from paper_2512_11624_b200 import synthetic
    from paper_2512_11624_b200.device_setup import DeviceStacks, device_init_field, device_point_batch
    cfg = synthetic.CONFIGS["cfg3"]
    stacks, _ = synthetic.make_stacks(cfg, seed=0)
    icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
    t0 = time.perf_counter()
    hb = g.build_point_batch(stacks)
    t1 = time.perf_counter()
    hf = g.init_field(g.sample_init_positions(stacks, icfg), stacks, icfg)
    t2 = time.perf_counter()
    for rep in range(2):
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        ds = DeviceStacks(stacks)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        db = device_point_batch(ds)
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        df = device_init_field(ds, icfg)
        torch.cuda.synchronize()
        t6 = time.perf_counter()
    print(f"cfg3 setup: host batch {t1 - t0:.3f} s, host init {t2 - t1:.3f} s; device: upload {t4 - t3:.3f} s, "
          f"batch {t5 - t4:.3f} s, init {t6 - t5:.3f} s")
    assert _same(db.lifted, hb.lifted)
    assert _same(db.slice_ids, hb.slice_ids)
    assert _same(db.intensities, hb.intensities)
    assert _same(df.means, hf.means)
    assert _same(df.intensities, hf.intensities)


@pytest.mark.parametrize("nbytes", [8, (4 << 20) - 8, (4 << 20) + 8, (32 << 20) * 5 + 24, (32 << 20) * 9])
def test_copy_d2h_any_destination(g, nbytes):
    """gsvr_copy_d2h (rasterize's result copy): pageable numpy destinations
    through the pinned staging ring (pieces of 32 MB, ring of 4), pinned ones
    directly; sizes around every piece / ring boundary."""
    import torch
    from paper_2512_11624_b200 import _dev
    n = nbytes // 8
    src = torch.arange(n, dtype=torch.float64, device="cuda") * 1.5 - 7.0
    want = src.cpu().numpy()
    dst = np.full(n, np.nan)
    _dev.copy_to_numpy(dst, src)
    assert np.array_equal(dst, want)
    pinned = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
    _dev.copy_to_numpy(pinned.numpy(), src)
    assert np.array_equal(pinned.numpy(), want)
