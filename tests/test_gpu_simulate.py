"""CUDA PSF quadrature (simulate.py:142-205) through the package's simulator vs
the reference simulator's own stacks: the 64^3 @ 0.5 mm motion desk acquisition
(noisy and clean, tests/golden/desk_motion*_data.npz) and cfg1 (1 mm / 4 mm,
cfg1_data.npz, stored float32).  Intensities rtol 1e-10 (float64), masks and
true slice states exact."""
import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    import torch
    assert torch.cuda.is_available()
    from paper_2512_11624_b200 import simulate
    return simulate


@pytest.mark.parametrize("tag,noise", [("desk_motion", 0.02), ("desk_motion_clean", 0.0)])
def test_desk_stacks_match_reference(sim, tag, noise):
    z = dict(np.load(GOLDEN / f"{tag}_data.npz"))
    gt = sim.make_phantom(64, seed=0)
    assert np.array_equal(gt.data, z["gt_data"])
    stacks, truths = sim.simulate_protocol(gt, sim.AcquisitionParams(inplane=0.5, thickness=3.0, noise_std=noise),
                                           sim.MotionParams(rot_max=6.0, trans_max=4.0, seed=0))
    for i, s in enumerate(stacks):
        ref = z[f"s{i}_data"]
        assert s.data.shape == ref.shape
        np.testing.assert_allclose(s.data, ref, rtol=1e-10, atol=1e-13)
        assert np.array_equal(s.mask, z[f"s{i}_mask"])
        np.testing.assert_array_equal(s.affine, z[f"s{i}_affine"])
    q = np.concatenate([t.quaternions for t in truths])
    t = np.concatenate([t.translations for t in truths])
    np.testing.assert_allclose(q, z["truth_q"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(t, z["truth_t"], rtol=0, atol=1e-13)


def test_cfg1_stacks_match_reference(sim):
    z = dict(np.load(GOLDEN / "cfg1_data.npz"))
    gt = sim.make_phantom(64, seed=0, spacing=1.0)
    stacks, _ = sim.simulate_protocol(gt, sim.AcquisitionParams(inplane=1.0, thickness=4.0, noise_std=0.0),
                                      sim.MotionParams(0.0, 0.0, seed=0))
    for i, s in enumerate(stacks):
        ref = z[f"s{i}_data"]  # float32 fixture
        assert np.all(np.abs(s.data - ref) <= 1e-7 * np.maximum(np.abs(ref), 1e-3))
        assert np.array_equal(s.mask, z[f"s{i}_mask"])


def test_quadrature_single_axes_and_validation(sim):
    """sid = NULL uses axes[0] for every centre; bad node counts are rejected."""
    import ctypes
    from paper_2512_11624_b200 import _dev
    from paper_2512_11624_b200._native import lib
    gt = sim.make_phantom(32, seed=1, spacing=1.0)
    r = sim._DeviceRaster(gt)
    rng = np.random.default_rng(0)
    c = rng.uniform(-10, 10, size=(500, 3))
    ax = np.eye(3)[None]
    nodes = [sim._axis_nodes(s, 2) for s in (0.4, 0.4, 1.2)]
    a = r.quadrature(r.vol, c, np.zeros(500, np.int32), ax, nodes)
    # host restatement of simulate.py:168-205 for a few centres
    inv = np.linalg.inv(gt.affine)[:3]
    vol = gt.data
    def tri(ix, iy, iz):
        nx, ny, nz = vol.shape
        if min(ix, iy, iz) < 0 or ix > nx - 1 or iy > ny - 1 or iz > nz - 1:
            return 0.0
        x0, y0, z0 = min(int(ix), nx - 2), min(int(iy), ny - 2), min(int(iz), nz - 2)
        fx, fy, fz = ix - x0, iy - y0, iz - z0
        v = vol[x0:x0 + 2, y0:y0 + 2, z0:z0 + 2]
        c0 = (v[0, 0, 0] * (1 - fx) + v[1, 0, 0] * fx) * (1 - fy) + (v[0, 1, 0] * (1 - fx) + v[1, 1, 0] * fx) * fy
        c1 = (v[0, 0, 1] * (1 - fx) + v[1, 0, 1] * fx) * (1 - fy) + (v[0, 1, 1] * (1 - fx) + v[1, 1, 1] * fx) * fy
        return c0 * (1 - fz) + c1 * fz
    for p in range(0, 500, 97):
        acc = 0.0
        for oa, wa in zip(*nodes[0]):
            for ob, wb in zip(*nodes[1]):
                for oc, wc in zip(*nodes[2]):
                    x = c[p] + np.array([oa, ob, oc])
                    i = inv[:, :3] @ x + inv[:, 3]
                    acc += wa * wb * wc * tri(*i)
        assert abs(a[p] - acc) <= 1e-12 * max(1.0, abs(acc))
    M = 10
    out = _dev.empty((M,), np.float64)
    cd = _dev.to_dev(c[:M], np.float64)
    ad = _dev.to_dev(ax, np.float64)
    nd = _dev.to_dev(np.zeros(6), np.float64)
    inv12 = (ctypes.c_double * 12)(*inv.ravel())
    rc = lib().gsvr_psf_quadrature(32, 32, 32, _dev.ptr(r.vol), ctypes.addressof(inv12), M, _dev.ptr(cd), None,
                                   _dev.ptr(ad), 0, 1, 1, _dev.ptr(nd), _dev.ptr(out), _dev.stream_ptr())
    assert rc == 1
