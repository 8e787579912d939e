"""Host half of the simulator (simulate.py:66-135, 208-242): the GT phantom
raster bit-identical to the reference's (tests/golden/desk_motion_data.npz),
stack geometry and parameter validation.  CPU only."""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_11624_b200 import InvalidParameterError
from paper_2512_11624_b200 import simulate as sim


def test_phantom_bit_identical_to_reference():
    z = np.load(GOLDEN / "desk_motion_data.npz")
    gt = sim.make_phantom(64, seed=0)
    assert np.array_equal(gt.data, z["gt_data"])
    assert np.array_equal(gt.mask, z["gt_mask"])
    np.testing.assert_array_equal(gt.affine, z["gt_affine"])


def test_stack_affines_match_reference():
    z = np.load(GOLDEN / "desk_motion_data.npz")
    gt = sim.make_phantom(64, seed=0)
    acq = sim.AcquisitionParams(inplane=0.5, thickness=3.0)
    for i, o in enumerate(acq.orientations):
        aff, n = sim._stack_affine(gt, acq, o)
        np.testing.assert_array_equal(aff, z[f"s{i}_affine"])
        assert tuple(n) == z[f"s{i}_data"].shape


def test_axis_nodes_and_validation():
    off, w = sim._axis_nodes(1.0, 3)
    assert len(off) == 19 and abs(w.sum() - 1.0) < 1e-15 and off[9] == 0.0
    off, w = sim._axis_nodes(0.0, 3)
    assert off.tolist() == [0.0] and w.tolist() == [1.0]
    with pytest.raises(InvalidParameterError):
        sim.MotionParams(rot_max=-1)
    with pytest.raises(InvalidParameterError):
        sim.AcquisitionParams(orientations=((0, 0, 1),))
    with pytest.raises(InvalidParameterError):
        sim.make_phantom(16)
