"""render.render_observed (render.py:22-65) on the device vs the reference's
own outputs (oracle/gen_render_golden.py): shared and per-point rotations,
per-point sigma, float64 (rtol 1e-10) and float32 (1e-5 rel + 1e-9 abs) fields,
and the reference's validation errors."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    assert torch.cuda.is_available()
    import paper_2512_11624_b200 as pkg
    return pkg


def _field(g, d, dtype=np.float64):
    return g.GaussianField(d["means"], d["log_scales"], d["quaternions"],
                           d["intensities"]).astype(dtype)


def test_render_observed_matches_reference(g):
    from paper_2512_11624_b200.render import render_observed
    d = load_golden("render_observed_cases")
    psf = g.build_psf(float(d["psf_inplane"]), float(d["psf_thickness"]))
    f = _field(g, d)
    got = render_observed(d["points"], d["R_shared"], f, psf, d["nbr"])
    np.testing.assert_allclose(got, d["out_shared64"], rtol=1e-10, atol=1e-14)
    got = render_observed(d["points"], d["R_per"], f, psf, d["nbr"], sigma_slice=d["sigma_per"])
    np.testing.assert_allclose(got, d["out_per64"], rtol=1e-10, atol=1e-14)
    got32 = render_observed(d["points"], d["R_per"], _field(g, d, np.float32), psf, d["nbr"],
                            sigma_slice=d["sigma_per"])
    assert got32.dtype == np.float32
    ref = d["out_per32"].astype(np.float64)
    assert np.all(np.abs(got32 - ref) <= 1e-5 * np.abs(ref) + 1e-9)


def test_render_observed_validation(g):
    from paper_2512_11624_b200.render import render_observed
    d = load_golden("render_observed_cases")
    psf = g.build_psf(0.5, 3.0)
    f = _field(g, d)
    with pytest.raises(g.InvalidParameterError, match="rows must match"):
        render_observed(d["points"], d["R_shared"], f, psf, d["nbr"][:-1])
    bad = d["nbr"].copy()
    bad[3, 2] = f.count
    with pytest.raises(g.InvalidParameterError, match="out of range"):
        render_observed(d["points"], d["R_shared"], f, psf, bad)
    with pytest.raises(g.InvalidParameterError, match="slice_rotations"):
        render_observed(d["points"], np.eye(2), f, psf, d["nbr"])
