"""PSF constants and helpers (row a4) against the reference's own constants
(/root/reference/pkg/tests/test_psf.py:11-13) and reference-generated goldens
(oracle/gen_render_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import load_golden
from paper_2512_11624_b200 import InvalidParameterError
from paper_2512_11624_b200.geometry import build_covariance, quat_to_rotation, unpack_sym6
from paper_2512_11624_b200.psf import (FWHM_TO_SIGMA, PsfModel, build_psf, convolve_covariance,
                                       rotated_psf_cov6)

# the reference's frozen constants (tests/test_psf.py:11-13)
FWHM_TO_SIGMA_ORACLE = 0.42466090014400953
INPLANE_SIGMA_05MM = 0.25479654008640573
THROUGH_SIGMA_3MM = 1.2739827004320285


def test_fwhm_conversion_constant():
    assert abs(FWHM_TO_SIGMA - FWHM_TO_SIGMA_ORACLE) < 1e-15
    fwhm = 1.0 / FWHM_TO_SIGMA
    assert abs(np.exp(-0.5 * (fwhm / 2) ** 2) - 0.5) < 1e-12


def test_build_psf_standard_acquisition():
    psf = build_psf(0.5, 3.0)
    assert abs(psf.sigma_inplane[0] - INPLANE_SIGMA_05MM) < 1e-15
    assert abs(psf.sigma_inplane[1] - INPLANE_SIGMA_05MM) < 1e-15
    assert abs(psf.sigma_through - THROUGH_SIGMA_3MM) < 1e-15
    np.testing.assert_allclose(np.diag(psf.covariance),
                               [INPLANE_SIGMA_05MM ** 2] * 2 + [THROUGH_SIGMA_3MM ** 2])


def test_build_psf_anisotropic_and_validation():
    psf = build_psf((0.5, 1.0), 2.0)
    assert abs(psf.sigma_inplane[1] - 2 * psf.sigma_inplane[0]) < 1e-15
    for args in ((-0.5, 3.0), (0.5, 0.0), ((0.5, 0.5, 0.5), 3.0)):
        with pytest.raises(InvalidParameterError):
            build_psf(*args)


def test_slice_psf_diags_matches_constants():
    from paper_2512_11624_b200 import PointBatch, slice_psf_diags
    from paper_2512_11624_b200.motion import SliceStack, build_point_batch
    aff = np.diag([0.5, 0.5, 3.0, 1.0])
    st = SliceStack(np.ones((4, 3, 2)), aff, np.array([0.5, 0.5]), 3.0)
    b = build_point_batch([st])
    d = slice_psf_diags(b, [st])
    np.testing.assert_allclose(d, [[INPLANE_SIGMA_05MM ** 2] * 2 + [THROUGH_SIGMA_3MM ** 2]] * 2,
                               rtol=1e-15)
    assert np.all(slice_psf_diags(b, [st], use_psf=False) == 0)
    assert isinstance(b, PointBatch)


def test_rotated_psf_cov6_matches_reference():
    d = load_golden("render_observed_cases")
    got = rotated_psf_cov6(d["psf_R5"], build_psf(0.8, 2.5))
    np.testing.assert_allclose(got, d["psf_cov6_R5"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(unpack_sym6(got),
                               np.einsum("nik,kl,njl->nij", d["psf_R5"],
                                         build_psf(0.8, 2.5).covariance, d["psf_R5"]), atol=1e-13)


def test_convolve_covariance_matches_reference():
    d = load_golden("render_observed_cases")
    got = convolve_covariance(d["conv_cov"], d["conv_R"], build_psf(0.5, 3.0))
    np.testing.assert_allclose(got, d["conv_out"], rtol=0, atol=1e-15)
    # identity frame is the plain sum; disabled PSF leaves the covariance alone
    cov = build_covariance(np.log([0.9, 1.1, 1.4]), np.array([0.9, -0.1, 0.3, 0.2]))
    psf = build_psf(0.5, 3.0)
    np.testing.assert_allclose(convolve_covariance(cov, np.eye(3), psf), cov + psf.covariance,
                               atol=1e-15)
    np.testing.assert_array_equal(convolve_covariance(cov, np.eye(3), PsfModel.disabled()), cov)


def test_through_plane_dominates_along_slice_normal():
    psf = build_psf(0.5, 3.0)
    R = quat_to_rotation(np.array([0.9, 0.2, -0.3, 0.1]))
    added = convolve_covariance(np.zeros((3, 3)), R, psf)
    n = R[:, 2]
    assert abs(n @ added @ n - THROUGH_SIGMA_3MM ** 2) < 1e-12
    assert R[:, 0] @ added @ R[:, 0] < 0.1 * (n @ added @ n)
