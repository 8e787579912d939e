"""Field container and NIfTI-1 interchange vs the reference (tests/golden/io_cases.npz,
made by oracle/gen_io_golden.py): writers byte-identical, readers returning the
reference's values / affine / window on crafted files (int16 + scl, qform with
qfac -1, pixdim only, uint8 with vox_offset 0, 4-D float64, .hdr/.img pair)."""
import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def d():
    return load_golden("io_cases")


def test_field_container_bytes_and_roundtrip(d, tmp_path):
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200 import io
    f = g.GaussianField(d["field_means"], d["field_log_scales"], d["field_quats"], d["field_cvals"])
    io.write_field(f, tmp_path / "f.gsvr")
    assert (tmp_path / "f.gsvr").read_bytes() == d["field_bytes"].tobytes()
    back = io.read_field(tmp_path / "f.gsvr")
    for a, b in ((back.means, f.means), (back.log_scales, f.log_scales), (back.quaternions, f.quaternions),
                 (back.intensities, f.intensities)):
        assert a.dtype == np.float32
        np.testing.assert_array_equal(a, b.astype(np.float32))
    (tmp_path / "bad.gsvr").write_bytes(b"GSVX" + d["field_bytes"].tobytes()[4:])
    with pytest.raises(g.UnsupportedFormatError):
        io.read_field(tmp_path / "bad.gsvr")
    (tmp_path / "short.gsvr").write_bytes(d["field_bytes"].tobytes()[:-4])
    with pytest.raises(g.UnsupportedFormatError):
        io.read_field(tmp_path / "short.gsvr")


def test_write_nifti_bytes(d, tmp_path):
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200 import io
    io.write_nifti(g.VolumeGrid(d["grid_data"], d["grid_affine"]), tmp_path / "g.nii")
    assert (tmp_path / "g.nii").read_bytes() == d["grid_bytes"].tobytes()


@pytest.mark.parametrize("kind", ["int16_scl", "qform", "uint8", "float64_4d", "pair", "plain"])
def test_read_nifti_matches_reference(d, kind, tmp_path):
    from paper_2512_11624_b200 import io
    p = tmp_path / (kind + (".hdr" if (kind + "_img") in d else ".nii"))
    p.write_bytes(d[kind + "_raw"].tobytes())
    if (kind + "_img") in d:
        p.with_suffix(".img").write_bytes(d[kind + "_img"].tobytes())
    for norm in (0, 1):
        grid, win = io.read_nifti(p, normalize=bool(norm))
        np.testing.assert_array_equal(grid.data, d[f"{kind}_n{norm}_data"])
        np.testing.assert_array_equal(grid.affine, d[f"{kind}_n{norm}_affine"])
        np.testing.assert_array_equal([win.lo, win.hi], d[f"{kind}_n{norm}_window"])
    st, _ = io.read_stack(p)
    np.testing.assert_array_equal(st.inplane_spacing, d[kind + "_stack_spacing"])
    assert st.thickness == float(d[kind + "_stack_thickness"])


def test_nifti_errors(d, tmp_path):
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200 import io
    raw = bytearray(d["plain_raw"].tobytes())
    bad = tmp_path / "bad.nii"
    bad.write_bytes(bytes(raw[:100]))
    with pytest.raises(g.UnsupportedFormatError):
        io.read_nifti(bad)
    raw2 = bytearray(raw)
    raw2[344:348] = b"xx1\x00"
    bad.write_bytes(bytes(raw2))
    with pytest.raises(g.UnsupportedFormatError):
        io.read_nifti(bad)
    raw3 = bytearray(raw)
    raw3[70:72] = np.int16(32).tobytes()  # complex64: outside the subset
    bad.write_bytes(bytes(raw3))
    with pytest.raises(g.UnsupportedFormatError):
        io.read_nifti(bad)
