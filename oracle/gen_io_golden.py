"""Golden interchange cases from the REFERENCE (this container only).

    python oracle/gen_io_golden.py

* the reference's write_field / write_nifti bytes for a small field / grid;
* crafted NIfTI-1 files (int16 + scl rescale, qform-only with qfac -1,
  pixdim-only, uint8, float64, a 4-D file with unit trailing dims, a
  header/image pair) and what the reference's read_nifti / read_stack return
  for them (values, affine, window), with and without normalisation.
-> tests/golden/io_cases.npz (bytes stored as uint8 arrays).
"""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsvr_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "io_cases.npz"


def crafted(kind, rng):
    """Header bytes + payload for a crafted case (independent of both implementations)."""
    from paper_2512_11624_b200.io import NIFTI_HEADER
    shape = (5, 4, 3)
    h = np.zeros((), NIFTI_HEADER)
    h["sizeof_hdr"] = 348
    h["dim"] = [3, *shape, 1, 1, 1, 1]
    h["pixdim"] = [1.0, 1.2, 0.9, 3.0, 0, 0, 0, 0]
    h["vox_offset"] = 352
    h["magic"] = b"n+1"
    code, dt = 16, "<f4"
    data = rng.normal(size=shape) * 40 + 100
    if kind == "int16_scl":
        code, dt = 4, "<i2"
        data = rng.integers(-300, 900, size=shape)
        h["scl_slope"], h["scl_inter"] = 0.5, -7.0
        h["sform_code"] = 2
        h["srow"] = [[0.0, 0.9, 0.1, -4.0], [1.2, 0.0, 0.0, 2.0], [0.0, 0.05, 3.0, 7.5]]
    elif kind == "qform":
        h["qform_code"] = 1
        h["pixdim"][0] = -1.0
        h["quatern"] = [0.1, -0.2, 0.3]
        h["qoffset"] = [10.0, -20.0, 5.0]
    elif kind == "uint8":
        code, dt = 2, "<u1"
        data = rng.integers(0, 255, size=shape)
        h["vox_offset"] = 0  # 0 -> 352
    elif kind == "float64_4d":
        code, dt = 64, "<f8"
        h["dim"] = [4, *shape, 1, 1, 1, 1]
    elif kind == "pair":
        h["magic"] = b"ni1"
        h["vox_offset"] = 0
    h["datatype"] = code
    h["bitpix"] = np.dtype(dt).itemsize * 8
    payload = np.asarray(data).astype(dt).tobytes(order="F")
    if kind == "pair":
        return h.tobytes(), payload
    pad = b"\x00" * (352 - 348)
    return h.tobytes() + pad + payload, None


def main():
    from gsvr.field import GaussianField
    from gsvr.formats import write_field
    from gsvr.nifti import read_nifti, read_stack, write_nifti
    from gsvr.volume import VolumeGrid
    rng = np.random.default_rng(12)
    d = {}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        n = 37
        f = GaussianField(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 4)),
                          rng.random(n))
        write_field(f, tmp / "f.gsvr")
        d["field_means"], d["field_log_scales"] = f.means, f.log_scales
        d["field_quats"], d["field_cvals"] = f.quaternions, f.intensities
        d["field_bytes"] = np.frombuffer((tmp / "f.gsvr").read_bytes(), np.uint8)
        aff = np.array([[0.0, 1.1, 0.2, -3.0], [0.9, 0.0, 0.0, 4.0], [0.1, 0.0, 2.5, 1.0], [0, 0, 0, 1]])
        g = VolumeGrid(rng.normal(size=(6, 5, 4)), aff)
        write_nifti(g, tmp / "g.nii")
        d["grid_data"], d["grid_affine"] = g.data, aff
        d["grid_bytes"] = np.frombuffer((tmp / "g.nii").read_bytes(), np.uint8)
        kinds = ["int16_scl", "qform", "uint8", "float64_4d", "pair", "plain"]
        for k in kinds:
            raw, img = crafted(k, rng)
            p = tmp / (k + (".hdr" if img is not None else ".nii"))
            p.write_bytes(raw)
            if img is not None:
                p.with_suffix(".img").write_bytes(img)
                d[k + "_img"] = np.frombuffer(img, np.uint8)
            d[k + "_raw"] = np.frombuffer(raw, np.uint8)
            for norm in (False, True):
                grid, win = read_nifti(p, normalize=norm)
                d[f"{k}_n{int(norm)}_data"] = grid.data
                d[f"{k}_n{int(norm)}_affine"] = grid.affine
                d[f"{k}_n{int(norm)}_window"] = np.array([win.lo, win.hi])
            st, _ = read_stack(p, normalize=True)
            d[k + "_stack_spacing"] = np.asarray(st.inplane_spacing, dtype=np.float64)
            d[k + "_stack_thickness"] = np.float64(st.thickness)
        d["kinds"] = np.array(kinds)
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
