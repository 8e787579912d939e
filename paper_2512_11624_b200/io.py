"""Field and volume interchange: the reference's native
field container (formats.py:37-74) and its NIfTI-1 subset (nifti.py).

Host-side byte formats, no device work.  The NIfTI-1 header is a numpy
structured dtype laid out as the NIfTI-1 standard defines it (348 bytes,
little-endian); the read/write contract follows the reference:

* field file: magic ``GSVR``, u32 version 1, u64 count N, then little-endian
  float32 means (N,3), log_scales (N,3), quaternions (N,4), intensities (N,)
  (formats.py:37-74); arrays come back float32.
* read: little-endian NIfTI-1, magic ``n+1\\0`` (data at vox_offset, 0 meaning
  352) or ``ni1\\0`` (data in the sibling ``.img``); uint8 / int16 / float32 /
  float64; 3-D (trailing unit dims allowed); affine from the sform when
  sform_code > 0, else the qform, else the pixdim diagonal; scl_slope /
  scl_inter rescale (slope 0 = 1); optional [0, 1] window from the 0.5 / 99.5
  percentiles (nifti.py:126-168).
* write: single-file float32, sform affine, vox_offset 352 (348-byte header +
  4 zero bytes), pixdim = column norms of the affine, deterministic bytes
  (nifti.py:192-227) -- byte-identical to the reference writer (tested).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path
from typing import Tuple, Union

import numpy as np

from .errors import UnsupportedFormatError
from .field import GaussianField
from .geometry import quat_to_rotation
from .motion import SliceStack
from .volume import VolumeGrid

PathLike = Union[str, Path]

# ---------------------------------------------------------------------------
# native field container (formats.py:37-74)

FIELD_MAGIC = b"GSVR"
FIELD_VERSION = 1
_FIELD_HEAD = np.dtype([("magic", "S4"), ("version", "<u4"), ("count", "<u8")])


def write_field(field: GaussianField, path: PathLike) -> None:
    """formats.py:37-46: the field as the native little-endian float32 container."""
    head = np.zeros((), _FIELD_HEAD)
    head["magic"], head["version"], head["count"] = FIELD_MAGIC, FIELD_VERSION, field.count
    parts = [head.tobytes()] + [np.ascontiguousarray(a, dtype="<f4").tobytes()
                                for a in (field.means, field.log_scales, field.quaternions,
                                          field.intensities)]
    Path(path).write_bytes(b"".join(parts))


def read_field(path: PathLike) -> GaussianField:
    """formats.py:49-74: load a field container (float32 arrays)."""
    path = Path(path)
    raw = path.read_bytes()
    if len(raw) < _FIELD_HEAD.itemsize:
        raise UnsupportedFormatError(f"{path}: too short for a field file")
    head = np.frombuffer(raw, _FIELD_HEAD, count=1)[0]
    if bytes(raw[:4]) != FIELD_MAGIC:
        raise UnsupportedFormatError(f"{path}: magic {bytes(raw[:4])!r} is not {FIELD_MAGIC!r}")
    if int(head["version"]) != FIELD_VERSION:
        raise UnsupportedFormatError(f"{path}: unsupported field file version {int(head['version'])}")
    n = int(head["count"])
    widths = (3, 3, 4, 1)
    expected = _FIELD_HEAD.itemsize + 4 * n * sum(widths)
    if len(raw) != expected:
        raise UnsupportedFormatError(f"{path}: expected {expected} bytes for N={n}, file has {len(raw)}")
    body = np.frombuffer(raw, "<f4", offset=_FIELD_HEAD.itemsize)
    cuts = np.cumsum([0] + [w * n for w in widths])
    arr = [body[cuts[i]:cuts[i + 1]].copy() for i in range(4)]
    return GaussianField(means=arr[0].reshape(-1, 3), log_scales=arr[1].reshape(-1, 3),
                         quaternions=arr[2].reshape(-1, 4), intensities=arr[3])


# ---------------------------------------------------------------------------
# NIfTI-1 (nifti.py)

NIFTI_HEADER = np.dtype([
    ("sizeof_hdr", "<i4"), ("data_type", "S10"), ("db_name", "S18"), ("extents", "<i4"),
    ("session_error", "<i2"), ("regular", "S1"), ("dim_info", "u1"), ("dim", "<i2", (8,)),
    ("intent_p", "<f4", (3,)), ("intent_code", "<i2"), ("datatype", "<i2"), ("bitpix", "<i2"),
    ("slice_start", "<i2"), ("pixdim", "<f4", (8,)), ("vox_offset", "<f4"), ("scl_slope", "<f4"),
    ("scl_inter", "<f4"), ("slice_end", "<i2"), ("slice_code", "u1"), ("xyzt_units", "u1"),
    ("cal_max", "<f4"), ("cal_min", "<f4"), ("slice_duration", "<f4"), ("toffset", "<f4"),
    ("glmax", "<i4"), ("glmin", "<i4"), ("descrip", "S80"), ("aux_file", "S24"),
    ("qform_code", "<i2"), ("sform_code", "<i2"), ("quatern", "<f4", (3,)), ("qoffset", "<f4", (3,)),
    ("srow", "<f4", (3, 4)), ("intent_name", "S16"), ("magic", "S4"),
])
assert NIFTI_HEADER.itemsize == 348
SINGLE_FILE_OFFSET = 352
_CODES = {2: np.dtype("<u1"), 4: np.dtype("<i2"), 16: np.dtype("<f4"), 64: np.dtype("<f8")}
_WINDOW = (0.5, 99.5)
_DESCRIP = b"gaussian slice-to-volume reconstruction"


@dataclass(frozen=True)
class IntensityNormalization:
    """nifti.py:41-56: affine window raw -> [0, 1] (clipped) and back."""

    lo: float
    hi: float

    @staticmethod
    def identity() -> "IntensityNormalization":
        return IntensityNormalization(0.0, 1.0)

    def normalize(self, values) -> np.ndarray:
        return np.clip((np.asarray(values, dtype=np.float64) - self.lo) / (self.hi - self.lo), 0.0, 1.0)

    def denormalize(self, values) -> np.ndarray:
        return np.asarray(values, dtype=np.float64) * (self.hi - self.lo) + self.lo


def _header(raw: bytes, path: Path) -> np.void:
    if len(raw) < NIFTI_HEADER.itemsize:
        raise UnsupportedFormatError(f"{path}: {len(raw)} bytes is shorter than a NIfTI-1 header")
    h = np.frombuffer(raw, NIFTI_HEADER, count=1)[0]
    if int(h["sizeof_hdr"]) != NIFTI_HEADER.itemsize:
        swapped = int(np.frombuffer(raw[:4], ">i4")[0]) == NIFTI_HEADER.itemsize
        raise UnsupportedFormatError(f"{path}: big-endian NIfTI is not supported" if swapped
                                     else f"{path}: sizeof_hdr {int(h['sizeof_hdr'])} is not 348")
    magic = bytes(raw[344:348])
    if magic not in (b"n+1\x00", b"ni1\x00"):
        raise UnsupportedFormatError(f"{path}: magic {magic!r} is not n+1\\0 or ni1\\0")
    return h


def _shape(h, path: Path) -> Tuple[int, int, int]:
    dim = [int(d) for d in h["dim"]]
    rank = dim[0]
    if not 1 <= rank <= 7:
        raise UnsupportedFormatError(f"{path}: dim[0] = {rank} is not a valid rank")
    if rank < 3 or any(d > 1 for d in dim[4:1 + rank]):
        raise UnsupportedFormatError(f"{path}: dim {tuple(dim[:1 + rank])} is not a 3-D volume (header field dim)")
    shape = tuple(dim[1:4])
    if min(shape) < 1:
        raise UnsupportedFormatError(f"{path}: non-positive size in dim {shape}")
    return shape


def _affine(h) -> np.ndarray:
    A = np.eye(4)
    if int(h["sform_code"]) > 0:
        A[:3, :] = np.asarray(h["srow"], dtype=np.float64)
        return A
    pix = [float(v) for v in h["pixdim"]]
    spacing = np.array([max(v, 0.0) or 1.0 for v in pix[1:4]])
    if int(h["qform_code"]) > 0:
        b, c, d = (float(v) for v in h["quatern"])
        a = math.sqrt(max(0.0, 1.0 - b * b - c * c - d * d))
        qfac = -1.0 if pix[0] < 0 else 1.0
        A[:3, :3] = quat_to_rotation(np.array([a, b, c, d])) * spacing * np.array([1.0, 1.0, qfac])
        A[:3, 3] = np.asarray(h["qoffset"], dtype=np.float64)
        return A
    A[:3, :3] = np.diag(spacing)
    return A


def _load(path: PathLike, normalize: bool):
    path = Path(path)
    raw = path.read_bytes()
    h = _header(raw, path)
    shape = _shape(h, path)
    code = int(h["datatype"])
    if code not in _CODES:
        raise UnsupportedFormatError(f"{path}: datatype code {code} is outside the supported subset "
                                     "(header field datatype)")
    dt = _CODES[code]
    if bytes(h["magic"]) == b"ni1":
        img = path.with_suffix(".img")
        if not img.exists():
            raise UnsupportedFormatError(f"{path}: paired data file {img} is missing")
        payload, offset = img.read_bytes(), int(float(h["vox_offset"]))
    else:
        payload, offset = raw, int(float(h["vox_offset"])) or SINGLE_FILE_OFFSET
    count = int(np.prod(shape))
    if len(payload) < offset + count * dt.itemsize:
        raise UnsupportedFormatError(f"{path}: expected {offset + count * dt.itemsize} bytes of data, "
                                     f"file has {len(payload)}")
    data = np.frombuffer(payload, dt, count=count, offset=offset).reshape(shape, order="F")
    slope = float(h["scl_slope"]) or 1.0
    inter = float(h["scl_inter"])
    values = data.astype(np.float64) * slope + inter if (slope != 1.0 or inter != 0.0) else data.copy()
    norm = IntensityNormalization.identity()
    if normalize:
        lo, hi = np.percentile(values.astype(np.float64), _WINDOW)
        if hi <= lo:
            hi = lo + 1.0  # constant volume: keep the window invertible
        norm = IntensityNormalization(float(lo), float(hi))
        values = norm.normalize(values)
    return values, _affine(h), norm


def read_nifti(path: PathLike, normalize: bool = True) -> Tuple[VolumeGrid, IntensityNormalization]:
    """nifti.py:171-175: a NIfTI-1 volume and the intensity window applied."""
    values, affine, norm = _load(path, normalize)
    return VolumeGrid(data=values, affine=affine), norm


def read_stack(path: PathLike, normalize: bool = True) -> Tuple[SliceStack, IntensityNormalization]:
    """nifti.py:178-189: axes 0, 1 in-plane, axis 2 = slices; thickness = axis-2 spacing."""
    values, affine, norm = _load(path, normalize)
    spacing = np.linalg.norm(affine[:3, :3], axis=0)
    return SliceStack(data=values, affine=affine, inplane_spacing=spacing[:2],
                      thickness=float(spacing[2])), norm


def write_nifti(grid: VolumeGrid, path: PathLike, norm: IntensityNormalization = None) -> None:
    """nifti.py:192-227: single-file float32 NIfTI-1, sform affine, vox_offset 352."""
    data = np.asarray(grid.data)
    if norm is not None:
        data = norm.denormalize(data)
    A = np.asarray(grid.affine, dtype=np.float64)
    h = np.zeros((), NIFTI_HEADER)
    h["sizeof_hdr"] = NIFTI_HEADER.itemsize
    h["regular"] = b"r"
    h["dim"] = [3, *data.shape, 1, 1, 1, 1]
    h["datatype"], h["bitpix"] = 16, 32
    h["pixdim"] = [1.0, *np.linalg.norm(A[:3, :3], axis=0), 0.0, 0.0, 0.0, 0.0]
    h["vox_offset"] = SINGLE_FILE_OFFSET
    h["scl_slope"], h["scl_inter"] = 1.0, 0.0
    h["xyzt_units"] = 2  # mm
    h["descrip"] = _DESCRIP
    h["qform_code"], h["sform_code"] = 0, 1
    h["srow"] = A[:3, :]
    h["magic"] = b"n+1"
    body = np.asarray(data, dtype="<f4").tobytes(order="F")
    Path(path).write_bytes(h.tobytes() + b"\x00\x00\x00\x00" + body)
