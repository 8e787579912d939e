"""Device plumbing: numpy / torch arrays <-> contiguous CUDA tensors and raw pointers.

torch is used only for device memory, streams and host<->device copies; all
compute goes through the C ABI in _native.py.
"""
from __future__ import annotations

import numpy as np
import torch

_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
          np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
          np.dtype(np.uint8): torch.uint8}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_11624_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def to_dev(x, dtype) -> torch.Tensor:
    """Contiguous CUDA tensor of the given numpy dtype (copies only when needed)."""
    tdt = _TORCH[np.dtype(dtype)]
    if isinstance(x, torch.Tensor):
        t = x.to(device=device(), dtype=tdt)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x), dtype=dtype)
    if not a.flags.writeable:  # read-only views (broadcasts, np.load mmaps): torch needs a writable buffer
        a = a.copy()
    return torch.from_numpy(a).to(device(), non_blocking=False)


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=_TORCH[np.dtype(dtype)], device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=_TORCH[np.dtype(dtype)], device=device())


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def write_back(dst, src: torch.Tensor) -> None:
    """Copy a device result into a caller-owned numpy array or tensor, in place."""
    if isinstance(dst, torch.Tensor):
        dst.copy_(src.reshape(dst.shape), non_blocking=False)
    else:
        np.copyto(dst, to_host(src).reshape(dst.shape).astype(dst.dtype, copy=False))


def torch_dtype(dtype) -> torch.dtype:
    return _TORCH[np.dtype(dtype)]


def copy_to_numpy(dst: np.ndarray, src: torch.Tensor) -> None:
    """Device tensor -> a C-contiguous numpy array of the same dtype and size,
    in place (pageable destinations through pinned staging pieces moved out
    by host threads, csrc/train.cu gsvr_copy_d2h)."""
    from ._native import check, lib
    if not dst.flags.c_contiguous or dst.dtype != np.dtype(str(src.dtype).replace("torch.", "")):
        raise ValueError("copy_to_numpy needs a C-contiguous destination of the source dtype")
    if dst.size != src.numel():
        raise ValueError("copy_to_numpy: size mismatch")
    src = src.contiguous()
    check(lib().gsvr_copy_d2h(dst.ctypes.data, src.data_ptr(), dst.nbytes, stream_ptr()), "device->host copy")
