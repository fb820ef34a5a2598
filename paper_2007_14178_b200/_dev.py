"""Host <-> device plumbing for the numpy-facing drop-in API (torch owns the
device memory and streams; the arithmetic is in libxnorb200.so)."""
from __future__ import annotations

import numpy as np
import torch

from ._lib import lib

_NP2TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
             np.dtype(np.int8): torch.int8, np.dtype(np.int32): torch.int32,
             np.dtype(np.uint64): torch.int64, np.dtype(np.int64): torch.int64}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream(device()).cuda_stream


def to_dev(arr: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).to(device())


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=_NP2TORCH[np.dtype(dtype)], device=device())


def to_host(t: torch.Tensor, dtype=None) -> np.ndarray:
    a = t.cpu().numpy()
    if dtype is not None and np.dtype(dtype) == np.uint64:
        return a.view(np.uint64)
    return a


def L():
    return lib()
