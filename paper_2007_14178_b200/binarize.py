"""Sign binarization and closed-form scales (drop-in for xnorconv.binarize,
/root/reference/pkg/src/xnorconv/binarize.py).  sign(0) = sign(-0.0) = +1.
Signs and alpha are computed on the device (xnc_sign_plane, xnc_filter_words)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import check
from .tensor import Tensor2, Tensor3


@dataclass(frozen=True)
class SignPlane:
    """(height, width) plane of exactly +1 / -1 (int8)."""

    signs: np.ndarray

    def __post_init__(self):
        arr = np.array(self.signs, dtype=np.int8, order="C", copy=True)
        if arr.ndim != 2:
            raise ValueError(f"expected 2-d signs, got shape {arr.shape}")
        if not np.all((arr == 1) | (arr == -1)):
            raise ValueError("sign plane entries must be +1 or -1")
        arr.setflags(write=False)
        object.__setattr__(self, "signs", arr)

    height = property(lambda self: self.signs.shape[0])
    width = property(lambda self: self.signs.shape[1])


@dataclass(frozen=True)
class BinaryWeightApprox:
    """Per-channel sign planes and one non-negative filter scale."""

    signs: tuple
    scale: float

    def __post_init__(self):
        if len(self.signs) == 0:
            raise ValueError("at least one channel required")
        if self.scale < 0:
            raise ValueError("scale must be >= 0")


def _device_signs(values: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    x = _dev.to_dev(v)
    out = _dev.empty(v.shape, np.int8)
    check(_dev.L().xnc_sign_plane(x.data_ptr(), v.size, out.data_ptr(), _dev.stream()), "xnc_sign_plane")
    return _dev.to_host(out)


def sign_plane(x: Tensor2) -> SignPlane:
    """Elementwise sign with sign(0) = +1 (binarize.py:60-62)."""
    return SignPlane(_device_signs(x.data))


def filter_scales(w: np.ndarray, tile_w: int = 8):
    """(tile-layout weight words u64 [O][C], alpha f64 [O]) for a bank w [O][C][kh][kw]."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    O, C, kh, kw = w.shape
    words = _dev.empty((O, C), np.uint64)
    alpha = _dev.empty((O,), np.float64)
    check(_dev.L().xnc_filter_words(_dev.to_dev(w).data_ptr(), O, C, kh, kw, tile_w, words.data_ptr(),
                                    alpha.data_ptr(), _dev.stream()), "xnc_filter_words")
    return _dev.to_host(words, np.uint64), _dev.to_host(alpha)


def sign_binarize(w: Tensor3) -> BinaryWeightApprox:
    """Signs per channel plus alpha = sum|w| / n, accumulated sequentially in
    float64 in index order (binarize.py:65-75) -- on the device."""
    signs = _device_signs(w.data)
    return BinaryWeightApprox(tuple(SignPlane(s) for s in signs), float(flat_alpha(w.data)))


def flat_alpha(values: np.ndarray) -> float:
    """sum |v| / n over the flattened values, sequential float64 (any shape):
    xnc_pack_weights_f64 with one filter of n 1x1 channels has exactly that order."""
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    n = v.size
    wbits = _dev.empty(((n + 31) // 32,), np.int32)
    a32 = _dev.empty((1,), np.float32)
    a64 = _dev.empty((1,), np.float64)
    check(_dev.L().xnc_pack_weights_f64(_dev.to_dev(v).data_ptr(), 1, n, 1, 1, wbits.data_ptr(),
                                        a32.data_ptr(), a64.data_ptr(), _dev.stream()),
          "xnc_pack_weights_f64")
    return float(_dev.to_host(a64)[0])


def combined_scale(weight_scale: float, input_scale: float) -> float:
    """Product of the two scale factors (binarize.py:78-82)."""
    if weight_scale < 0 or input_scale < 0:
        raise ValueError("scale factors must be >= 0")
    return weight_scale * input_scale
