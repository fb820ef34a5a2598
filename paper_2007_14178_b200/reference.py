"""Slow, obviously-correct convolutions (drop-in for xnorconv.reference,
/root/reference/pkg/src/xnorconv/reference.py).

The reference keeps these scalar loops as the truth its verify and bench gates
check the packed engine against.  Here they run on the device as naive CUDA
kernels (csrc/xnc_verify.cu: one thread per output, the reference's (ch, ky, kx)
order, one rounding per operation) that share no code with the packed engine:
no bit packing, no popcount, no K map.  Same names, arguments, validation and
error messages as reference.py:19-122."""
from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _dev
from ._lib import check
from .binarize import BinaryWeightApprox, SignPlane
from .engine import IntOutputPlane
from .tensor import Tensor2, Tensor3


def _out_dims(h: int, w: int, kh: int, kw: int, pad: int) -> tuple[int, int]:
    """reference.py:19-27."""
    if pad < 0:
        raise ValueError("pad must be >= 0")
    out_h = h + 2 * pad - kh + 1
    out_w = w + 2 * pad - kw + 1
    if out_h < 1 or out_w < 1:
        raise ValueError(f"kernel {kh}x{kw} larger than padded {h}x{w} input")
    return out_h, out_w


def _conv_f64(x: np.ndarray, w: np.ndarray, pad: int, bwn: bool, scale: float) -> np.ndarray:
    c, h, wd = x.shape
    kh, kw = w.shape[1:]
    oh, ow = _out_dims(h, wd, kh, kw, pad)
    xd, wdv = _dev.to_dev(np.ascontiguousarray(x, np.float64)), _dev.to_dev(np.ascontiguousarray(w, np.float64))
    out = _dev.empty((oh, ow), np.float64)
    check(_dev.L().xnc_ref_conv2d_f64(xd.data_ptr(), wdv.data_ptr(), c, h, wd, kh, kw, pad, int(bwn),
                                      float(scale), out.data_ptr(), _dev.stream()), "xnc_ref_conv2d_f64")
    return _dev.to_host(out)


def conv2d_float(input: Tensor3, weights: Tensor3, pad: int = 0) -> Tensor2:
    """Full-precision cross-correlation, zero padding, unit stride (reference.py:30-54)."""
    if input.channels != weights.channels:
        raise ValueError(f"{input.channels} input channels vs {weights.channels} weight channels")
    _out_dims(input.height, input.width, weights.height, weights.width, pad)
    return Tensor2(_conv_f64(input.data, weights.data, pad, False, 1.0))


def sign_conv2d_int(input_signs: Sequence[SignPlane], weight_signs: Sequence[SignPlane],
                    pad: int = 0) -> IntOutputPlane:
    """Integer cross-correlation of +-1 planes summed over channels; padding
    pixels count as +1 (reference.py:57-90)."""
    if len(input_signs) != len(weight_signs):
        raise ValueError(f"{len(input_signs)} input channels vs {len(weight_signs)} weight channels")
    h, w = input_signs[0].height, input_signs[0].width
    kh, kw = weight_signs[0].height, weight_signs[0].width
    oh, ow = _out_dims(h, w, kh, kw, pad)
    s = _dev.to_dev(np.stack([p.signs for p in input_signs]).astype(np.int8))
    ws = _dev.to_dev(np.stack([p.signs for p in weight_signs]).astype(np.int8))
    out = _dev.empty((oh, ow), np.int32)
    check(_dev.L().xnc_ref_sign_conv2d(s.data_ptr(), ws.data_ptr(), len(input_signs), h, w, kh, kw, pad,
                                       out.data_ptr(), _dev.stream()), "xnc_ref_sign_conv2d")
    return IntOutputPlane(_dev.to_host(out))


def bwn_conv(input: Tensor3, w_approx: BinaryWeightApprox, pad: int = 0) -> Tensor2:
    """Convolution against +-1 weights (adds/subtracts only), times the scale
    (reference.py:93-122)."""
    if input.channels != len(w_approx.signs):
        raise ValueError(f"{input.channels} input channels vs {len(w_approx.signs)} weight channels")
    kh, kw = w_approx.signs[0].height, w_approx.signs[0].width
    _out_dims(input.height, input.width, kh, kw, pad)
    wsig = np.stack([p.signs for p in w_approx.signs]).astype(np.float64)
    return Tensor2(_conv_f64(input.data, wsig, pad, True, w_approx.scale))
