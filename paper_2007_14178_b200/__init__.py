"""B200-native (sm_100a) XNOR-Net binary-convolution forward path.

A from-scratch rebuild of the reference `xnorconv` package's hot path
(arXiv 2007.14178): sign binarization + channel bit-packing, the K scaling
map, the XNOR-popcount convolution and the alpha*K epilogue run as
hand-written CUDA kernels in libxnorb200.so (C-ABI: include/xnorb200.h).
The public names mirror the reference's operator API (xnorconv/__init__.py)
so the package is a drop-in for that path; `XnorConv2d` / `xnor_conv2d_layer`
add the batched layer the reference does not have.
"""
from .layer import XnorConv2d, default_pad, xnor_conv2d_layer  # noqa: F401
from . import ops  # noqa: F401

__version__ = "0.1.0"
