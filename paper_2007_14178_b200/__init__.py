"""B200-native (sm_100a) XNOR-Net binary-convolution forward path.

A from-scratch rebuild of the reference `xnorconv` package's hot path
(arXiv 2007.14178): sign binarization + channel bit-packing, the K scaling
map, the XNOR-popcount convolution and the alpha*K epilogue run as
hand-written CUDA kernels in libxnorb200.so (C-ABI: include/xnorb200.h).

The public names mirror the reference's operator API
(/root/reference/pkg/src/xnorconv/__init__.py:10-62) so the package is a
drop-in for that path; every compute function runs on the device.
`XnorConv2d` / `xnor_conv2d_layer` add the batched layer the reference lacks
(out[n, o] == xnor_conv(x[n], w[o]) for a whole batch in one pass); a layer can
hand the next binary layer its input in packed-sign form (`PackedInput`,
`XnorConv2d.forward(..., emit_signs=True)`), and `XnorNetAlexNet` is the
XNOR-Net AlexNet forward built from these layers.
"""
from . import ops  # noqa: F401
from .ops import PackedInput  # noqa: F401
from .binarize import BinaryWeightApprox, SignPlane, combined_scale, sign_binarize, sign_plane
from .engine import (BinaryFilter, GeometryMismatchError, IntOutputPlane, build_filter,
                     popcount_to_signed, xnor_conv2d, xnor_conv_multichannel, xnor_tile)
from .layer import XnorConv2d, default_pad, xnor_conv2d_layer
from .pack import OverlapMismatchError, PackedTileGrid, TileGeometry, pack, tile_grid_shape, unpack
from .pipeline import ConvWorkspace, xnor_conv
from .scaling import ScalingField, apply_scaling, box_kernel, input_scale_map, input_scaling_field
from .tensor import (BadMagicError, DimensionOverflowError, Tensor2, Tensor3, TensorFileError,
                     TruncatedPayloadError, channel_abs_mean, load_tensor, save_tensor, zero_pad)
from .network import XnorNetAlexNet  # noqa: F401

__version__ = "0.1.0"

DEFAULT_BACKEND = "b200"
HAVE_COMPILED = True  # the only backend; see compiled_available() for a live check


def compiled_available() -> bool:
    """True when libxnorb200.so loads and a CUDA device is present (the
    reference's equivalent reports its Cython extension, __init__.py:60-62)."""
    try:
        import torch

        from ._lib import lib
        lib()
        return torch.cuda.is_available()
    except Exception:
        return False
