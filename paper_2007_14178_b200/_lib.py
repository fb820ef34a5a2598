"""ctypes binding of libxnorb200.so (include/xnorb200.h).

The product path has exactly one implementation: the sm_100a kernels in this
library.  If the library is missing or no CUDA device is present, every
operator raises -- there is no CPU fallback (BASELINE.json north star)."""
from __future__ import annotations

import ctypes
import os

from ._build import LIB_PATH

_LIB = None


class XncError(RuntimeError):
    """A libxnorb200 call returned a non-zero status."""


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    # XNC_LIB: an alternative build of the same library (tuning experiments only)
    path = os.environ.get("XNC_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise RuntimeError(
            f"libxnorb200.so not built ({path}); run `python -c \"import __graft_entry__ as g; "
            "g.build()\"` -- the B200 path has no CPU fallback")
    L = ctypes.CDLL(path)
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    LG, D, U64 = ctypes.c_long, ctypes.c_double, ctypes.c_uint64
    sig = {
        "xnc_abi_version": ([], I),
        "xnc_strerror": ([I], ctypes.c_char_p),
        "xnc_pack_input": ([P, I, I, I, I, P, P, P], I),
        "xnc_pack_weights": ([P, I, I, I, I, P, P, P, P], I),
        "xnc_pack_weights_f64": ([P, I, I, I, I, P, P, P, P], I),
        "xnc_scale_map": ([P, I, I, I, I, I, I, P, P], I),
        "xnc_xnor_conv": ([P, P, P, P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_xnor_conv_variant": ([I, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_layer_workspace_bytes": ([I, I, I, I, I, I, I], S),
        "xnc_umma_weight_bytes": ([I, I, I, I], S),
        "xnc_umma_supported": ([I, I, I, I, I, I, I, I], I),
        "xnc_pack_weights_umma": ([P, I, I, I, I, I, P, P, P], I),
        "xnc_xnor_conv_umma": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_umma_profile": ([P, I], I),
        "xnc_pack_input_affine": ([P, I, I, I, I, P, P, P, P, P], I),
        "xnc_xnor_conv_umma_affine": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P], I),
        "xnc_umma_split_ws_bytes": ([I, I, I, I, I, I, I, I], S),
        "xnc_umma_emit_supported": ([I, I, I, I, I, I, I, I], I),
        "xnc_xnor_conv_umma_emit": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P], I),
        "xnc_max_pool": ([P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_pad_space_to_depth": ([P, I, I, I, I, I, I, I, P, P], I),
        "xnc_plane_affine": ([P, I, I, LG, P, P, P], I),
        "xnc_pack_input_nhwc": ([P, I, I, I, I, P, P, P, P, P], I),
        "xnc_pack_input_pool": ([P, I, I, I, I, I, I, P, P, P, P, P], I),
        "xnc_pack_input_pool_nhwc": ([P, I, I, I, I, I, I, I, P, P, P, P, P, P], I),
        "xnc_xnor_conv_umma_ws": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P, P], I),
        "xnc_layer_forward": ([P, P, P, I, I, I, I, I, I, I, I, P, P, P, P], I),
        "xnc_layer_forward_umma": ([P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P], I),
        "xnc_pack_plane": ([P, I, I, I, I, I, I, I, I, I, P, P], I),
        "xnc_unpack_plane": ([P, I, I, I, I, I, I, P, P, P], I),
        "xnc_sign_plane": ([P, LG, P, P], I),
        "xnc_xnor_accumulate": ([P, I, I, I, P, U64, I, I, I, I, P, I, I, P], I),
        "xnc_filter_words": ([P, I, I, I, I, I, P, P, P], I),
        "xnc_box_mean": ([P, I, I, I, I, I, D, P, P, P], I),
        "xnc_scale_rows": ([P, I, I, I, I, I, P, P], I),
        "xnc_scale_join": ([P, I, P, I, D, D, I, I, P, P], I),
        "xnc_xnor_reconstruct": ([P, U64, I, I, I, I, I, P, I, I, I, I, I, I, D, D, P, P], I),
        "xnc_channel_abs_mean_f64": ([P, I, I, I, P, P], I),
        "xnc_apply_scaling_f64": ([P, P, D, LG, P, P], I),
        "xnc_ref_sign_conv2d": ([P, P, I, I, I, I, I, I, P, P], I),
        "xnc_ref_conv2d_f64": ([P, P, I, I, I, I, I, I, I, D, P, P], I),
        "xnc_vanilla_conv": ([P, I, I, I, I, P, I, I, P, P], I),
        "xnc_xnor_conv_umma_nhwc": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P], I),
        "xnc_xnor_conv_umma_nhwc_emit": ([P, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P, P, P], I),
        "xnc_conv1_weight_bytes": ([], S),
        "xnc_conv1_pack_weights": ([P, P, P], I),
        "xnc_conv1_forward": ([P, I, P, P, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = L
    return L


def exported_symbols() -> list[str]:
    """Names the header declares (kept in sync by tests/test_capi.py)."""
    return ["xnc_abi_version", "xnc_strerror", "xnc_pack_input", "xnc_pack_weights",
            "xnc_pack_weights_f64", "xnc_scale_map", "xnc_xnor_conv", "xnc_xnor_conv_variant",
            "xnc_layer_workspace_bytes", "xnc_layer_forward", "xnc_layer_forward_umma", "xnc_umma_weight_bytes",
            "xnc_umma_supported", "xnc_pack_weights_umma", "xnc_xnor_conv_umma", "xnc_umma_profile", "xnc_pack_input_affine", "xnc_xnor_conv_umma_affine",
            "xnc_umma_split_ws_bytes", "xnc_xnor_conv_umma_ws", "xnc_max_pool", "xnc_pad_space_to_depth", "xnc_plane_affine",
            "xnc_pack_input_nhwc", "xnc_pack_input_pool", "xnc_pack_input_pool_nhwc", "xnc_umma_emit_supported", "xnc_xnor_conv_umma_emit", "xnc_pack_plane", "xnc_unpack_plane",
            "xnc_sign_plane", "xnc_xnor_accumulate", "xnc_filter_words", "xnc_box_mean",
            "xnc_scale_rows", "xnc_scale_join", "xnc_xnor_reconstruct", "xnc_channel_abs_mean_f64",
            "xnc_apply_scaling_f64", "xnc_ref_sign_conv2d", "xnc_ref_conv2d_f64", "xnc_vanilla_conv",
            "xnc_conv1_weight_bytes", "xnc_conv1_pack_weights", "xnc_conv1_forward",
            "xnc_xnor_conv_umma_nhwc", "xnc_xnor_conv_umma_nhwc_emit"]

DTYPE_F32, DTYPE_F64, DTYPE_I8 = 0, 1, 2
XNC_ENOTSUP = 2  # include/xnorb200.h: shape outside what the kernels support


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().xnc_strerror(rc).decode()
        raise XncError(f"{what} failed: {msg} (code {rc})")
