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
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libxnorb200.so not built ({LIB_PATH}); run `python -c \"import __graft_entry__ as g; "
            "g.build()\"` -- the B200 path has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    sig = {
        "xnc_abi_version": ([], I),
        "xnc_strerror": ([I], ctypes.c_char_p),
        "xnc_pack_input": ([P, I, I, I, I, P, P, P], I),
        "xnc_pack_weights": ([P, I, I, I, I, P, P, P, P], I),
        "xnc_scale_map": ([P, I, I, I, I, I, I, P, P], I),
        "xnc_xnor_conv": ([P, P, P, P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_xnor_conv_variant": ([I, P, P, P, P, I, I, I, I, I, I, I, I, P, P, P], I),
        "xnc_layer_workspace_bytes": ([I, I, I, I, I, I, I], S),
        "xnc_layer_forward": ([P, P, P, I, I, I, I, I, I, I, I, P, P, P, P], I),
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
            "xnc_scale_map", "xnc_xnor_conv", "xnc_xnor_conv_variant",
            "xnc_layer_workspace_bytes", "xnc_layer_forward"]


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().xnc_strerror(rc).decode()
        raise XncError(f"{what} failed: {msg} (code {rc})")
