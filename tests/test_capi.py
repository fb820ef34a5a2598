"""CPU-side checks of the drop-in boundary: libxnorb200.so builds for sm_100a,
loads, and exports every entry point include/xnorb200.h declares; the product
package never reaches the oracle (no CPU fallback)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2007_14178_b200")


def declared_symbols():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names += re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(xnc_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2007_14178_b200._build import build_library
    path = build_library()
    lib = ctypes.CDLL(path)
    names = declared_symbols()
    assert len(names) >= 8
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2007_14178_b200 import _lib
    assert sorted(_lib.exported_symbols()) == names


def test_library_carries_sm100a_cubins():
    from paper_2007_14178_b200._build import LIB_PATH, build_library
    build_library()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_errors_without_gpu():
    from paper_2007_14178_b200._lib import lib
    L = lib()
    assert L.xnc_abi_version() == 1
    assert L.xnc_strerror(0) == b"ok"
    # argument validation happens before any device work
    assert L.xnc_pack_input(None, 1, 1, 1, 1, None, None, None) == 1
    assert L.xnc_xnor_conv(None, None, None, None, 1, 1, 1, 1, 1, 3, 3, 1, None, None, None) == 1
    assert L.xnc_layer_workspace_bytes(1, 64, 8, 8, 9, 9, 1) == 0  # k > 8 rejected


def test_newer_entry_points_validate_before_device_work():
    """The network / binary-stack / K-split entry points reject bad arguments with
    XNC_EINVAL (1) before any CUDA call, so this runs without a GPU."""
    from paper_2007_14178_b200._lib import lib
    L = lib()
    EINVAL = 1
    # max-pool: NULL tensors, pool larger than the map, kernel > 8
    assert L.xnc_max_pool(None, 1, 1, 8, 8, 3, 2, 0, 0, None, None, None) == EINVAL
    assert L.xnc_max_pool(1, 1, 1, 2, 2, 3, 2, 0, 0, None, 1, None) == EINVAL
    assert L.xnc_max_pool(1, 1, 1, 16, 16, 9, 2, 0, 0, None, 1, None) == EINVAL
    # pad + space-to-depth: padded size not a multiple of r
    assert L.xnc_pad_space_to_depth(1, 1, 3, 9, 10, 1, 4, 0, 1, None) == EINVAL
    assert L.xnc_pad_space_to_depth(None, 1, 3, 224, 224, 2, 4, 0, 1, None) == EINVAL
    # channels-last K1: NULL x, and a scale without a shift
    assert L.xnc_pack_input_nhwc(None, 1, 8, 4, 4, None, None, 1, None, None) == EINVAL
    assert L.xnc_pack_input_nhwc(1, 1, 8, 4, 4, 1, None, 1, None, None) == EINVAL
    # sign-emitting conv: no next_bits buffer
    assert L.xnc_xnor_conv_umma_emit(1, 1, 1, 1, 1, 1, 64, 8, 8, 32, 3, 3, 1, None, None, None, None,
                                     None) == EINVAL
    # K-split conv: neither y nor acc
    assert L.xnc_xnor_conv_umma_ws(1, 1, 1, 1, 1, 1, 64, 8, 8, 32, 3, 3, 1, None, None, None, None, None,
                                   None) == EINVAL
    # size queries: impossible shapes report 0
    assert L.xnc_umma_split_ws_bytes(1, 64, 8, 8, 0, 3, 3, 1) == 0
    assert L.xnc_umma_emit_supported(1, 64, 8, 8, 0, 3, 3, 1) == 0


def test_product_package_never_imports_the_oracle():
    for path in glob.glob(os.path.join(PKG, "**", "*.py"), recursive=True):
        src = open(path).read()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), path
        assert "liboracle" not in src and "_kernels_cy" not in src, path


def test_ops_refuse_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2007_14178_b200 import ops
    with pytest.raises(ValueError, match="no CPU fallback"):
        ops.pack_input(torch.zeros((1, 3, 4, 4)))
