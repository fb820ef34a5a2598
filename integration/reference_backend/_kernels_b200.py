"""Device backend for the reference `xnorconv` package: its kernel interface
(the seven caller-fills-output functions `_backend.get_kernels` returns,
/root/reference/pkg/src/xnorconv/_backend.py:28-41, signatures
_kernels_cy.pyx:42-354 / _kernels_py.py:45-193) bound to libxnorb200.so over
its C ABI (include/xnorb200.h) with ctypes.  No torch.

This file is what a reference maintainer drops into `pkg/src/xnorconv/`
(INTEGRATION.md section 1); `install.py` next to it does that to a copy of the
package, and tests/test_gpu_reference_backend.py runs the reference's own
ConvWorkspace / pack / xnor_conv_multichannel / run_verification through it.

Conventions kept from the reference: numpy arrays in, outputs filled in place,
None returned; C-contiguous typed buffers are required (the Cython boundary's
`[:, ::1]` memoryviews raise ValueError otherwise); `threads` is accepted and
ignored (the device grid replaces the OpenMP bands).  Each call is synchronous:
inputs are copied host -> device, the kernel runs on the legacy default stream,
outputs are copied back before returning.  This is the drop-in seam, not the
fast path (that is the batched layer).
"""
import ctypes
import glob
import os
import sys

import numpy as np

__all__ = ["pack_plane", "xnor_accumulate", "box_mean", "scale_rows", "scale_join",
           "xnor_reconstruct", "vanilla_conv"]


def _load_lib():
    path = os.environ.get("XNORB200_LIB", "libxnorb200.so")
    return ctypes.CDLL(path)


def _load_cudart():
    """The CUDA runtime for the host-side buffers (libxnorb200.so links its own
    copy statically; both drive the same primary context)."""
    cands = ["libcudart.so.12", "libcudart.so"]
    for base in sys.path:
        cands += glob.glob(os.path.join(base, "nvidia", "cuda_runtime", "lib", "libcudart.so.1*"))
    cands += ["/usr/local/cuda/lib64/libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"]
    err = None
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError as e:  # try the next location
            err = e
    raise OSError(f"no CUDA runtime found for the b200 backend: {err}")


_lib = _load_lib()
_rt = _load_cudart()
_P, _I, _D, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
_DT = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int8): 2}

_lib.xnc_pack_plane.argtypes = [_P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P]
_lib.xnc_xnor_accumulate.argtypes = [_P, _I, _I, _I, _P, _U64, _I, _I, _I, _I, _P, _I, _I, _P]
_lib.xnc_box_mean.argtypes = [_P, _I, _I, _I, _I, _I, _D, _P, _P, _P]
_lib.xnc_scale_rows.argtypes = [_P, _I, _I, _I, _I, _I, _P, _P]
_lib.xnc_scale_join.argtypes = [_P, _I, _P, _I, _D, _D, _I, _I, _P, _P]
_lib.xnc_xnor_reconstruct.argtypes = [_P, _U64, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I,
                                      _D, _D, _P, _P]
_lib.xnc_vanilla_conv.argtypes = [_P, _I, _I, _I, _I, _P, _I, _I, _P, _P]
_lib.xnc_strerror.argtypes = [_I]
_lib.xnc_strerror.restype = ctypes.c_char_p
_rt.cudaMalloc.argtypes = [ctypes.POINTER(_P), ctypes.c_size_t]
_rt.cudaFree.argtypes = [_P]
_rt.cudaMemcpy.argtypes = [_P, _P, ctypes.c_size_t, _I]
_rt.cudaDeviceSynchronize.argtypes = []
_H2D, _D2H = 1, 2


def _rt_ok(rc, what):
    if rc:
        raise RuntimeError(f"b200 backend: {what} failed (cudaError {rc})")


def _ok(rc, what):
    if rc:
        raise RuntimeError(f"b200 backend: {what}: {_lib.xnc_strerror(rc).decode()}")


def _contig(a, name, dtypes):
    """The Cython boundary's typed `::1` memoryview check."""
    if not isinstance(a, np.ndarray) or not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous")
    if a.dtype not in dtypes:
        raise ValueError(f"{name}: buffer dtype mismatch, got {a.dtype}")
    return a


class _Dev:
    """cudaMalloc'd mirror of a host array: H2D on entry (upload=True), D2H on demand."""

    def __init__(self, host, upload=True):
        self.host = host
        self.ptr = _P()
        _rt_ok(_rt.cudaMalloc(ctypes.byref(self.ptr), max(host.nbytes, 1)), "cudaMalloc")
        if upload and host.nbytes:
            _rt_ok(_rt.cudaMemcpy(self.ptr, host.ctypes.data, host.nbytes, _H2D), "cudaMemcpy H2D")

    def download(self):
        if self.host.nbytes:
            _rt_ok(_rt.cudaMemcpy(self.host.ctypes.data, self.ptr, self.host.nbytes, _D2H), "cudaMemcpy D2H")

    def __del__(self):
        if self.ptr:
            _rt.cudaFree(self.ptr)
            self.ptr = _P()


_F = (np.dtype(np.float32), np.dtype(np.float64))
_U = (np.dtype(np.uint64),)
_I32 = (np.dtype(np.int32),)


def pack_plane(plane, tiles_y, tiles_x, tile_h, tile_w, stride_y, stride_x, out_words, threads) -> None:
    """_kernels_cy.pyx:42-73 -> xnc_pack_plane."""
    _contig(plane, "plane", tuple(_DT))
    _contig(out_words, "out_words", _U)
    p, o = _Dev(plane), _Dev(out_words, upload=False)
    _ok(_lib.xnc_pack_plane(p.ptr, _DT[plane.dtype], plane.shape[0], plane.shape[1], tiles_y, tiles_x,
                            tile_h, tile_w, stride_y, stride_x, o.ptr, None), "pack_plane")
    o.download()


def xnor_accumulate(words, weight_words, mask, tile_w, stride_y, stride_x, k_area, out, threads) -> None:
    """_kernels_cy.pyx:76-104 -> xnc_xnor_accumulate."""
    _contig(words, "words", _U)
    _contig(weight_words, "weight_words", _U)
    _contig(out, "out", _I32)
    w, ww, o = _Dev(words), _Dev(weight_words), _Dev(out, upload=False)
    c, ty, tx = words.shape
    _ok(_lib.xnc_xnor_accumulate(w.ptr, c, ty, tx, ww.ptr, int(mask), tile_w, stride_y, stride_x, k_area,
                                 o.ptr, out.shape[0], out.shape[1], None), "xnor_accumulate")
    o.download()


def box_mean(a, kh, kw, scale, tmp, out, threads) -> None:
    """_kernels_cy.pyx:126-148 -> xnc_box_mean (tmp and out filled)."""
    _contig(a, "a", _F)
    _contig(tmp, "tmp", (a.dtype,))
    _contig(out, "out", (a.dtype,))
    d, t, o = _Dev(a), _Dev(tmp, upload=False), _Dev(out, upload=False)
    _ok(_lib.xnc_box_mean(d.ptr, _DT[a.dtype], a.shape[0], a.shape[1], kh, kw, scale, t.ptr, o.ptr, None),
        "box_mean")
    t.download()
    o.download()


def scale_rows(padded, kw, tmp, threads) -> None:
    """_kernels_cy.pyx:151-186 -> xnc_scale_rows."""
    _contig(padded, "padded", _F)
    _contig(tmp, "tmp", (padded.dtype,))
    p, t = _Dev(padded), _Dev(tmp, upload=False)
    c, h, w = padded.shape
    _ok(_lib.xnc_scale_rows(p.ptr, _DT[padded.dtype], c, h, w, kw, t.ptr, None), "scale_rows")
    t.download()


def scale_join(tmp, ints, kh, scale, weight_scale, out, threads) -> None:
    """_kernels_cy.pyx:189-204 -> xnc_scale_join."""
    _contig(tmp, "tmp", _F)
    _contig(ints, "ints", _I32)
    _contig(out, "out", (tmp.dtype,))
    t, i, o = _Dev(tmp), _Dev(ints), _Dev(out, upload=False)
    _ok(_lib.xnc_scale_join(t.ptr, _DT[tmp.dtype], i.ptr, kh, scale, weight_scale, out.shape[0],
                            out.shape[1], o.ptr, None), "scale_join")
    o.download()


def xnor_reconstruct(weight_words, mask, tile_h, tile_w, stride_y, stride_x, k_area, padded, kh, kw,
                     scale, weight_scale, out, threads) -> None:
    """_kernels_cy.pyx:242-354 -> xnc_xnor_reconstruct (race-free for every kh)."""
    _contig(weight_words, "weight_words", _U)
    _contig(padded, "padded", _F)
    _contig(out, "out", (padded.dtype,))
    ww, p, o = _Dev(weight_words), _Dev(padded), _Dev(out, upload=False)
    c, ph, pw = padded.shape
    _ok(_lib.xnc_xnor_reconstruct(ww.ptr, int(mask), tile_h, tile_w, stride_y, stride_x, k_area, p.ptr,
                                  _DT[padded.dtype], c, ph, pw, kh, kw, scale, weight_scale, o.ptr, None),
        "xnor_reconstruct")
    _rt_ok(_rt.cudaDeviceSynchronize(), "cudaDeviceSynchronize")
    o.download()


def vanilla_conv(padded, weights, out, threads) -> None:
    """_kernels_cy.pyx:107-123 -> xnc_vanilla_conv: the bench's float baseline,
    (ch, ky, kx) order, one rounding per multiply and per add."""
    _contig(padded, "padded", _F)
    _contig(weights, "weights", (padded.dtype,))
    _contig(out, "out", (padded.dtype,))
    p, w, o = _Dev(padded), _Dev(weights), _Dev(out, upload=False)
    c, ph, pw = padded.shape
    _ok(_lib.xnc_vanilla_conv(p.ptr, _DT[padded.dtype], c, ph, pw, w.ptr, weights.shape[1], weights.shape[2],
                              o.ptr, None), "vanilla_conv")
    o.download()
