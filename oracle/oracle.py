"""Python face of the CPU oracle -- TEST INFRASTRUCTURE ONLY (see __init__.py).

Three tiers, each citing the reference it restates (/root/reference/pkg/src/xnorconv):

1. ``liboracle.so`` (xnor_oracle.c): tile pack, masked XNOR decode, float32
   scale map in the reference's exact op order, the per-(image, filter) layer.
2. numpy restatements for small cases: ``sign_conv2d_int`` (reference.py:58-90,
   padding = +1), ``alpha`` (binarize.py:65-75), ``channel_abs_mean``.
3. ``RefKernels``: the reference's own compiled Cython kernels
   (oracle/_ref, built by build_ref.sh) driven the way ConvWorkspace.run drives
   them (pipeline.py:124-151) -- the CPU baseline and a second checker.
"""
from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile liboracle.so (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return os.path.join(HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        src = os.path.join(HERE, "xnor_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(path)
        c_long, c_int = ctypes.c_long, ctypes.c_int
        L.xo_pack_plane_f32.argtypes = [_f32p, c_long, c_long, c_int, c_int, c_int, c_int, c_int, c_int, _u64p]
        L.xo_pack_plane_i8.argtypes = [_i8p, c_long, c_long, c_int, c_int, c_int, c_int, c_int, c_int, _u64p]
        L.xo_xnor_accumulate.argtypes = [_u64p, c_long, c_long, c_long, _u64p, ctypes.c_uint64, c_int,
                                         c_int, c_int, c_int, _i32p, c_long, c_long]
        L.xo_build_filter.argtypes = [_f64p, c_int, c_int, c_int, c_int, _u64p,
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)]
        L.xo_scale_map_f32.argtypes = [_f32p, c_int, c_int, c_int, c_int, c_int, c_int,
                                       ctypes.c_void_p, _f32p]
        L.xo_channel_abs_mean_f64.argtypes = [_f64p, c_int, c_int, c_int, _f64p]
        L.xo_box_mean_f64.argtypes = [_f64p, c_long, c_long, c_int, c_int, ctypes.c_double, _f64p]
        L.xo_conv_pairs.argtypes = [_f32p, _f32p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                    c_int, c_int, _i32p, c_int, _i32p, c_int, _f32p, ctypes.c_void_p]
        L.xo_conv_pairs.restype = c_int
        _LIB = L
    return _LIB


# --------------------------------------------------------------------------- geometry
TILE_SHAPES = {64: (8, 8), 32: (8, 4)}  # pack.py:30


def out_dims(h, w, kh, kw, pad):
    return h + 2 * pad - kh + 1, w + 2 * pad - kw + 1


def grid_shape(word_bits, kh, kw, out_h, out_w):
    th, tw = TILE_SHAPES[word_bits]
    sy, sx = th - kh + 1, tw - kw + 1
    return -(-out_h // sy), -(-out_w // sx)


# --------------------------------------------------------------------------- tier 1
def pack_plane(plane, word_bits, kh, kw):
    """Reference tile words of an (already padded) plane (pack.py:105-120)."""
    plane = np.ascontiguousarray(plane)
    th, tw = TILE_SHAPES[word_bits]
    h, w = plane.shape
    ty, tx = grid_shape(word_bits, kh, kw, h - kh + 1, w - kw + 1)
    out = np.zeros((ty, tx), dtype=np.uint64)
    if plane.dtype == np.int8:
        lib().xo_pack_plane_i8(plane, h, w, ty, tx, th, tw, th - kh + 1, tw - kw + 1, out)
    else:
        lib().xo_pack_plane_f32(plane.astype(np.float32), h, w, ty, tx, th, tw, th - kh + 1, tw - kw + 1, out)
    return out


def build_filter(w_ckk, word_bits=64):
    """(weight_words u64[C], base_mask int, alpha float) (engine.py:102-120)."""
    w = np.ascontiguousarray(w_ckk, dtype=np.float64)
    c, kh, kw = w.shape
    tw = TILE_SHAPES[word_bits][1]
    words = np.zeros(c, dtype=np.uint64)
    mask = ctypes.c_uint64()
    alpha = ctypes.c_double()
    lib().xo_build_filter(w, c, kh, kw, tw, words, ctypes.byref(mask), ctypes.byref(alpha))
    return words, int(mask.value), float(alpha.value)


def xnor_accumulate(words, weight_words, mask, word_bits, kh, kw, out_h, out_w):
    th, tw = TILE_SHAPES[word_bits]
    words = np.ascontiguousarray(words, dtype=np.uint64)
    c, ty, tx = words.shape
    out = np.zeros((out_h, out_w), dtype=np.int32)
    lib().xo_xnor_accumulate(words, c, ty, tx, np.ascontiguousarray(weight_words, dtype=np.uint64),
                             mask, tw, th - kh + 1, tw - kw + 1, kh * kw, out, out_h, out_w)
    return out


def scale_map_f32(x_chw, kh, kw, pad):
    """(A f32 [H,W], K f32 [H',W']) in the pipeline's float32 order."""
    x = np.ascontiguousarray(x_chw, dtype=np.float32)
    c, h, w = x.shape
    oh, ow = out_dims(h, w, kh, kw, pad)
    A = np.zeros((h, w), dtype=np.float32)
    K = np.zeros((oh, ow), dtype=np.float32)
    lib().xo_scale_map_f32(x, c, h, w, kh, kw, pad, A.ctypes.data, K)
    return A, K


def channel_abs_mean_f64(x_chw):
    x = np.ascontiguousarray(x_chw, dtype=np.float64)
    c, h, w = x.shape
    out = np.zeros((h, w), dtype=np.float64)
    lib().xo_channel_abs_mean_f64(x, c, h, w, out)
    return out


def box_mean_f64(padded, kh, kw):
    a = np.ascontiguousarray(padded, dtype=np.float64)
    h, w = a.shape
    out = np.zeros((h - kh + 1, w - kw + 1), dtype=np.float64)
    lib().xo_box_mean_f64(a, h, w, kh, kw, 1.0 / (kh * kw), out)
    return out


def conv_layer(x, w, pad, n_idx=None, o_idx=None, word_bits=64, want_ints=False):
    """out[i, j] == reference xnor_conv(x[n_idx[i]], w[o_idx[j]], pad) (f32), and ints."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    N, C, H, W = x.shape
    O, C2, kh, kw = w.shape
    assert C == C2
    n_idx = np.arange(N, dtype=np.int32) if n_idx is None else np.asarray(n_idx, dtype=np.int32)
    o_idx = np.arange(O, dtype=np.int32) if o_idx is None else np.asarray(o_idx, dtype=np.int32)
    oh, ow = out_dims(H, W, kh, kw, pad)
    out = np.zeros((len(n_idx), len(o_idx), oh, ow), dtype=np.float32)
    ints = np.zeros(out.shape, dtype=np.int32) if want_ints else None
    rc = lib().xo_conv_pairs(x, w, N, C, H, W, O, kh, kw, pad, word_bits,
                             np.ascontiguousarray(n_idx), len(n_idx), np.ascontiguousarray(o_idx), len(o_idx),
                             out, ints.ctypes.data if ints is not None else None)
    if rc != 0:
        raise ValueError(f"oracle rejected the geometry (rc={rc})")
    return (out, ints) if want_ints else out


# --------------------------------------------------------------------------- tier 2
def signs(a):
    """+1 / -1 int8 with sign(0) = sign(-0.0) = +1 (binarize.py:56-57)."""
    return np.where(np.asarray(a) >= 0, 1, -1).astype(np.int8)


def sign_conv2d_int(x_chw, w_ckk, pad):
    """Integer cross-correlation of sign planes, padding pixels = +1
    (reference.py:58-90), vectorised over output pixels."""
    xs = signs(x_chw).astype(np.int32)
    ws = signs(w_ckk).astype(np.int32)
    c, h, w = xs.shape
    _, kh, kw = ws.shape
    oh, ow = out_dims(h, w, kh, kw, pad)
    p = np.ones((c, h + 2 * pad, w + 2 * pad), dtype=np.int32)
    p[:, pad:pad + h, pad:pad + w] = xs
    out = np.zeros((oh, ow), dtype=np.int64)
    for ch in range(c):
        for ky in range(kh):
            for kx in range(kw):
                out += p[ch, ky:ky + oh, kx:kx + ow] * ws[ch, ky, kx]
    return out.astype(np.int32)


def alpha(w_ckk):
    """(sum |w| in index order, sequential float64) / n (binarize.py:72-75)."""
    total = 0.0
    flat = np.asarray(w_ckk, dtype=np.float64).ravel().tolist()
    for v in flat:
        total += abs(v)
    return total / len(flat)


def f32_exact(rng, shape, lo=-1.0, hi=1.0):
    """float32-exact data (tests/helpers.py:16-18 of the reference)."""
    return rng.uniform(lo, hi, shape).astype(np.float32)


# --------------------------------------------------------------------------- tier 3
class RefKernels:
    """The reference's compiled kernels (oracle/_ref/_kernels_cy*.so)."""

    def __init__(self):
        paths = glob.glob(os.path.join(HERE, "_ref", "_kernels_cy*.so"))
        if not paths:
            raise FileNotFoundError("oracle/_ref/_kernels_cy*.so not built (oracle/build_ref.sh)")
        spec = importlib.util.spec_from_file_location("xnorconv._kernels_cy", paths[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        self.mod = mod
        self.path = paths[0]

    @staticmethod
    def available() -> bool:
        return bool(glob.glob(os.path.join(HERE, "_ref", "_kernels_cy*.so")))

    def workspace(self, x_chw, pad, kh, kw, word_bits=64):
        """The state ConvWorkspace.__init__/load_input builds (pipeline.py:43-93)."""
        x = np.asarray(x_chw, dtype=np.float32)
        c, h, w = x.shape
        padded = np.zeros((c, h + 2 * pad, w + 2 * pad), dtype=np.float32)
        padded[:, pad:pad + h, pad:pad + w] = x
        oh, ow = out_dims(h, w, kh, kw, pad)
        return padded, np.empty((oh, ow), dtype=np.float32)

    def run(self, padded, out, filt, kh, kw, threads=1, word_bits=64):
        """One fused ConvWorkspace.run() (pipeline.py:142-150 -> _kernels_cy.pyx:242)."""
        words, mask, a = filt
        th, tw = TILE_SHAPES[word_bits]
        self.mod.xnor_reconstruct(words, mask, th, tw, th - kh + 1, tw - kw + 1, kh * kw, padded,
                                  kh, kw, 1.0 / (kh * kw), a, out, threads)
        return out

    def conv_layer(self, x, w, pad, threads=1, word_bits=64):
        x = np.asarray(x, dtype=np.float32)
        w = np.asarray(w, dtype=np.float32)
        N, C, H, W = x.shape
        O, _, kh, kw = w.shape
        filters = [build_filter(w[o], word_bits) for o in range(O)]
        oh, ow = out_dims(H, W, kh, kw, pad)
        res = np.zeros((N, O, oh, ow), dtype=np.float32)
        for n in range(N):
            padded, out = self.workspace(x[n], pad, kh, kw, word_bits)
            for o in range(O):
                res[n, o] = self.run(padded, out, filters[o], kh, kw, threads, word_bits)
        return res
