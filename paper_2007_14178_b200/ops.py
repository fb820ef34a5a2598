"""Device-tensor operators over libxnorb200.so (torch is plumbing: memory and
streams; all arithmetic runs in the sm_100a kernels).

Every function takes CUDA tensors, allocates its outputs with torch on the
same device, and enqueues on torch's current stream.  Shapes follow the
layouts documented in include/xnorb200.h.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import XNC_ENOTSUP, check, lib

ABI_VERSION = 1


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _need_cuda(t: torch.Tensor, name: str, dtype: torch.dtype, channels_last_ok: bool = False) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the B200 path has no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not (t.is_contiguous() or (channels_last_ok and t.is_contiguous(memory_format=torch.channels_last))):
        raise ValueError(f"{name} must be contiguous")


def out_dims(h: int, w: int, kh: int, kw: int, pad: int) -> tuple[int, int]:
    """(H', W') of a stride-1 conv with zero padding `pad` (pipeline.py:62-66)."""
    return h + 2 * pad - kh + 1, w + 2 * pad - kw + 1


def words(c: int) -> int:
    return (c + 31) // 32


def _affine(aff, n: int, device, what: str):
    """(scale, shift) f32 [n] device tensors, or (None, None)."""
    if aff is None:
        return None, None
    sc, sh = aff
    for t, nm in ((sc, "scale"), (sh, "shift")):
        _need_cuda(t, f"{what} {nm}", torch.float32)
        if t.numel() != n or not t.is_contiguous():
            raise ValueError(f"{what} {nm} must be a contiguous f32 vector of {n}")
    return sc, sh


def pool_dims(H: int, W: int, in_pool) -> tuple[int, int]:
    """Spatial dims after the optional input max-pool (kernel, stride), no padding."""
    if in_pool is None:
        return H, W
    k, s = in_pool
    if k < 1 or s < 1 or H < k or W < k:
        raise ValueError(f"pool {in_pool} does not fit a {H}x{W} input")
    return (H - k) // s + 1, (W - k) // s + 1


def _channels_last(x: torch.Tensor) -> bool:
    return not x.is_contiguous() and x.is_contiguous(memory_format=torch.channels_last)


def max_pool(x: torch.Tensor, k: int, s: int, relu: bool = False,
             bias: torch.Tensor | None = None) -> torch.Tensor:
    """Max-pool k x k / stride s, no padding (torch.max_pool2d values), on the
    device; bias f32 [C]: pool of x + bias (a conv's bias, added after the max:
    exact); relu=True: torch.relu first, in the same pass.  A channels-last x gives
    a channels-last result."""
    _need_cuda(x, "x", torch.float32, channels_last_ok=True)
    nhwc = _channels_last(x)
    if not nhwc:
        x = x.contiguous()
    N, C, H, W = x.shape
    Ho, Wo = pool_dims(H, W, (k, s))
    fmt = torch.channels_last if nhwc else torch.contiguous_format
    out = torch.empty((N, C, Ho, Wo), dtype=torch.float32, device=x.device, memory_format=fmt)
    if bias is not None:
        _need_cuda(bias, "bias", torch.float32)
        if bias.numel() != C:
            raise ValueError(f"bias must have {C} entries")
    check(lib().xnc_max_pool(x.data_ptr(), N, C, H, W, int(k), int(s), int(bool(relu)), int(nhwc),
                             _ptr(bias), out.data_ptr(), _stream(x.device)), "xnc_max_pool")
    return out


def pad_space_to_depth(x: torch.Tensor, pad: int, r: int, channels_last: bool = False) -> torch.Tensor:
    """F.pixel_unshuffle(F.pad(x, (pad,) * 4), r) in one device pass (x NCHW);
    channels_last=True stores the result channels-last."""
    _need_cuda(x, "x", torch.float32)
    x = x.contiguous()
    N, C, H, W = x.shape
    if (H + 2 * pad) % r or (W + 2 * pad) % r:
        raise ValueError(f"padded {H}x{W} input is not a multiple of {r}")
    fmt = torch.channels_last if channels_last else torch.contiguous_format
    out = torch.empty((N, C * r * r, (H + 2 * pad) // r, (W + 2 * pad) // r), dtype=torch.float32,
                      device=x.device, memory_format=fmt)
    check(lib().xnc_pad_space_to_depth(x.data_ptr(), N, C, H, W, int(pad), int(r), int(bool(channels_last)),
                                       out.data_ptr(), _stream(x.device)), "xnc_pad_space_to_depth")
    return out


def conv1_pack_weights(w: torch.Tensor) -> torch.Tensor:
    """XNOR-Net AlexNet conv1 weights f32 [96, 3, 11, 11] -> the tcgen05 TF32 kernel's
    B operand (27 (c, tap) blocks x 96 filters x 16 space-to-depth phases, TF32-rounded)."""
    _need_cuda(w, "w", torch.float32)
    if tuple(w.shape) != (96, 3, 11, 11):
        raise ValueError(f"conv1 weights must be [96, 3, 11, 11], got {tuple(w.shape)}")
    wq = torch.empty(lib().xnc_conv1_weight_bytes() // 4, dtype=torch.float32, device=w.device)
    check(lib().xnc_conv1_pack_weights(w.contiguous().data_ptr(), wq.data_ptr(), _stream(w.device)),
          "xnc_conv1_pack_weights")
    return wq


def conv1_forward(x: torch.Tensor, wq: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """conv1 (11x11, stride 4, pad 2, no bias) of x f32 [N, 3, 224, 224] on the tcgen05
    TF32 kernel -> f32 [N, 96, 55, 55] stored channels-last (the layout the network's
    bias + ReLU + pool pass and conv2's K1 read)."""
    _need_cuda(x, "x", torch.float32)
    x = x.contiguous()
    if x.shape[1:] != (3, 224, 224):
        raise ValueError(f"conv1 input must be [N, 3, 224, 224], got {tuple(x.shape)}")
    N = x.shape[0]
    if out is None:
        out = torch.empty((N, 96, 55, 55), dtype=torch.float32, device=x.device,
                          memory_format=torch.channels_last)
    elif (tuple(out.shape) != (N, 96, 55, 55) or out.dtype != torch.float32 or out.device != x.device
          or not out.is_contiguous(memory_format=torch.channels_last)):
        raise ValueError("out must be a channels-last f32 [N, 96, 55, 55] tensor on x's device")
    check(lib().xnc_conv1_forward(x.data_ptr(), N, wq.data_ptr(), out.data_ptr(), _stream(x.device)),
          "xnc_conv1_forward")
    return out


def pack_input(x: torch.Tensor, want_A: bool = True, in_affine=None, in_pool=None, pool_relu: bool = False,
               pool_bias: torch.Tensor | None = None):
    """K1: x f32 [N,C,H,W] -> (bits i32 [N,H,W,Cw] (u32 payload), A f32 [N,H,W]).

    in_affine = (scale, shift) f32 [C]: binarize and average x*scale + shift (one
    rounding per op) instead of x -- a folded batch norm before the sign.
    in_pool = (kernel, stride): x is the pre-pool tensor, max-pooled first (no
    padding; xnc_max_pool, with its relu / bias = pool_relu / pool_bias) --
    XNOR-Net's pool -> BN -> sign; bits / A then have the pooled spatial shape."""
    _need_cuda(x, "x", torch.float32, channels_last_ok=True)
    if pool_bias is not None:
        _need_cuda(pool_bias, "pool_bias", torch.float32)
        if pool_bias.numel() != x.shape[1]:
            raise ValueError(f"pool_bias must have {x.shape[1]} entries")
    if in_pool is not None and _channels_last(x):
        # pool (+ bias, ReLU) fused into K1 on the channels-last map (xnc_pack_input_pool_nhwc)
        N, C, Hin, Win = x.shape
        H, W = pool_dims(Hin, Win, in_pool)
        bits = torch.empty((N, H, W, words(C)), dtype=torch.int32, device=x.device)
        A = torch.empty((N, H, W), dtype=torch.float32, device=x.device) if want_A else None
        sc, sh = _affine(in_affine, C, x.device, "in_affine")
        rc = lib().xnc_pack_input_pool_nhwc(x.data_ptr(), N, C, Hin, Win, int(in_pool[0]), int(in_pool[1]),
                                            int(bool(pool_relu)), _ptr(pool_bias), _ptr(sc), _ptr(sh),
                                            bits.data_ptr(), _ptr(A), _stream(x.device))
        if rc == 0:
            return bits, A
        if rc != XNC_ENOTSUP:
            check(rc, "xnc_pack_input_pool_nhwc")
    elif in_pool is not None and not pool_relu and pool_bias is None:
        # pool fused into K1 (xnc_pack_input_pool) when the pooled map takes its path
        xc = x.contiguous()
        N, C, Hin, Win = xc.shape
        H, W = pool_dims(Hin, Win, in_pool)
        bits = torch.empty((N, H, W, words(C)), dtype=torch.int32, device=x.device)
        A = torch.empty((N, H, W), dtype=torch.float32, device=x.device) if want_A else None
        sc, sh = _affine(in_affine, C, x.device, "in_affine")
        rc = lib().xnc_pack_input_pool(xc.data_ptr(), N, C, Hin, Win, int(in_pool[0]), int(in_pool[1]), _ptr(sc),
                                       _ptr(sh), bits.data_ptr(), _ptr(A), _stream(x.device))
        if rc == 0:
            return bits, A
        if rc != XNC_ENOTSUP:
            check(rc, "xnc_pack_input_pool")
    if in_pool is not None:
        x = max_pool(x, *in_pool, relu=pool_relu, bias=pool_bias)
    N, C, H, W = x.shape
    bits = torch.empty((N, H, W, words(C)), dtype=torch.int32, device=x.device)
    A = torch.empty((N, H, W), dtype=torch.float32, device=x.device) if want_A else None
    sc, sh = _affine(in_affine, C, x.device, "in_affine")
    if _channels_last(x):  # channels-last maps (the network's front end) are packed in place
        check(lib().xnc_pack_input_nhwc(x.data_ptr(), N, C, H, W, _ptr(sc), _ptr(sh), bits.data_ptr(), _ptr(A),
                                        _stream(x.device)), "xnc_pack_input_nhwc")
    elif sc is None:
        check(lib().xnc_pack_input(x.data_ptr(), N, C, H, W, bits.data_ptr(), _ptr(A), _stream(x.device)),
              "xnc_pack_input")
    else:
        check(lib().xnc_pack_input_affine(x.data_ptr(), N, C, H, W, sc.data_ptr(), sh.data_ptr(),
                                          bits.data_ptr(), _ptr(A), _stream(x.device)), "xnc_pack_input_affine")
    return bits, A


def pack_input_into(x: torch.Tensor, bits: torch.Tensor, A: torch.Tensor | None) -> None:
    """K1 into preallocated buffers."""
    N, C, H, W = x.shape
    check(lib().xnc_pack_input(x.data_ptr(), N, C, H, W, bits.data_ptr(), _ptr(A), _stream(x.device)),
          "xnc_pack_input")


@dataclass
class PackedFilters:
    """Binarized filter bank on the device (build_filter for every filter)."""

    wbits: torch.Tensor    # i32 [Cw, kh, kw, O]
    alpha: torch.Tensor    # f32 [O]
    alpha64: torch.Tensor  # f64 [O] (BinaryFilter.scale)
    O: int
    C: int
    kh: int
    kw: int
    wq: torch.Tensor | None = None   # u8 tensor-core layout (xnc_pack_weights_umma)
    sw: torch.Tensor | None = None   # i32 [O] sum of each filter's signs


def attach_umma_weights(filt: PackedFilters, w: torch.Tensor) -> PackedFilters:
    """Add the tcgen05 (kind::i8) weight layout to a PackedFilters (f32 or f64 w)."""
    if w.dtype not in (torch.float32, torch.float64):
        raise TypeError("weights must be float32 or float64")
    _need_cuda(w, "w", w.dtype)
    O, C, kh, kw = w.shape
    nbytes = int(lib().xnc_umma_weight_bytes(O, C, kh, kw))
    filt.wq = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=w.device)
    filt.sw = torch.empty(O, dtype=torch.int32, device=w.device)
    check(lib().xnc_pack_weights_umma(w.data_ptr(), 0 if w.dtype == torch.float32 else 1, O, C, kh, kw,
                                      filt.wq.data_ptr(), filt.sw.data_ptr(), _stream(w.device)),
          "xnc_pack_weights_umma")
    return filt


def umma_supported(N: int, C: int, H: int, W: int, O: int, kh: int, kw: int, pad: int) -> bool:
    return bool(lib().xnc_umma_supported(N, C, H, W, O, kh, kw, pad))


def pack_weights(w: torch.Tensor) -> PackedFilters:
    """w f32 [O,C,kh,kw] -> PackedFilters (engine.py:102-120, binarize.py:65-75)."""
    _need_cuda(w, "w", torch.float32)
    O, C, kh, kw = w.shape
    wbits = torch.empty((words(C), kh, kw, O), dtype=torch.int32, device=w.device)
    alpha = torch.empty(O, dtype=torch.float32, device=w.device)
    alpha64 = torch.empty(O, dtype=torch.float64, device=w.device)
    check(lib().xnc_pack_weights(w.data_ptr(), O, C, kh, kw, wbits.data_ptr(), alpha.data_ptr(),
                                 alpha64.data_ptr(), _stream(w.device)), "xnc_pack_weights")
    return PackedFilters(wbits, alpha, alpha64, O, C, kh, kw)


def pack_weights_f64(w: torch.Tensor) -> PackedFilters:
    """Same from float64 weights (the reference's Tensor3 values, unrounded)."""
    _need_cuda(w, "w", torch.float64)
    O, C, kh, kw = w.shape
    wbits = torch.empty((words(C), kh, kw, O), dtype=torch.int32, device=w.device)
    alpha = torch.empty(O, dtype=torch.float32, device=w.device)
    alpha64 = torch.empty(O, dtype=torch.float64, device=w.device)
    check(lib().xnc_pack_weights_f64(w.data_ptr(), O, C, kh, kw, wbits.data_ptr(), alpha.data_ptr(),
                                     alpha64.data_ptr(), _stream(w.device)), "xnc_pack_weights_f64")
    return PackedFilters(wbits, alpha, alpha64, O, C, kh, kw)


def scale_map_into(A: torch.Tensor, kh: int, kw: int, pad: int, K: torch.Tensor) -> None:
    N, H, W = A.shape
    check(lib().xnc_scale_map(A.data_ptr(), N, H, W, kh, kw, pad, K.data_ptr(), _stream(A.device)),
          "xnc_scale_map")


def scale_map(A: torch.Tensor, kh: int, kw: int, pad: int) -> torch.Tensor:
    """K2: A f32 [N,H,W] -> K f32 [N,H',W'] (float32 reconstruct order)."""
    _need_cuda(A, "A", torch.float32)
    N, H, W = A.shape
    oh, ow = out_dims(H, W, kh, kw, pad)
    K = torch.empty((N, oh, ow), dtype=torch.float32, device=A.device)
    check(lib().xnc_scale_map(A.data_ptr(), N, H, W, kh, kw, pad, K.data_ptr(), _stream(A.device)),
          "xnc_scale_map")
    return K


VARIANTS = {"popc": 0, "b1mma": 1, "umma": 2}


@dataclass
class PackedInput:
    """A binary layer's input in K1 form: bits i32 [N,H,W,Cw] (u32 payload) and
    A f32 [N,H,W] for C channels -- what pack_input returns, or what a previous
    layer's sign-emitting epilogue wrote (xnor_conv_emit)."""

    bits: torch.Tensor
    A: torch.Tensor
    C: int

    @property
    def shape(self) -> tuple[int, int, int, int]:
        N, H, W, _ = self.bits.shape
        return N, self.C, H, W


def umma_emit_supported(N: int, C: int, H: int, W: int, O: int, kh: int, kw: int, pad: int) -> bool:
    return bool(lib().xnc_umma_emit_supported(N, C, H, W, O, kh, kw, pad))


def xnor_conv_emit(bits: torch.Tensor, filt: PackedFilters, K: torch.Tensor, pad: int,
                   out_affine=None) -> PackedInput:
    """tcgen05 conv whose epilogue writes the NEXT binary layer's K1 output (sign words
    and A of y' = alpha*K*acc [*scale + shift]) instead of y: bit-identical to
    pack_input(y', ...) without the float map ever reaching HBM."""
    _need_cuda(bits, "bits", torch.int32)
    _need_cuda(K, "K", torch.float32)
    if filt.wq is None:
        raise ValueError("the sign-emitting epilogue runs on the tcgen05 kernel: attach_umma_weights() first")
    N, H, W, Cw = bits.shape
    C = filt.C
    if words(C) != Cw:
        raise ValueError(f"bits hold {Cw} words per pixel; filters have {C} channels")
    if not umma_emit_supported(N, C, H, W, filt.O, filt.kh, filt.kw, pad):
        raise ValueError(f"no tcgen05 sign-emitting plan for N={N} C={C} {H}x{W} O={filt.O} "
                         f"k={filt.kh}x{filt.kw} pad={pad}")
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    dev = bits.device
    nbits = torch.empty((N, oh, ow, words(filt.O)), dtype=torch.int32, device=dev)
    nA = torch.empty((N, oh, ow), dtype=torch.float32, device=dev)
    osc, osh = _affine(out_affine, filt.O, dev, "out_affine")
    check(lib().xnc_xnor_conv_umma_emit(bits.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(), K.data_ptr(),
                                        filt.alpha.data_ptr(), N, C, H, W, filt.O, filt.kh, filt.kw, pad,
                                        _ptr(osc), _ptr(osh), nbits.data_ptr(), nA.data_ptr(), _stream(dev)),
          "xnc_xnor_conv_umma_emit")
    return PackedInput(nbits, nA, filt.O)


def _check_out(t: torch.Tensor | None, name: str, dtype: torch.dtype, shape, device) -> None:
    """A caller-supplied output must be exactly what the kernel writes: a kernel
    told N*O*H'*W' elements of the wrong buffer would write out of bounds."""
    if t is None:
        return
    if not t.is_cuda or t.device != device:
        raise ValueError(f"{name} must be a CUDA tensor on {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def resolve_variant(variant: str, filt: PackedFilters, N: int, C: int, H: int, W: int, pad: int) -> str:
    """'auto' -> 'umma' when the filters carry the tcgen05 layout and its plan fits
    the shape, else 'popc'; explicit variants pass through."""
    if variant == "auto":
        if filt.wq is not None and umma_supported(N, C, H, W, filt.O, filt.kh, filt.kw, pad):
            return "umma"
        return "popc"
    if variant not in ("popc", "b1mma", "umma"):
        raise ValueError(f"unknown variant {variant!r}")
    return variant


# s32 partial-sum buffers of the K split (S slices, every entry written by the split
# kernel), one per (device, stream), allocated once, not per call.
_SPLIT_WS: dict[tuple, torch.Tensor] = {}


def _split_ws(nbytes: int, dev: torch.device) -> torch.Tensor:
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    buf = _SPLIT_WS.get(key)
    if buf is None or buf.numel() * 4 < nbytes:
        buf = torch.empty(nbytes // 4, dtype=torch.int32, device=dev)
        _SPLIT_WS[key] = buf
    return buf


def plane_affine_(y: torch.Tensor, out_affine) -> torch.Tensor:
    """y[n, o] = y[n, o] * scale[o] + shift[o] in place on the device, with the fused
    epilogue's two roundings (xnc_plane_affine)."""
    _need_cuda(y, "y", torch.float32)
    N, O = y.shape[:2]
    plane = y[0, 0].numel() if y.numel() else 0
    osc, osh = _affine(out_affine, O, y.device, "out_affine")
    check(lib().xnc_plane_affine(y.data_ptr(), N, O, plane, osc.data_ptr(), osh.data_ptr(), _stream(y.device)),
          "xnc_plane_affine")
    return y


def xnor_conv(bits: torch.Tensor, filt: PackedFilters, K: torch.Tensor | None, pad: int,
              C: int | None = None, want_y: bool = True, want_acc: bool = False,
              variant: str = "auto", y: torch.Tensor | None = None,
              acc: torch.Tensor | None = None, W: int | None = None, out_affine=None):
    """K3+K4: (y f32 [N,O,H',W'] or None, acc i32 [N,O,H',W'] or None).

    Every variant reads the packed bits `bits` (i32 [N,H,W,Cw], from pack_input).
    variant 'auto' (default) runs the tcgen05 kernel when the filters carry its
    layout (attach_umma_weights) and its plan fits the shape, else popc."""
    C = filt.C if C is None else C
    _need_cuda(bits, "bits", torch.int32)
    N, H, W, Cw = bits.shape
    if words(C) != Cw or filt.C != C:
        raise ValueError(f"bits hold {Cw} words per pixel; filters have {filt.C} channels")
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    if oh < 1 or ow < 1:
        raise ValueError("kernel larger than the padded input")
    dev = bits.device
    variant = resolve_variant(variant, filt, N, C, H, W, pad)
    oshape = (N, filt.O, oh, ow)
    if not want_y:
        y = None
    _check_out(y, "y", torch.float32, oshape, dev)
    _check_out(acc, "acc", torch.int32, oshape, dev)
    if want_y and y is None:
        y = torch.empty(oshape, dtype=torch.float32, device=dev)
    if want_acc and acc is None:
        acc = torch.empty(oshape, dtype=torch.int32, device=dev)
    if want_y:
        if K is None:
            raise ValueError("K map required for the float output")
        _check_out(K, "K", torch.float32, (N, oh, ow), dev)
    if variant == "umma":
        if filt.wq is None:
            raise ValueError("umma variant needs attach_umma_weights() first")
        osc, osh = _affine(out_affine, filt.O, dev, "out_affine")
        # a K split (fully connected shapes) needs an s32 partial-sum buffer (S slices)
        ws_bytes = lib().xnc_umma_split_ws_bytes(N, C, H, W, filt.O, filt.kh, filt.kw, pad)
        split_ws = _split_ws(ws_bytes, dev) if ws_bytes else None
        check(lib().xnc_xnor_conv_umma_ws(bits.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(), _ptr(K),
                                          filt.alpha.data_ptr(), N, C, H, W, filt.O, filt.kh, filt.kw, pad,
                                          _ptr(osc), _ptr(osh), _ptr(split_ws), _ptr(y), _ptr(acc),
                                          _stream(dev)),
              "xnc_xnor_conv_umma")
    else:
        check(lib().xnc_xnor_conv_variant(VARIANTS[variant], bits.data_ptr(), filt.wbits.data_ptr(),
                                          _ptr(K), filt.alpha.data_ptr(), N, C, H, W, filt.O, filt.kh,
                                          filt.kw, pad, _ptr(y), _ptr(acc), _stream(dev)),
              "xnc_xnor_conv")
        if out_affine is not None and y is not None:  # same two roundings as the fused epilogue
            plane_affine_(y, out_affine)
    return y, acc


def xnor_conv_nhwc(bits: torch.Tensor, filt: PackedFilters, K: torch.Tensor, pad: int,
                   out: torch.Tensor | None = None, out_affine=None, emit: bool = False):
    """tcgen05 K3+K4 with y written channels-last: bits i32 [N,H,W,Cw], K f32
    [N,H',W'] -> y f32 [N,O,H',W'] in channels-last memory (the kernel writes
    [N][H'][W'][O] directly, xnc_xnor_conv_umma_nhwc).  Fully connected layers pass
    the batch as a 1 x P image (N = 1, H = 1, W = P) and view y as [P, O].
    emit=True (O % 32 == 0, O <= 4096) also returns the next binary layer's K1 of y,
    (y, bits i32 [P, O/32], A f32 [P]) for the P = N*H'*W' pixels
    (xnc_xnor_conv_umma_nhwc_emit)."""
    _need_cuda(bits, "bits", torch.int32)
    N, H, W, Cw = bits.shape
    if words(filt.C) != Cw or filt.wq is None:
        raise ValueError("xnor_conv_nhwc takes tcgen05 filters matching the bits' channel words")
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    _check_out(K, "K", torch.float32, (N, oh, ow), bits.device)
    if out is None:
        out = torch.empty((N, filt.O, oh, ow), dtype=torch.float32, device=bits.device,
                          memory_format=torch.channels_last)
    elif (tuple(out.shape) != (N, filt.O, oh, ow) or out.dtype != torch.float32 or out.device != bits.device
          or not out.is_contiguous(memory_format=torch.channels_last)):
        raise ValueError(f"out must be a channels-last f32 {(N, filt.O, oh, ow)} tensor on {bits.device}")
    osc, osh = _affine(out_affine, filt.O, bits.device, "out_affine")
    ws_bytes = lib().xnc_umma_split_ws_bytes(N, filt.C, H, W, filt.O, filt.kh, filt.kw, pad)
    split_ws = _split_ws(ws_bytes, bits.device) if ws_bytes else None
    if emit:
        if filt.O % 32 or filt.O > 4096:
            raise ValueError("emit needs O % 32 == 0 and O <= 4096")
        P = N * oh * ow
        nb = torch.empty((P, filt.O // 32), dtype=torch.int32, device=bits.device)
        nA = torch.empty((P,), dtype=torch.float32, device=bits.device)
        check(lib().xnc_xnor_conv_umma_nhwc_emit(bits.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(),
                                                 K.data_ptr(), filt.alpha.data_ptr(), N, filt.C, H, W, filt.O,
                                                 filt.kh, filt.kw, pad, _ptr(osc), _ptr(osh), _ptr(split_ws),
                                                 out.data_ptr(), nb.data_ptr(), nA.data_ptr(), _stream(bits.device)),
              "xnc_xnor_conv_umma_nhwc_emit")
        return out, nb, nA
    check(lib().xnc_xnor_conv_umma_nhwc(bits.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(), K.data_ptr(),
                                        filt.alpha.data_ptr(), N, filt.C, H, W, filt.O, filt.kh, filt.kw, pad,
                                        _ptr(osc), _ptr(osh), _ptr(split_ws), out.data_ptr(), _stream(bits.device)),
          "xnc_xnor_conv_umma_nhwc")
    return out


def _check_layer_bufs(x, filt, pad, workspace, y, acc) -> None:
    N, C, H, W = x.shape
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    if oh < 1 or ow < 1:
        raise ValueError("kernel larger than the padded input")
    _check_out(y, "y", torch.float32, (N, filt.O, oh, ow), x.device)
    _check_out(acc, "acc", torch.int32, (N, filt.O, oh, ow), x.device)
    need = layer_workspace_bytes(N, C, H, W, filt.kh, filt.kw, pad)
    if not workspace.is_cuda or workspace.device != x.device or not workspace.is_contiguous():
        raise ValueError(f"workspace must be a contiguous CUDA tensor on {x.device}")
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace holds {workspace.numel() * workspace.element_size()} bytes; "
                         f"this shape needs {need}")


def layer_workspace_bytes(N: int, C: int, H: int, W: int, kh: int, kw: int, pad: int) -> int:
    return int(lib().xnc_layer_workspace_bytes(N, C, H, W, kh, kw, pad))


def layer_forward(x: torch.Tensor, filt: PackedFilters, pad: int, workspace: torch.Tensor,
                  y: torch.Tensor | None = None, acc: torch.Tensor | None = None):
    """K1 -> K2 -> K3+K4 in one C-ABI call (xnc_layer_forward)."""
    _need_cuda(x, "x", torch.float32)
    N, C, H, W = x.shape
    if C != filt.C:
        raise ValueError(f"{C} input channels vs {filt.C} filter channels")
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    _check_layer_bufs(x, filt, pad, workspace, y, acc)
    if y is None:
        y = torch.empty((N, filt.O, oh, ow), dtype=torch.float32, device=x.device)
    check(lib().xnc_layer_forward(x.data_ptr(), filt.wbits.data_ptr(), filt.alpha.data_ptr(), N, C,
                                  H, W, filt.O, filt.kh, filt.kw, pad, workspace.data_ptr(), _ptr(y),
                                  _ptr(acc), _stream(x.device)), "xnc_layer_forward")
    return y


def layer_forward_umma(x: torch.Tensor, filt: PackedFilters, pad: int, workspace: torch.Tensor,
                       y: torch.Tensor | None = None, acc: torch.Tensor | None = None):
    """K1 -> K2 -> tcgen05 K3+K4 in one C-ABI call (xnc_layer_forward_umma)."""
    _need_cuda(x, "x", torch.float32)
    N, C, H, W = x.shape
    if C != filt.C:
        raise ValueError(f"{C} input channels vs {filt.C} filter channels")
    if filt.wq is None:
        raise ValueError("layer_forward_umma needs attach_umma_weights() first")
    oh, ow = out_dims(H, W, filt.kh, filt.kw, pad)
    _check_layer_bufs(x, filt, pad, workspace, y, acc)
    if y is None:
        y = torch.empty((N, filt.O, oh, ow), dtype=torch.float32, device=x.device)
    check(lib().xnc_layer_forward_umma(x.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(),
                                       filt.alpha.data_ptr(), N, C, H, W, filt.O, filt.kh, filt.kw, pad,
                                       workspace.data_ptr(), _ptr(y), _ptr(acc), _stream(x.device)),
          "xnc_layer_forward_umma")
    return y
