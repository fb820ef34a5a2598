"""Batched binary conv layer: y[n, o] == xnor_conv(x[n], w[o]) for a whole
batch and filter bank in one K1 -> K2 -> K3+K4 pass.

This is the B200 build's generalisation of the reference's one-image x
one-filter unit of work (pipeline.py:176-201): the reference re-binarizes,
re-packs and recomputes K for every (image, filter) pair; here the input is
packed once per image, K once per image, and the filters are packed once per
layer (untimed, like ConvWorkspace.set_weights, pipeline.py:77-83).
"""
from __future__ import annotations

import torch

from . import ops


def default_pad(kernel_h: int, kernel_w: int) -> int:
    """'Same' padding for square odd kernels (pipeline.py:31-37)."""
    if kernel_h != kernel_w or kernel_h % 2 == 0:
        raise ValueError(
            f"no default pad for a {kernel_h}x{kernel_w} kernel; pass pad explicitly")
    return (kernel_h - 1) // 2


class XnorConv2d:
    """Binary conv layer with packed weights resident on one device."""

    def __init__(self, weight: torch.Tensor, pad: int | None = None, variant: str = "popc"):
        if weight.dim() != 4:
            raise ValueError(f"weight must be [O, C, kh, kw], got {tuple(weight.shape)}")
        O, C, kh, kw = weight.shape
        if not (1 <= kh <= 8 and 1 <= kw <= 8):
            raise ValueError(f"kernel {kh}x{kw} does not fit an 8x8 tile")
        self.pad = default_pad(kh, kw) if pad is None else int(pad)
        if self.pad < 0:
            raise ValueError("pad must be >= 0")
        w = weight.detach().to(dtype=torch.float32).contiguous()
        if not w.is_cuda:
            w = w.cuda()
        self.filters = ops.pack_weights(w)
        self.O, self.C, self.kh, self.kw = O, C, kh, kw
        self.variant = variant
        self._ws: dict[tuple, torch.Tensor] = {}

    @property
    def alpha64(self) -> torch.Tensor:
        return self.filters.alpha64

    def out_shape(self, x_shape) -> tuple[int, int, int, int]:
        N, C, H, W = x_shape
        oh, ow = ops.out_dims(H, W, self.kh, self.kw, self.pad)
        if oh < 1 or ow < 1:
            raise ValueError("kernel larger than the padded input")
        return N, self.O, oh, ow

    def workspace(self, x: torch.Tensor) -> torch.Tensor:
        key = (tuple(x.shape), x.device)
        ws = self._ws.get(key)
        if ws is None:
            N, C, H, W = x.shape
            nbytes = ops.layer_workspace_bytes(N, C, H, W, self.kh, self.kw, self.pad)
            ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=x.device)
            self._ws[key] = ws
        return ws

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None,
                want_acc: bool = False):
        """x f32 [N, C, H, W] (CUDA) -> y f32 [N, O, H', W'] (and acc i32 if asked)."""
        if x.dim() != 4 or x.shape[1] != self.C:
            raise ValueError(f"input {tuple(x.shape)} does not match {self.C} filter channels")
        x = x.contiguous()
        self.out_shape(x.shape)
        if self.variant == "popc" and not want_acc:
            return ops.layer_forward(x, self.filters, self.pad, self.workspace(x), y=out)
        bits, A = ops.pack_input(x)
        K = ops.scale_map(A, self.kh, self.kw, self.pad)
        y, acc = ops.xnor_conv(bits, self.filters, K, self.pad, want_acc=want_acc,
                               variant=self.variant, y=out)
        return (y, acc) if want_acc else y

    __call__ = forward


def xnor_conv2d_layer(x: torch.Tensor, weight: torch.Tensor, pad: int | None = None,
                      want_acc: bool = False, variant: str = "popc"):
    """Functional batched layer (packs the weights on every call)."""
    return XnorConv2d(weight, pad, variant).forward(x, want_acc=want_acc)
