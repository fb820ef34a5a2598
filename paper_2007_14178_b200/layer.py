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

    def __init__(self, weight: torch.Tensor, pad: int | None = None, variant: str = "auto",
                 in_affine=None, out_affine=None, in_pool=None, out_channels_last: bool = False):
        """in_affine = (scale, shift) f32 [C]: the layer binarizes x*scale + shift
        (a folded batch norm in front of the sign, computed inside K1); out_affine =
        (scale, shift) f32 [O]: y*scale + shift is written instead of y (the next
        binary layer's batch norm, fused into the conv epilogue); in_pool = (kernel,
        stride): the input is max-pooled first (no padding, xnc_max_pool) --
        forward() then takes the pre-pool tensor.

        variant: 'auto' (default) runs the tcgen05 kernel whenever its plan fits
        the shape (kernel_for), else popc; 'umma' / 'popc' / 'b1mma' force one.
        out_channels_last=True: the tcgen05 epilogue writes y channels-last ([N][H'][W'][O]
        memory, same values) -- for a map that a channels-last pool / K1 reads next."""
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
        self.weight = w  # the float filters (kept for inspection / re-packing)
        self.filters = ops.pack_weights(w)
        if variant in ("umma", "auto"):
            ops.attach_umma_weights(self.filters, w)
        elif variant not in ("popc", "b1mma"):
            raise ValueError(f"unknown variant {variant!r}")
        self.O, self.C, self.kh, self.kw = O, C, kh, kw
        self.variant = variant
        dev = w.device
        self.in_affine = None if in_affine is None else tuple(
            t.detach().to(device=dev, dtype=torch.float32).contiguous() for t in in_affine)
        self.out_affine = None if out_affine is None else tuple(
            t.detach().to(device=dev, dtype=torch.float32).contiguous() for t in out_affine)
        self.in_pool = None if in_pool is None else (int(in_pool[0]), int(in_pool[1]))
        self.out_channels_last = bool(out_channels_last)
        self._ws: dict[tuple, torch.Tensor] = {}

    @property
    def alpha64(self) -> torch.Tensor:
        return self.filters.alpha64

    def conv_in_shape(self, x_shape) -> tuple[int, int, int, int]:
        """The shape the convolution sees: x's, after the optional input pool."""
        N, C, H, W = x_shape
        return (N, C) + ops.pool_dims(H, W, self.in_pool)

    def out_shape(self, x_shape) -> tuple[int, int, int, int]:
        N, C, H, W = self.conv_in_shape(x_shape)
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

    def forward(self, x, out: torch.Tensor | None = None, want_acc: bool = False,
                emit_signs: bool = False):
        """x f32 [N, C, H, W] -> y f32 [N, O, H', W'] (and acc i32 if asked).

        A CUDA x runs on the device and returns a device y.  A host (CPU) x runs
        the pipelined host path (`forward_host`) and returns a host y.  x may also
        be an ops.PackedInput (a previous layer's emitted signs): K1 is skipped.
        emit_signs=True returns the NEXT binary layer's input as an
        ops.PackedInput (sign words + A of y [* out_affine]) instead of y, written
        by the conv epilogue itself (tcgen05 kernel): the float map never
        reaches HBM."""
        if isinstance(x, ops.PackedInput):
            return self._forward_packed(x, out, want_acc, emit_signs)
        if x.dim() != 4 or x.shape[1] != self.C:
            raise ValueError(f"input {tuple(x.shape)} does not match {self.C} filter channels")
        if not x.is_cuda:
            if want_acc or emit_signs:
                raise ValueError("want_acc / emit_signs are only supported for device inputs")
            return self.forward_host(x, out=out)
        if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
            x = x.contiguous()  # NCHW or channels-last maps are taken as they are
        self.out_shape(x.shape)
        return self._forward_device(x, out, want_acc, emit_signs)

    def _forward_device(self, x: torch.Tensor, out: torch.Tensor | None = None,
                        want_acc: bool = False, emit_signs: bool = False):
        variant = self.kernel_for(self.conv_in_shape(x.shape))
        plain = (self.in_affine is None and self.out_affine is None and self.in_pool is None
                 and not self.out_channels_last
                 and x.is_contiguous() and not want_acc and not emit_signs)
        if variant == "popc" and plain:
            return ops.layer_forward(x, self.filters, self.pad, self.workspace(x), y=out)
        if variant == "umma" and plain:  # one C-ABI call: K1 -> K2 -> tcgen05 K3+K4
            return ops.layer_forward_umma(x, self.filters, self.pad, self.workspace(x), y=out)
        bits, A = ops.pack_input(x, in_affine=self.in_affine, in_pool=self.in_pool)
        return self._conv_packed(ops.PackedInput(bits, A, self.C), variant, out, want_acc, emit_signs)

    def _forward_packed(self, p: "ops.PackedInput", out, want_acc: bool, emit_signs: bool):
        if p.C != self.C:
            raise ValueError(f"packed input has {p.C} channels, the filters {self.C}")
        if self.in_affine is not None or self.in_pool is not None:
            raise ValueError("a packed input is already normalised / pooled: in_affine / in_pool do not apply")
        self.out_shape(p.shape)
        return self._conv_packed(p, self.kernel_for(p.shape), out, want_acc, emit_signs)

    def forward_k1(self, p: "ops.PackedInput", out: torch.Tensor | None = None, emit_signs: bool = False):
        """The conv on an input whose K1 the caller produced WITH this layer's
        in_affine / in_pool applied (fused into its own pass, e.g. the network's
        front end: conv1's pool + this layer's batch norm + sign in one kernel)."""
        if p.C != self.C:
            raise ValueError(f"packed input has {p.C} channels, the filters {self.C}")
        N, C, H, W = p.shape  # already the conv's input shape (pooled, if in_pool)
        oh, ow = ops.out_dims(H, W, self.kh, self.kw, self.pad)
        if oh < 1 or ow < 1:
            raise ValueError("kernel larger than the padded input")
        return self._conv_packed(p, self.kernel_for(p.shape), out, False, emit_signs)

    def _conv_packed(self, p: "ops.PackedInput", variant: str, out, want_acc: bool, emit_signs: bool):
        """K2 -> K3+K4 on a K1-form input."""
        if variant in ("popc-fc", "umma-fc"):
            if emit_signs:
                if want_acc or out is not None:
                    raise ValueError("emit_signs returns the next layer's input: no out / want_acc")
                return self._fc_packed_emit(p, variant)
            return self._fc_packed(p, out, want_acc, variant)
        K = ops.scale_map(p.A, self.kh, self.kw, self.pad)
        if emit_signs:
            if variant != "umma":
                raise ValueError("emit_signs needs the tcgen05 kernel (variant 'umma' or 'auto')")
            return ops.xnor_conv_emit(p.bits, self.filters, K, self.pad, out_affine=self.out_affine)
        if (self.out_channels_last and variant == "umma" and not want_acc and self.O % 4 == 0
                and (out is None or out.is_contiguous(memory_format=torch.channels_last))):
            return ops.xnor_conv_nhwc(p.bits, self.filters, K, self.pad, out=out, out_affine=self.out_affine)
        y, acc = ops.xnor_conv(p.bits, self.filters, K, self.pad, want_acc=want_acc,
                               variant=variant, y=out, out_affine=self.out_affine)
        return (y, acc) if want_acc else y

    def kernel_for(self, x_shape) -> str:
        """The conv kernel a forward of this input shape runs: 'auto' picks the
        tcgen05 kernel whenever its shared-memory plan fits the shape; a fully
        connected shape (kernel == input, pad 0, 1x1 output) runs the popc kernel
        with the batch laid out as the image width ('popc-fc'); else popc."""
        N, C, H, W = x_shape
        if self.variant != "auto":
            return self.variant
        if self._fc_shape(x_shape):
            # 1x1 output: one 'pixel' per image, so the batch becomes the image width
            # (a 1 x N image of kh*kw*C channels); tensor cores when the plan fits
            Cp = self.kh * self.kw * C
            if self.filters.wq is not None and ops.umma_supported(1, Cp, 1, N, self.O, 1, 1, 0):
                return "umma-fc"
            return "popc-fc"
        if ops.umma_supported(N, C, H, W, self.O, self.kh, self.kw, self.pad):
            return "umma"
        return "popc"

    def _fc_shape(self, x_shape) -> bool:
        N, C, H, W = x_shape
        return self.pad == 0 and self.kh == H and self.kw == W and C % 32 == 0 and N > 1

    def _fc_packed(self, p: "ops.PackedInput", out, want_acc: bool, variant: str):
        """Fully connected binary layer (kernel covers the whole input): every image
        is one 'pixel' of a 1-row image whose channels are the (y, x, c) words of
        the image, so the conv kernels' pixel tiling runs over the batch.  Same
        arithmetic as the conv view: C' = kh*kw*C valid bits, K = box mean of A
        over the whole input, alpha per filter (the reference's (c, ky, kx) sum)."""
        N, C, H, W = p.shape
        bits, A = p.bits, p.A
        K = self._fc_k(A)                                             # [N, 1, 1]
        fcf = self._fc_filters(umma=variant == "umma-fc")
        if variant == "umma-fc" and not want_acc and self.O % 4 == 0 and (
                out is None or out.is_contiguous()):
            # y written [batch][filters] by the kernel itself (channels-last of a 1 x N image)
            y = ops.xnor_conv_nhwc(bits.view(1, 1, N, H * W * ops.words(C)), fcf, K.view(1, 1, N), 0,
                                   out_affine=self.out_affine)                   # [1, O, 1, N] channels-last
            y = y.permute(0, 3, 2, 1).reshape(N, self.O, 1, 1)                   # a view: memory is [N][O]
            if out is not None:
                out.copy_(y)
                return out
            return y
        y1, acc1 = ops.xnor_conv(bits.view(1, 1, N, H * W * ops.words(C)), fcf, K.view(1, 1, N), 0,
                                 want_acc=want_acc, out_affine=self.out_affine,
                                 variant="umma" if variant == "umma-fc" else "popc")  # [1, O, 1, N]
        y = y1.view(self.O, N).t().reshape(N, self.O, 1, 1)
        if out is not None:
            out.copy_(y)
            y = out
        if want_acc:
            return y, acc1.view(self.O, N).t().reshape(N, self.O, 1, 1).contiguous()
        return y.contiguous()

    def _fc_k(self, A: torch.Tensor) -> torch.Tensor:
        """K of a fully connected layer: the box mean of A over the whole input; for a
        1 x 1 kernel that is A itself (K2's 0 + A, times f32(1/1), is A bit for bit), so
        no K2 launch."""
        if self.kh == 1 and self.kw == 1:
            return A
        return ops.scale_map(A, self.kh, self.kw, 0)

    def _fc_packed_emit(self, p: "ops.PackedInput", variant: str) -> "ops.PackedInput":
        """The fully connected layer with its output handed to the next binary layer in
        K1 form (sign words + A of y [* out_affine]): fused into the K-split finalize on
        the tcgen05 path (xnc_xnor_conv_umma_nhwc_emit), else K1 of y."""
        N, C, H, W = p.shape
        if variant == "umma-fc" and self.O % 32 == 0 and self.O <= 4096:
            K = self._fc_k(p.A)
            fcf = self._fc_filters(umma=True)
            y, nb, nA = ops.xnor_conv_nhwc(p.bits.view(1, 1, N, H * W * ops.words(C)), fcf, K.view(1, 1, N), 0,
                                           out_affine=self.out_affine, emit=True)
            return ops.PackedInput(nb.view(N, 1, 1, self.O // 32), nA.view(N, 1, 1), self.O)
        y = self._fc_packed(p, None, False, variant)
        bits, A = ops.pack_input(y.contiguous())
        return ops.PackedInput(bits, A, self.O)

    def _fc_filters(self, umma: bool = False) -> ops.PackedFilters:
        """The filters as 1x1 filters over kh*kw*C channels in (y, x, c) order; alpha
        stays the original filters' (summed in the reference's (c, ky, kx) order)."""
        f = getattr(self, "_fcf", None)
        if f is None:
            pf = self.filters
            wb = pf.wbits.permute(1, 2, 0, 3).contiguous()            # [kh, kw, Cw, O]
            f = ops.PackedFilters(wb.view(-1, 1, 1, self.O), pf.alpha, pf.alpha64, self.O,
                                  self.kh * self.kw * self.C, 1, 1)
            self._fcf = f
        if umma and f.wq is None:
            wp = self.weight.permute(0, 2, 3, 1).reshape(self.O, -1, 1, 1).contiguous()
            tmp = ops.PackedFilters(f.wbits, f.alpha, f.alpha64, f.O, f.C, 1, 1)
            ops.attach_umma_weights(tmp, wp)                           # signs + S_w only
            f.wq, f.sw = tmp.wq, tmp.sw
        return f

    __call__ = forward

    # ------------------------------------------------------------------ host path
    def forward_host(self, x_host: torch.Tensor, out: torch.Tensor | None = None,
                     chunk: int | None = None, device: torch.device | None = None,
                     non_blocking: bool = False) -> torch.Tensor:
        """Host x in, host y out, with the PCIe copies overlapped with compute.

        Returns once `out` holds the result (the last device->host copy is waited
        for on the host).  non_blocking=True returns as soon as the work is queued:
        the caller must then synchronise the current stream (which waits for the
        copies) before reading `out`.

        The batch is cut into chunks; chunk i+1 is copied host->device on one
        stream while chunk i runs K1 -> K2 -> K3+K4 on a second and chunk i-1
        is copied device->host on a third (two device buffers per direction,
        events order buffer reuse).  Pinned host memory is used for both ends
        (x is staged into a pinned buffer if it is not pinned already)."""
        dev = device or torch.device("cuda", torch.cuda.current_device())
        N = x_host.shape[0]
        _, O, oh, ow = self.out_shape(x_host.shape)
        if out is None:
            out = torch.empty((N, O, oh, ow), dtype=torch.float32, pin_memory=True)
        if not x_host.is_pinned():
            x_host = x_host.contiguous().pin_memory()
        if chunk is None:
            chunk = max(1, N // 16)
        st = self._host_state(dev, x_host.shape, chunk)
        s_in, s_cmp, s_out = st["streams"]
        cur = torch.cuda.current_stream(dev)
        s_in.wait_stream(cur)
        n_chunks = (N + chunk - 1) // chunk
        for i in range(n_chunks):
            a, b = i * chunk, min(N, (i + 1) * chunk)
            slot = i % 2
            xb = st["x"][slot][: b - a]
            yb = st["y"][slot][: b - a]
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(st["x_free"][slot])
                xb.copy_(x_host[a:b], non_blocking=True)
                st["x_ready"][slot].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(st["x_ready"][slot])
                if i >= 2:
                    s_cmp.wait_event(st["y_free"][slot])
                self._forward_device(xb, yb)
                st["x_free"][slot].record(s_cmp)
                st["y_ready"][slot].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(st["y_ready"][slot])
                out[a:b].copy_(yb, non_blocking=True)
                st["y_free"][slot].record(s_out)
        cur.wait_stream(s_out)
        if not non_blocking:
            st["done"].record(s_out)
            st["done"].synchronize()  # the D2H copies have landed in `out`
        return out

    def _host_state(self, dev, x_shape, chunk):
        key = ("host", dev, tuple(x_shape[1:]), chunk)
        st = self._ws.get(key)
        if st is None:
            _, C, H, W = x_shape
            _, O, oh, ow = self.out_shape((chunk, C, H, W))
            xs = [torch.empty((chunk, C, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
            st = {"streams": tuple(torch.cuda.Stream(dev) for _ in range(3)),
                  "x": xs,
                  "y": [torch.empty((chunk, O, oh, ow), dtype=torch.float32, device=dev) for _ in range(2)],
                  "ws": self.workspace(xs[0]),
                  "done": torch.cuda.Event(),
                  **{k: [torch.cuda.Event() for _ in range(2)]
                     for k in ("x_ready", "x_free", "y_ready", "y_free")}}
            self._ws[key] = st
        return st


def xnor_conv2d_layer(x: torch.Tensor, weight: torch.Tensor, pad: int | None = None,
                      want_acc: bool = False, variant: str = "auto"):
    """Functional batched layer (packs the weights on every call)."""
    return XnorConv2d(weight, pad, variant).forward(x, want_acc=want_acc)
