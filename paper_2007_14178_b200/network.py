"""XNOR-Net / AlexNet forward (BASELINE.json configs 4 and 5).

The reference has no network object, so the
network is composed from reference-expressible binary layers -- stride-1
binary convolutions with k <= 8 and explicit padding -- with the rest of
XNOR-Net AlexNet in full precision through torch (cuDNN), off the binary hot
path:

    conv1  11x11/4, 3 -> 96      full precision      224 -> 55  (as 3x3 over 4x4 space-to-depth)
    pool   3/2                                       55 -> 27
    bn2 -> conv2  5x5 pad 2, 96 -> 256  BINARY (XnorConv2d) 27
    pool   3/2                                       27 -> 13  (conv3's in_pool: xnc_max_pool)
    bn3 -> conv3  3x3 pad 1, 256 -> 384 BINARY       13  (epilogue applies bn4)
    conv4  3x3 pad 1, 384 -> 384 BINARY              13  (epilogue applies bn5)
    conv5  3x3 pad 1, 384 -> 256 BINARY              13
    pool   3/2                                       13 -> 6   (fc6's in_pool)
    bn6 -> fc6  6x6 valid, 256 -> 4096 BINARY (a k = H = W conv)  1x1  (epilogue applies bn7)
    fc7    1x1, 4096 -> 4096     BINARY              1x1
    fc8    4096 -> 1000          full precision

Binary MACs per image: 1.026e9.  Every binary layer
is the reference semantics end to end: sign(0) = +1, +1 padding, per-filter
alpha, K from the channel mean of |input| (xnor_conv(x[n], w[o]) for every
pair).  Weights are random-init (no checkpoints offline).
"""
from __future__ import annotations

import contextlib

import torch
import torch.nn.functional as F

from . import ops
from .layer import XnorConv2d


@contextlib.contextmanager
def _tf32_full_precision_layers():
    """TF32 tensor cores + cuDNN autotuning for conv1 / fc8, restored on exit."""
    saved = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32,
             torch.backends.cudnn.benchmark)
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    torch.backends.cudnn.benchmark = True
    try:
        yield
    finally:
        (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32,
         torch.backends.cudnn.benchmark) = saved

BINARY_LAYERS = (  # name, C_in, C_out, k, pad
    ("conv2", 96, 256, 5, 2),
    ("conv3", 256, 384, 3, 1),
    ("conv4", 384, 384, 3, 1),
    ("conv5", 384, 256, 3, 1),
    ("fc6", 256, 4096, 6, 0),
    ("fc7", 4096, 4096, 1, 0),
)
POOLED_INPUT = ("conv3", "fc6")  # layers whose input is max-pool 3/2 of the previous output
EMITS_NEXT = ("conv3", "conv4", "fc6")  # binary -> binary with no pool between: the next layer's K1
                                        # comes from the conv (epilogue, or fc6's K-split finalize)
BINARY_MACS_PER_IMAGE = (27 * 27 * 256 * 96 * 25 + 13 * 13 * 384 * 256 * 9 + 13 * 13 * 384 * 384 * 9
                         + 13 * 13 * 256 * 384 * 9 + 4096 * 256 * 36 + 4096 * 4096)


class XnorNetAlexNet:
    """Random-init XNOR-Net AlexNet resident on one device."""

    def __init__(self, device: torch.device | str = "cuda", num_classes: int = 1000, seed: int = 0,
                 variant: str = "auto", emit_signs: bool = True, conv1: str = "tcgen05"):
        dev = torch.device(device)
        g = torch.Generator().manual_seed(seed)

        def rnd(*shape, scale=1.0):
            return ((torch.rand(shape, generator=g) * 2 - 1) * scale).to(dev)

        self.device = dev
        self.emit_signs = emit_signs and variant in ("auto", "umma")
        self.conv1_w = rnd(96, 3, 11, 11, scale=(3 * 121) ** -0.5)
        self.conv1_b = rnd(96, scale=0.1)
        # conv1 as a 3x3/1 conv over the 4x4 space-to-depth input (48 channels):
        # the 11x11 kernel zero-padded to 12x12 and split into 4x4 phases.  Same
        # products and sums as the 11x11/4 conv, in a shape cuDNN runs ~2x faster
        # (tools/conv1_probe.py: 1.18 vs 2.13 ms at batch 256 incl. ReLU + pool).
        w12 = F.pad(self.conv1_w, (0, 1, 0, 1))
        self.conv1_w_s2d = (w12.view(96, 3, 3, 4, 3, 4).permute(0, 1, 3, 5, 2, 4)
                            .reshape(96, 48, 3, 3).contiguous())
        self.conv1_w_s2d_cl = self.conv1_w_s2d.contiguous(memory_format=torch.channels_last)
        # conv1 engine: 'tcgen05' = our kind::tf32 kernel on the raw images (no
        # space-to-depth pass; csrc/xnc_conv1.cu), 'cudnn' = the s2d + cuDNN TF32 path
        if conv1 not in ("tcgen05", "cudnn"):
            raise ValueError(f"conv1 must be 'tcgen05' or 'cudnn', got {conv1!r}")
        self.conv1 = conv1
        self.conv1_wq = ops.conv1_pack_weights(self.conv1_w) if conv1 == "tcgen05" else None
        # XNOR-Net's binary block is BatchNorm -> BinActiv -> BinConv (-> Pool); the
        # batch norms are folded to a per-channel affine (scale, shift), random-init
        # like everything else.  After a pool it runs inside K1 of the next layer
        # (in_affine); between two binary layers it is fused into the first layer's
        # conv epilogue (out_affine), so the stored feature map is already normalised.
        def bn(c, center):
            gamma = 0.8 + 0.4 * torch.rand(c, generator=g)
            beta = 0.2 * torch.rand(c, generator=g) - 0.1
            mean = center * torch.rand(c, generator=g)
            var = 0.5 + torch.rand(c, generator=g)
            scale = gamma / torch.sqrt(var + 1e-5)
            return scale.to(dev), (beta - mean * scale).to(dev)

        self.bn = {"conv2": bn(96, 0.6), "conv3": bn(256, 0.5), "conv4": bn(384, 0.2),
                   "conv5": bn(384, 0.2), "fc6": bn(256, 0.3), "fc7": bn(4096, 0.2)}
        fused_out = {"conv3": "conv4", "conv4": "conv5", "fc6": "fc7"}  # BN of the next layer
        self.binary: dict[str, XnorConv2d] = {}
        for name, cin, cout, k, pad in BINARY_LAYERS:
            in_aff = None if name in fused_out.values() else self.bn[name]
            out_aff = self.bn[fused_out[name]] if name in fused_out else None
            # the max-pools after conv2 / conv5 are the next layer's in_pool (our pool kernel)
            in_pool = (3, 2) if name in POOLED_INPUT else None
            # (out_channels_last for conv2 / conv5, so their pools and the next K1 run
            # channels-last, measured no faster: the NHWC epilogue's per-pixel 64-byte runs
            # cost what the coalesced pool saves; DESIGN 4b.  Again with the final fused
            # channels-last pool + K1: C4 0.700 / 0.695 / 0.701 ms for conv2 / conv5 / both
            # vs 0.694 NCHW)
            self.binary[name] = XnorConv2d(rnd(cout, cin, k, k), pad=pad, variant=variant,
                                           in_affine=in_aff, out_affine=out_aff, in_pool=in_pool)
        self.fc8_w = rnd(num_classes, 4096, scale=4096 ** -0.5)
        self.fc8_b = rnd(num_classes, scale=0.1)

    @torch.no_grad()
    def forward(self, x: torch.Tensor, return_features: bool = False):
        """x f32 [N, 3, 224, 224] (CUDA) -> logits f32 [N, num_classes].

        conv1 / fc8 run on cuDNN / cuBLAS with TF32 tensor cores (full precision
        layers of XNOR-Net, outside the binary path); the binary layers are
        exact reference semantics."""
        with _tf32_full_precision_layers():
            return self._forward(x, return_features)

    @torch.no_grad()
    def front_end(self, x: torch.Tensor) -> torch.Tensor:
        """conv1 (11x11, stride 4, pad 2; full precision, via space-to-depth) -> ReLU
        -> max-pool 3/2: the input of the first binary layer (the same cuDNN
        settings as inside forward())."""
        with _tf32_full_precision_layers():
            # pad + space-to-depth and ReLU + pool are one pass each (our data-movement
            # kernels, same values as F.pad / F.pixel_unshuffle and F.relu / F.max_pool2d),
            # channels-last end to end: cuDNN's NHWC TF32 conv is 0.39 vs 0.60 ms NCHW, and
            # conv2's K1 reads the channels-last map directly (tools/front_probe.py)
            return ops.max_pool(self._conv1_map(x), 3, 2, relu=True, bias=self.conv1_b)

    def _conv1_map(self, x: torch.Tensor) -> torch.Tensor:
        """conv1 without its bias: f32 [N, 96, 55, 55] channels-last."""
        if self.conv1 == "tcgen05" and tuple(x.shape[1:]) == (3, 224, 224):
            return ops.conv1_forward(x, self.conv1_wq)  # TF32 tensor cores, channels-last out
        xs = ops.pad_space_to_depth(x, 2, 4, channels_last=True)
        return F.conv2d(xs, self.conv1_w_s2d_cl)  # bias folded into the pool (exact: see max_pool)

    def _forward(self, x: torch.Tensor, return_features: bool):
        feats = {}
        h = None
        for name, *_ in BINARY_LAYERS:
            # conv3 / fc6 take the pre-pool map (their in_pool); conv3 and conv4 hand the
            # next layer its input in packed-sign form (sign-emitting epilogue, exact)
            # unless the float feature maps are asked for
            emit = self.emit_signs and not return_features and name in EMITS_NEXT
            layer = self.binary[name]
            if h is None:
                # conv2's K1 fused with conv1's bias + ReLU + pool 3/2 and conv2's batch
                # norm: one pass over conv1's channels-last map, the pooled map never
                # written (xnc_pack_input_pool_nhwc; same bits / A as front_end() + K1)
                with _tf32_full_precision_layers():
                    pre = self._conv1_map(x)
                bits, A = ops.pack_input(pre, in_affine=layer.in_affine, in_pool=(3, 2), pool_relu=True,
                                         pool_bias=self.conv1_b)
                h = layer.forward_k1(ops.PackedInput(bits, A, layer.C), emit_signs=emit)
            else:
                h = layer.forward(h, emit_signs=emit)  # NCHW / channels-last / packed
            feats[name] = h
        logits = F.linear(h.flatten(1), self.fc8_w, self.fc8_b)  # full precision
        return (logits, feats) if return_features else logits

    __call__ = forward

    def capture(self, x_static: torch.Tensor):
        """Record one forward of the fixed input buffer x_static as a CUDA graph.

        Returns (graph, logits): after copying new images into x_static,
        graph.replay() recomputes logits in place.  Same kernels and results as
        forward() (the graph only removes the ~40 per-layer launches from the host
        path: 1.65 vs 1.71 ms at batch 256)."""
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):  # warm up: one-time smem opt-ins, cuDNN plans
            for _ in range(2):
                self.forward(x_static)
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            logits = self.forward(x_static)
        return graph, logits

    def binary_kernels(self, batch: int) -> dict[str, str]:
        """Which conv kernel (umma / popc) each binary layer runs at this batch."""
        shapes = {"conv2": (96, 27), "conv3": (256, 13), "conv4": (384, 13), "conv5": (384, 13),
                  "fc6": (256, 6), "fc7": (4096, 1)}
        return {n: self.binary[n].kernel_for((batch, c, s, s)) for n, (c, s) in shapes.items()}
