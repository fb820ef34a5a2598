"""End-to-end binary convolution, one image x one filter (drop-in for
xnorconv.pipeline, /root/reference/pkg/src/xnorconv/pipeline.py).

`ConvWorkspace` keeps the reference's lifecycle -- preallocated buffers for a
fixed shape, set_weights (untimed binarization), load_input (untimed copy),
run() (binarize + pack + XNOR decode + alpha*K, timed) -- but every buffer is
device memory and run() enqueues the sm_100a kernels K1 -> K2 -> K3+K4 with
N = O = 1.  The returned array is the reused float32 host output, as in the
reference (pipeline.py:124-151).  `threads` / `two_stream` are accepted for
signature compatibility; the GPU grid replaces both (race-free by
construction, unlike the reference's fused kernel at kh != 3)."""
from __future__ import annotations

import numpy as np
import torch

from . import _dev, ops
from ._lib import DTYPE_F32
from .engine import BinaryFilter, IntOutputPlane, build_filter
from .layer import default_pad  # noqa: F401  (re-exported: pipeline.default_pad)
from .pack import PackedTileGrid, TileGeometry, _check_backend, pack_device, tile_grid_shape
from .tensor import Tensor2, Tensor3


class ConvWorkspace:
    """Reusable device buffers and a packed filter for one convolution shape."""

    def __init__(self, channels: int, height: int, width: int, kernel_h: int, kernel_w: int,
                 pad: int, word_bits: int = 64, backend: str | None = None):
        if pad < 0:
            raise ValueError("pad must be >= 0")
        _check_backend(backend)
        self.geometry = TileGeometry(word_bits, kernel_h, kernel_w)
        self.channels, self.height, self.width, self.pad = channels, height, width, pad
        self.out_h = height + 2 * pad - kernel_h + 1
        self.out_w = width + 2 * pad - kernel_w + 1
        if self.out_h < 1 or self.out_w < 1:
            raise ValueError("kernel larger than the padded input")
        self.tiles = tile_grid_shape(self.geometry, self.out_h, self.out_w)
        dev = _dev.device()
        cw = ops.words(channels)
        self._x = torch.zeros((1, channels, height, width), dtype=torch.float32, device=dev)
        self._bits = torch.empty((1, height, width, cw), dtype=torch.int32, device=dev)
        self._A = torch.empty((1, height, width), dtype=torch.float32, device=dev)
        self._K = torch.empty((1, self.out_h, self.out_w), dtype=torch.float32, device=dev)
        self._y = torch.empty((1, 1, self.out_h, self.out_w), dtype=torch.float32, device=dev)
        self._acc = torch.empty((1, 1, self.out_h, self.out_w), dtype=torch.int32, device=dev)
        self.out = np.empty((self.out_h, self.out_w), dtype=np.float32)
        self.ints = np.zeros((self.out_h, self.out_w), dtype=np.int32)
        self.filter: BinaryFilter | None = None
        self._packed: ops.PackedFilters | None = None
        self.variant = "auto"  # conv kernel choice (ops.resolve_variant); tests pin 'popc' / 'umma' 

    def set_weights(self, weights: Tensor3) -> None:
        """Binarize one filter (untimed, pipeline.py:77-83): the reference-layout
        BinaryFilter plus the device-packed filter the conv kernel reads."""
        if weights.channels != self.channels:
            raise ValueError(f"{weights.channels} weight channels for a {self.channels}-channel workspace")
        self.filter = build_filter(weights, self.geometry)
        w64 = _dev.to_dev(weights.data[np.newaxis])
        self._packed = ops.pack_weights_f64(w64)
        # the tcgen05 layout too: run() takes that kernel whenever its plan fits
        # (ops.xnor_conv's 'auto'), else the popc kernel
        ops.attach_umma_weights(self._packed, w64)

    def load_input(self, t: Tensor3) -> None:
        """Copy the image to the device as float32 (the reference's cast, pipeline.py:85-93)."""
        if (t.channels, t.height, t.width) != (self.channels, self.height, self.width):
            raise ValueError(f"input {t.channels}x{t.height}x{t.width} does not match workspace "
                             f"{self.channels}x{self.height}x{self.width}")
        self._x.copy_(torch.from_numpy(t.data.astype(np.float32))[None])

    def _enqueue(self, want_y: bool, want_acc: bool) -> None:
        if self.filter is None or self._packed is None:
            raise RuntimeError("set_weights() before run()")
        k = self.geometry
        ops.pack_input_into(self._x, self._bits, self._A)
        if want_y:
            ops.scale_map_into(self._A, k.kernel_h, k.kernel_w, self.pad, self._K)
        ops.xnor_conv(self._bits, self._packed, self._K if want_y else None, self.pad,
                      want_y=want_y, want_acc=want_acc, y=self._y if want_y else None,
                      acc=self._acc if want_acc else None, variant=self.variant)

    @property
    def kernel(self) -> str:
        """The conv kernel run() launches for this shape ('umma' or 'popc')."""
        k = self.geometry
        return ops.resolve_variant(self.variant, self._packed, 1, self.channels, self.height, self.width,
                                   self.pad) if self._packed is not None else self.variant

    def run(self, threads: int = 1, two_stream: bool = False) -> np.ndarray:
        """One full convolution; returns the reused float32 host output array."""
        self._enqueue(True, False)
        self.out[...] = self._y[0, 0].cpu().numpy()
        return self.out

    def int_plane(self) -> IntOutputPlane:
        """Integer window sums of the loaded input (pipeline.py:164-173)."""
        self._enqueue(False, True)
        self.ints[...] = self._acc[0, 0].cpu().numpy()
        return IntOutputPlane(self.ints.copy())

    def grids(self) -> list[PackedTileGrid]:
        """Per-channel reference-layout tile grids of the loaded, padded input
        (pipeline.py:158-162), packed on the device."""
        p = self.pad
        padded = torch.nn.functional.pad(self._x[0], (p, p, p, p)).contiguous()
        ph, pw = padded.shape[1:]
        ty, tx = self.tiles
        return [PackedTileGrid(self.geometry, _dev.to_host(
            pack_device(padded[c], DTYPE_F32, ph, pw, self.geometry, ty, tx), np.uint64))
            for c in range(self.channels)]

    def close(self) -> None:
        """Nothing to shut down (no side thread); kept for API compatibility."""


def xnor_conv(input: Tensor3, weights: Tensor3, pad: int | None = None, word_bits: int = 64,
              threads: int = 1, backend: str | None = None, two_stream: bool | None = None) -> Tensor2:
    """One-shot wrapper: workspace, one run, Tensor2 result (pipeline.py:176-201)."""
    if input.channels != weights.channels:
        raise ValueError(f"{input.channels} input channels vs {weights.channels} weight channels")
    if pad is None:
        pad = default_pad(weights.height, weights.width)
    ws = ConvWorkspace(input.channels, input.height, input.width, weights.height, weights.width, pad,
                       word_bits, backend)
    ws.set_weights(weights)
    ws.load_input(input)
    try:
        return Tensor2(ws.run(threads=threads, two_stream=bool(two_stream)).copy())
    finally:
        ws.close()
