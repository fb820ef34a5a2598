"""Benchmark harness: vanilla vs bit-packed XNOR convolution on the device
(drop-in for xnorconv.bench, /root/reference/pkg/src/xnorconv/bench.py).

The reference's protocol, kept: deterministic float32-exact inputs from
(seed, size); buffers allocated and the input loaded outside the timed region;
binarization and packing timed as part of the XNOR convolution; `warmup`
untimed runs, then `repeats` timed runs; an equality gate against the naive
references before any timing (bench.py:131-207), aborting with BenchGateError.

What changes on a GPU: the reference's -1t/-mt thread variants become one
device implementation each, timed with CUDA events on the launching stream
(inputs resident, output left on the device):
  vanilla -- the reference's vanilla_conv (direct float32 conv in its
             (ch, ky, kx) order, csrc/xnc_verify.cu), on the pre-padded input;
  xnor    -- ConvWorkspace.run's device work, K1 -> K2 -> K3+K4.
The thread-count invariance gate becomes a run-to-run bit-identity gate.
`threads` is validated like the reference's and otherwise ignored."""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev
from ._lib import DTYPE_F32, check
from .binarize import sign_binarize, sign_plane
from .pipeline import ConvWorkspace
from .reference import bwn_conv, sign_conv2d_int
from .scaling import input_scale_map
from .tensor import Tensor2, Tensor3, channel_abs_mean, zero_pad

IMPLEMENTATIONS = ("vanilla", "xnor")
BASELINE_OF = {"xnor": "vanilla"}
DEFAULT_SIZES = (256, 512, 1024, 2048)
GATE_PROBE_SIZE = 48  # bench.py:36


class BenchGateError(RuntimeError):
    """Pre-timing equality gate failed; results would be meaningless."""


@dataclass
class BenchConfig:
    sizes: tuple[int, ...] = DEFAULT_SIZES
    kernel: int = 3
    channels: int = 1
    repeats: int = 100
    warmup: int = 10
    threads: int | str = "all"
    word_bits: int = 64
    seed: int = 0
    fmt: str = "table"
    backend: str | None = None

    def __post_init__(self) -> None:  # bench.py:56-82
        self.sizes = tuple(int(s) for s in self.sizes)
        if not self.sizes:
            raise ValueError("sizes must be non-empty")
        if any(s < self.kernel for s in self.sizes):
            raise ValueError("every size must be >= the kernel size")
        if self.kernel < 1 or self.kernel % 2 == 0:
            raise ValueError("kernel must be odd and >= 1")
        if self.channels < 1:
            raise ValueError("channels must be >= 1")
        if self.repeats < 1:
            raise ValueError("repeats must be >= 1")
        if self.warmup < 0:
            raise ValueError("warmup must be >= 0")
        if self.word_bits not in (32, 64):
            raise ValueError("word_bits must be 32 or 64")
        if self.fmt not in ("table", "csv"):
            raise ValueError("format must be 'table' or 'csv'")
        if self.threads != "all":
            self.threads = int(self.threads)
            if self.threads < 1:
                raise ValueError("threads must be >= 1 or 'all'")

    @property
    def thread_count(self) -> int:
        if self.threads == "all":
            return os.cpu_count() or 1
        return self.threads


@dataclass(frozen=True)
class BenchRow:
    impl: str
    size: int
    mean_ms: float
    std_ms: float
    speedup: float


@dataclass
class BenchReport:
    rows: list[BenchRow] = field(default_factory=list)


def _bench_data(cfg: BenchConfig, size: int) -> tuple[Tensor3, Tensor3]:
    """bench.py:100-108: float32-exact input and weights for one size."""
    rng = np.random.default_rng((cfg.seed, size))
    data = rng.uniform(-1.0, 1.0, (cfg.channels, size, size)).astype(np.float32).astype(np.float64)
    wdata = rng.uniform(-1.0, 1.0, (cfg.channels, cfg.kernel, cfg.kernel)).astype(np.float32).astype(np.float64)
    return Tensor3(data), Tensor3(wdata)


def _sign_dominated(cfg: BenchConfig, size: int, magnitude: float, w_magnitude: float):
    """bench.py:111-117: constant-magnitude random signs (the approximation is exact)."""
    rng = np.random.default_rng((cfg.seed, size, 1))
    signs = rng.integers(0, 2, (cfg.channels, size, size)) * 2 - 1
    wsigns = rng.integers(0, 2, (cfg.channels, cfg.kernel, cfg.kernel)) * 2 - 1
    return Tensor3(signs * magnitude), Tensor3(wsigns * w_magnitude)


def _interior(arr: np.ndarray, border: int) -> np.ndarray:
    return arr if border == 0 else arr[border:-border, border:-border]


def _rel_err(got: np.ndarray, want: np.ndarray) -> float:
    return float(np.abs(got - want).max()) / max(float(np.abs(want).max()), 1e-30)


def _workspace(cfg: BenchConfig, inp: Tensor3, wts: Tensor3, pad: int) -> ConvWorkspace:
    ws = ConvWorkspace(cfg.channels, inp.height, inp.width, cfg.kernel, cfg.kernel, pad, cfg.word_bits,
                       cfg.backend)
    ws.set_weights(wts)
    ws.load_input(inp)
    return ws


def _gate_small_probe(cfg: BenchConfig) -> None:
    """bench.py:131-176: exact ints vs the naive sign convolution, the pipeline
    vs its decomposition (<= 1e-5), and the interior vs bwn_conv on
    sign-dominated data (<= 1e-4)."""
    size = max(GATE_PROBE_SIZE, cfg.kernel)
    pad = (cfg.kernel - 1) // 2
    inp, wts = _bench_data(cfg, size)
    ws = _workspace(cfg, inp, wts, pad)
    got = ws.run(threads=1).copy()
    ints = ws.int_plane()
    ws.close()
    padded = zero_pad(inp, pad)
    approx = sign_binarize(wts)
    oracle_ints = sign_conv2d_int([sign_plane(Tensor2(ch)) for ch in padded.data], approx.signs, pad=0)
    if not np.array_equal(ints.values, oracle_ints.values):
        raise BenchGateError("XNOR integer output disagrees with the naive reference")
    scale_map = input_scale_map(channel_abs_mean(inp), cfg.kernel, cfg.kernel, pad)
    if _rel_err(got, oracle_ints.values * scale_map.data * approx.scale) > 1e-5:
        raise BenchGateError("pipeline output disagrees with its decomposition")
    probe_in, probe_w = _sign_dominated(cfg, size, 0.75, 0.5)
    ws = _workspace(cfg, probe_in, probe_w, pad)
    got_probe = ws.run(threads=1).copy()
    ws.close()
    want_bwn = bwn_conv(probe_in, sign_binarize(probe_w), pad)
    err = _rel_err(_interior(got_probe, pad), _interior(want_bwn.data, pad))
    if err > 1e-4:
        raise BenchGateError(f"XNOR vs binary-weight reference interior mismatch ({err:.2e})")


class _Vanilla:
    """The reference's vanilla_conv on the device over the workspace's padded input."""

    def __init__(self, cfg: BenchConfig, inp: Tensor3, wts: Tensor3, pad: int):
        p = pad
        x = torch.from_numpy(inp.data.astype(np.float32)).to(_dev.device())
        self.padded = torch.nn.functional.pad(x, (p, p, p, p)).contiguous()
        self.w = torch.from_numpy(wts.data.astype(np.float32)).to(_dev.device()).contiguous()
        self.C, self.ph, self.pw = self.padded.shape
        self.k = cfg.kernel
        self.out = torch.empty((self.ph - self.k + 1, self.pw - self.k + 1), dtype=torch.float32,
                               device=_dev.device())

    def __call__(self) -> torch.Tensor:
        check(_dev.L().xnc_vanilla_conv(self.padded.data_ptr(), DTYPE_F32, self.C, self.ph, self.pw,
                                        self.w.data_ptr(), self.k, self.k, self.out.data_ptr(),
                                        _dev.stream()), "xnc_vanilla_conv")
        return self.out


def _xnor_runner(ws: ConvWorkspace):
    def run() -> torch.Tensor:
        ws._enqueue(True, False)
        return ws._y[0, 0]
    return run


def _gate_size(cfg: BenchConfig, size: int, runners: dict) -> None:
    """bench.py:179-207: repeat runs bit-identical (the device form of the
    thread-count invariance gate), then XNOR vs vanilla on sign-dominated data."""
    for impl, fn in runners.items():
        a = fn().clone()
        if not torch.equal(a, fn()):
            raise BenchGateError(f"{impl} outputs differ between runs at {size}")
    pad = (cfg.kernel - 1) // 2
    probe_in, probe_w = _sign_dominated(cfg, size, 0.75, 0.5)
    ws = _workspace(cfg, probe_in, probe_w, pad)
    got = ws.run(threads=1).copy()
    ws.close()
    want = _Vanilla(cfg, probe_in, probe_w, pad)().cpu().numpy()
    err = _rel_err(_interior(got, pad), _interior(want, pad))
    if err > 1e-4:
        raise BenchGateError(f"XNOR vs vanilla interior mismatch at size {size} ({err:.2e})")


def _timed(fn, warmup: int, repeats: int) -> tuple[float, float]:
    """CUDA-event time of each call on the current stream: mean, std (ms)."""
    for _ in range(warmup):
        fn()
    s = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(repeats)]
    torch.cuda.synchronize()
    for e0, e1 in evs:
        e0.record(s)
        fn()
        e1.record(s)
    torch.cuda.synchronize()
    samples = np.array([e0.elapsed_time(e1) for e0, e1 in evs])
    return float(samples.mean()), float(samples.std(ddof=1)) if repeats > 1 else 0.0


def run_bench(cfg: BenchConfig) -> BenchReport:
    """Time every implementation at every size and derive speed-ups (bench.py:223-260)."""
    _gate_small_probe(cfg)
    report = BenchReport()
    pad = (cfg.kernel - 1) // 2
    for size in cfg.sizes:
        inp, wts = _bench_data(cfg, size)
        ws = _workspace(cfg, inp, wts, pad)
        runners = {"vanilla": _Vanilla(cfg, inp, wts, pad), "xnor": _xnor_runner(ws)}
        _gate_size(cfg, size, runners)
        stats = {impl: _timed(runners[impl], cfg.warmup, cfg.repeats) for impl in IMPLEMENTATIONS}
        ws.close()
        for impl in IMPLEMENTATIONS:
            mean, std = stats[impl]
            baseline = stats[BASELINE_OF.get(impl, impl)][0]
            report.rows.append(BenchRow(impl, size, mean, std, baseline / mean))
    return report


def emit_report(report: BenchReport, fmt: str = "table") -> str:
    """bench.py:263-282: aligned table or exact-round-trip CSV."""
    if fmt == "csv":
        lines = ["impl,size,mean_ms,std_ms,speedup"]
        for r in report.rows:
            lines.append(f"{r.impl},{r.size},{r.mean_ms!r},{r.std_ms!r},{r.speedup!r}")
        return "\n".join(lines) + "\n"
    if fmt != "table":
        raise ValueError(f"unknown format {fmt!r}")
    header = f"{'impl':<12} {'size':>6} {'mean_ms':>12} {'std_ms':>10} {'speed-up':>9}"
    lines = [header, "-" * len(header)]
    for r in report.rows:
        lines.append(f"{r.impl:<12} {r.size:>6} {r.mean_ms:>12.4f} {r.std_ms:>10.4f} {r.speedup:>8.2f}x")
    return "\n".join(lines) + "\n"


def parse_csv(text: str) -> BenchReport:
    """Inverse of emit_report(fmt='csv') (bench.py:285-297)."""
    lines = [ln for ln in text.strip().splitlines() if ln]
    if not lines or lines[0] != "impl,size,mean_ms,std_ms,speedup":
        raise ValueError("missing or unexpected CSV header")
    report = BenchReport()
    for ln in lines[1:]:
        impl, size, mean_ms, std_ms, speedup = ln.split(",")
        report.rows.append(BenchRow(impl, int(size), float(mean_ms), float(std_ms), float(speedup)))
    return report
