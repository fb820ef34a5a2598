#!/usr/bin/env python
"""Benchmark: XNOR-conv forward on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C3|C2k3|C2k5|C2k7|C1] [--variant popc|b1mma] [--no-cpu]

One STEP = one pass of the hot path over one batch: K1 sign+bit-pack+|x|-mean,
K2 K map, K3+K4 XNOR-popcount conv with the alpha*K epilogue, for every
(image, filter) pair of the layer.  Weight packing is outside the timed region
(the reference's set_weights is untimed too, bench.py:234-237).

Workload at N=1: BASELINE config 3 (the roofline headline): 3x3, C=O=256,
56x56, batch 256 per GPU (weak scaling under torchrun: every rank runs its own
256-image shard, no collective on the data path).  Inputs are 822 MB > L2
(126 MB), so no explicit L2 flush is needed between steps.

Prints ONE JSON line (rank 0).  `--impl reference` times the reference's own
CPU implementation (oracle/_ref: xnorconv._kernels_cy.xnor_reconstruct, built
from the reference .pyx) on the host cores, same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N per GPU, C, H, W, O, k)
    "C1": (1, 64, 32, 32, 64, 3),
    "C2k3": (64, 128, 64, 64, 128, 3),
    "C2k5": (64, 128, 64, 64, 128, 5),
    "C2k7": (64, 128, 64, 64, 128, 7),
    "C3": (256, 256, 56, 56, 256, 3),
}
NETWORK_CONFIGS = {"C4": 256, "C5": 2048}  # XNOR-Net AlexNet forward; C5 = global batch over ranks
CONFIG_TEXT = {
    "C4": "binary AlexNet/XNOR-Net full forward, random-init, 224x224 synthetic, batch 256 (BASELINE config 4)",
    "C5": "batch-sharded XNOR-Net forward, global batch 2048 over the ranks (BASELINE config 5)",
    "C1": "single XNOR conv layer 3x3, C_in=C_out=64, 32x32, batch 1",
    "C2k3": "XNOR conv 3x3, C=128, 64x64, batch 64", "C2k5": "XNOR conv 5x5, C=128, 64x64, batch 64",
    "C2k7": "XNOR conv 7x7, C=128, 64x64, batch 64",
    "C3": "ResNet-stage binary conv 3x3, C=256, 56x56, batch 256 (BASELINE config 3)",
}
METRIC = "XNOR-conv Gbinop/s and images/sec at 1/2/4/8 B200 vs host-CPU reference"
NCCL_LOG_DIR = os.path.join(ROOT, "gpurun_out")
POPC_LANES_PER_CLK_SM = 15.95  # measured, profiles/int_peaks_r1.jsonl
UMMA_I8_MAC_PER_CLK_SM = 7874.4  # measured tcgen05 kind::i8 M128 N256 K32, profiles/umma_probe_r1.jsonl


def binops(N, C, H, W, O, k):
    pad = (k - 1) // 2
    oh, ow = H + 2 * pad - k + 1, W + 2 * pad - k + 1
    return 2.0 * N * O * oh * ow * C * k * k  # 1 bit-MAC = 2 binops


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                     "--format=csv,noheader,nounits", "-lms", "100"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        while not self._stop.is_set():
            line = proc.stdout.readline()
            if not line:
                break
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass
        proc.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=2)

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        mask = 0
        for s in busy:
            mask |= s[2]
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": max(s[1] for s in busy),
                "reasons": [v for k, v in self.REASONS.items() if mask & k and k != 0x1],
                "samples": len(busy)}


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(dev=None):
    """One process group per bench process (NCCL on the GPU box, gloo for --dry-run),
    created on first use and kept for every leg of the run."""
    import torch.distributed as dist
    ws, _, _ = dist_env()
    if ws > 1 and not dist.is_initialized():
        if dev is None:
            dist.init_process_group("gloo")
        else:
            # log NCCL's communicator init (rank count, transports) to a per-process file,
            # never stdout (rank 0's stdout carries the one JSON line); device_id makes the
            # init eager, so the log exists before the first timed step
            os.makedirs(NCCL_LOG_DIR, exist_ok=True)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(NCCL_LOG_DIR, "nccl_init.%h.%p.log"))
            dist.init_process_group("nccl", device_id=dev)
    return ws


def comm_info():
    """What the data plane saw: backend and communicator size (the NCCL init lines
    themselves go to stderr when bench.py spawned the ranks: NCCL_DEBUG=INFO,
    NCCL_DEBUG_SUBSYS=INIT)."""
    import re
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return {"backend": None, "nranks": 1, "collectives_on_hot_path": 0}
    info = {"backend": dist.get_backend(), "nranks": dist.get_world_size(), "collectives_on_hot_path": 0}
    log = os.environ.get("NCCL_DEBUG_FILE", "").replace("%h", platform.node()).replace("%p", str(os.getpid()))
    if info["backend"] == "nccl" and log and os.path.exists(log):
        # NCCL's own record of the communicator: "... comm 0x.. rank 0 nRanks 8 nNodes 1 ..."
        with open(log) as fh:
            txt = fh.read()
        m = re.search(r"nRanks (\d+)", txt)
        info["nccl_comm_nranks"] = int(m.group(1)) if m else None
        lines = [ln.strip() for ln in txt.splitlines() if "nRanks" in ln or "NVLS" in ln]
        info["nccl_init_lines"] = [ln[-160:] for ln in lines[:4]]
    return info


def max_over_ranks(value: float, ws: int, device) -> float:
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU reference
def _ref_native_build():
    """Rebuild the reference kernels with the reference's -march=native on this host
    (setup.py:10) from the C that cython generated in the build container."""
    stamp = os.path.join(ROOT, "oracle", "_ref", ".native_host")
    host = platform.node()
    if os.path.exists(stamp) and open(stamp).read().strip() == host:
        return "native"
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "_kernels_cy.c")):
        return "prebuilt"
    try:
        subprocess.run([os.path.join(ROOT, "oracle", "build_ref.sh"), "--cc-only"], check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=300,
                       env=dict(os.environ, PYTHON=sys.executable))
        with open(stamp, "w") as fh:
            fh.write(host)
        return "native"
    except Exception:
        return "prebuilt"


class RefRunner:
    """The reference's fused ConvWorkspace.run (pipeline.py:142-150 ->
    _kernels_cy.pyx:242 xnor_reconstruct) over (image, filter) pairs, filters
    prebuilt and inputs padded outside the timing (the reference protocol,
    bench.py:5-7,234-237)."""

    def __init__(self, cfg, seed=0):
        import numpy as np
        from oracle import oracle as O
        self.march = _ref_native_build()
        self.O = O
        self.R = O.RefKernels()
        N, C, H, W, Oc, k = cfg
        self.cfg = cfg
        self.k = k
        self.pad = (k - 1) // 2
        rng = np.random.default_rng((seed, 3))
        n_img = min(N, 8)
        self.x = rng.uniform(-1, 1, (n_img, C, H, W)).astype(np.float32)
        w = rng.uniform(-1, 1, (Oc, C, k, k)).astype(np.float32)
        self.filters = [O.build_filter(w[o]) for o in range(Oc)]
        self.ws = [self.R.workspace(self.x[i], self.pad, k, k) for i in range(n_img)]
        self.threads = os.cpu_count() or 1

    def pair_rates(self, budget_s: float, threads=None, reps: int = 5):
        """reps samples of pair_rate over budget_s in total: [s_per_pair], pairs."""
        out, total = [], 0
        for _ in range(reps):
            sp, n = self.pair_rate(budget_s / reps, threads)
            out.append(sp)
            total += n
        return out, total

    def pair_rate(self, budget_s: float, threads=None):
        """Time (image, filter) pairs for ~budget_s seconds; returns (s_per_pair, pairs)."""
        threads = threads or self.threads
        padded, out = self.ws[0]
        self.R.run(padded, out, self.filters[0], self.k, self.k, threads)  # warm the OpenMP team
        pairs, t0 = 0, time.perf_counter()
        while True:
            padded, out = self.ws[(pairs // len(self.filters)) % len(self.ws)]
            self.R.run(padded, out, self.filters[pairs % len(self.filters)], self.k, self.k, threads)
            pairs += 1
            el = time.perf_counter() - t0
            if el >= budget_s and pairs >= 4:
                return el / pairs, pairs


# ------------------------------------------------------------------ GPU arm
def numa_local_cpus(dev) -> set[int] | None:
    """The host CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI device)."""
    import torch
    try:
        p = torch.cuda.get_device_properties(dev)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as fh:
            spec = fh.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


class numa_local:
    """Run the block (pinned host allocations, first touch) on the GPU-local NUMA
    node's CPUs, then restore the affinity (the CPU baseline uses every core)."""

    def __init__(self, dev):
        self.cpus = numa_local_cpus(dev)
        self.saved = None

    def __enter__(self):
        if self.cpus:
            self.saved = os.sched_getaffinity(0)
            os.sched_setaffinity(0, self.cpus)
        return self

    def __exit__(self, *a):
        if self.saved:
            os.sched_setaffinity(0, self.saved)


def pcie_peak(dev, nbytes: int = 256 << 20, reps: int = 5) -> dict:
    """Host<->device copy bandwidth of this box, measured in the same run with the
    same kind of buffers as e2e (pinned, GPU-local NUMA node): H2D alone, D2H alone,
    and both at once on two streams (what the pipelined e2e path overlaps)."""
    import torch
    with numa_local(dev):
        h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(h2d: bool, d2h: bool) -> float:
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_src, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_dst.copy_(d_b, non_blocking=True)
        s1.wait_stream(s2)
        e1.record(s1)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) * 1e-3

    timed(True, True)  # warm
    t_h2d, t_d2h, t_bi = timed(True, False), timed(False, True), timed(True, True)
    return {"h2d_GBs": nbytes * reps / t_h2d / 1e9, "d2h_GBs": nbytes * reps / t_d2h / 1e9,
            "bidir_GBs": 2 * nbytes * reps / t_bi / 1e9, "bytes_per_copy": nbytes,
            "numa_local_cpus": len(numa_local_cpus(dev) or ())}


def run_ours(args, cfg_name):
    import numpy as np
    import torch
    from paper_2007_14178_b200 import XnorConv2d, ops

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    init_dist(dev)
    N, C, H, W, Oc, k = CONFIGS[cfg_name]
    pad = (k - 1) // 2
    # synthetic data, seeded per rank: rank r holds images [r*N, (r+1)*N) of the global batch
    g = torch.Generator(device="cpu").manual_seed(1000 + rank)
    with numa_local(dev):  # the e2e host buffers live on the GPU's NUMA node
        x_host = (torch.rand((N, C, H, W), generator=g) * 2 - 1).pin_memory()
    w_host = torch.rand((Oc, C, k, k), generator=torch.Generator().manual_seed(7)) * 2 - 1
    x = x_host.to(dev)
    layer = XnorConv2d(w_host.to(dev), pad=pad, variant=args.variant)
    filt = layer.filters
    oh, ow = ops.out_dims(H, W, k, k, pad)
    y = torch.empty((N, Oc, oh, ow), dtype=torch.float32, device=dev)
    kernel = layer.kernel_for(x.shape)  # "auto" resolves per shape
    bits = torch.empty((N, H, W, ops.words(C)), dtype=torch.int32, device=dev)  # every conv kernel reads bits
    A = torch.empty((N, H, W), dtype=torch.float32, device=dev)
    K = torch.empty((N, oh, ow), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    from paper_2007_14178_b200._lib import check, lib
    L = lib()
    sptr = stream.cuda_stream
    pack_fn = L.xnc_pack_input

    def conv_call():
        if kernel == "umma":
            check(L.xnc_xnor_conv_umma(bits.data_ptr(), filt.wq.data_ptr(), filt.sw.data_ptr(), K.data_ptr(),
                                       filt.alpha.data_ptr(), N, C, H, W, Oc, k, k, pad, y.data_ptr(), None,
                                       sptr), "conv_umma")
        else:
            check(L.xnc_xnor_conv_variant(ops.VARIANTS[kernel], bits.data_ptr(), filt.wbits.data_ptr(),
                                          K.data_ptr(), filt.alpha.data_ptr(), N, C, H, W, Oc, k, k, pad,
                                          y.data_ptr(), None, sptr), "conv")

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        check(pack_fn(x.data_ptr(), N, C, H, W, bits.data_ptr(), A.data_ptr(), sptr), "pack")
        if ev is not None:
            ev[1].record(stream)
        check(L.xnc_scale_map(A.data_ptr(), N, H, W, k, k, pad, K.data_ptr(), sptr), "scale")
        if ev is not None:
            ev[2].record(stream)
        conv_call()
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        # keep the sampler alive over a short tail so very short runs still get samples
        if t_start.elapsed_time(t_end) < 500:
            for _ in range(max(1, int(500 / max(t_start.elapsed_time(t_end) / args.steps, 0.05)))):
                step()
            torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    ms_total = t_start.elapsed_time(t_end)
    ms_total = max_over_ranks(ms_total, ws, dev)
    ms_step = ms_total / args.steps
    per_kernel = {
        "pack_input": statistics.mean(e[0].elapsed_time(e[1]) for e in evs),
        "scale_map": statistics.mean(e[1].elapsed_time(e[2]) for e in evs),
        "xnor_conv": statistics.mean(e[2].elapsed_time(e[3]) for e in evs),
    }
    bops_rank = binops(N, C, H, W, Oc, k)
    value = bops_rank * ws / (ms_step * 1e-3) / 1e9
    imgs = N * ws / (ms_step * 1e-3)

    # ---- e2e: the public API call with HOST buffers: XnorConv2d.forward(x_host) copies
    # pinned x host->device, computes, and copies y device->host, the copies of one
    # chunk overlapped with the compute of the next (layer.forward_host).  Timed with
    # CUDA events bracketing all three streams (start before the first H2D is issued,
    # end after the last D2H completes).
    with numa_local(dev):
        y_host = torch.empty((N, Oc, oh, ow), dtype=torch.float32).pin_memory()
    e2e_steps = max(2, min(args.steps, 5))
    layer.forward(x_host, out=y_host)
    torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        layer.forward(x_host, out=y_host)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps, ws, dev)
    h2d_b, d2h_b = x_host.numel() * 4, y_host.numel() * 4
    e2e = {"value": bops_rank * ws / (e2e_ms * 1e-3) / 1e9, "unit": "Gbinop/s",
           "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
           "ms_per_step": e2e_ms,
           "api": "XnorConv2d.forward(host tensor) -> pipelined H2D / K1-K4 / D2H on 3 streams",
           "host_buffers": "pinned, allocated on the GPU's NUMA node"}
    try:  # e2e is PCIe-bound: report it against this box's copy bandwidth, same run
        pc = pcie_peak(dev)
        floor_ms = max(h2d_b / (pc["h2d_GBs"] * 1e9), d2h_b / (pc["d2h_GBs"] * 1e9),
                       (h2d_b + d2h_b) / (pc["bidir_GBs"] * 1e9)) * 1e3
        e2e["pcie"] = pc
        e2e["pcie_floor_ms"] = floor_ms
        e2e["frac_of_pcie_floor"] = floor_ms / e2e_ms
    except Exception as exc:
        e2e["pcie"] = {"error": repr(exc)}

    # ---- vanilla GPU row (Table 1): the same layer as a
    # full-precision cuDNN conv2d (FP32 and TF32), inputs resident, same event protocol
    def vanilla_ms(xv, wv, pad_v, tf32):
        import torch.nn.functional as F
        saved = (torch.backends.cudnn.allow_tf32, torch.backends.cudnn.benchmark)
        torch.backends.cudnn.allow_tf32, torch.backends.cudnn.benchmark = tf32, True
        try:
            for _ in range(3):
                F.conv2d(xv, wv, padding=pad_v)
            torch.cuda.synchronize(dev)
            a_v, b_v = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_v.record(stream)
            for _ in range(5):
                F.conv2d(xv, wv, padding=pad_v)
            b_v.record(stream)
            torch.cuda.synchronize(dev)
            return a_v.elapsed_time(b_v) / 5
        finally:
            torch.backends.cudnn.allow_tf32, torch.backends.cudnn.benchmark = saved

    vanilla = None
    if not args.no_ksweep and cfg_name == "C3":
        w_dev = w_host.to(dev)
        fp32_ms, tf32_ms = vanilla_ms(x, w_dev, pad, False), vanilla_ms(x, w_dev, pad, True)
        vanilla = {"what": "torch.nn.functional.conv2d (cuDNN), same x / w, float outputs, resident",
                   "fp32_ms": fp32_ms, "tf32_ms": tf32_ms, "xnor_step_ms": ms_step,
                   "speedup_vs_fp32": fp32_ms / ms_step, "speedup_vs_tf32": tf32_ms / ms_step}
        del w_dev

    # ---- k-sweep (BASELINE config 2): GPU throughput per kernel size, same protocol
    ksweep = None
    if not args.no_ksweep and cfg_name == "C3":
        ksweep = {}
        for kname in ("C2k3", "C2k5", "C2k7"):
            Nk, Ck, Hk, Wk, Ok, kk = CONFIGS[kname]
            xk = (torch.rand((Nk, Ck, Hk, Wk), generator=g) * 2 - 1).to(dev)
            lk = XnorConv2d((torch.rand((Ok, Ck, kk, kk), generator=g) * 2 - 1).to(dev), variant=args.variant)
            yk = lk.forward(xk)
            for _ in range(3):
                lk.forward(xk, out=yk)
            torch.cuda.synchronize(dev)
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 30  # C2k3 is ~0.09 ms: 10 reps left +-8 % run-to-run spread
            a_ev.record(stream)
            for _ in range(reps):
                lk.forward(xk, out=yk)
            b_ev.record(stream)
            torch.cuda.synchronize(dev)
            ms_k = a_ev.elapsed_time(b_ev) / reps
            # the same layer forward replayed from a CUDA graph: at these sizes the three
            # launches through Python leave the GPU idle between kernels
            ms_graph = None
            if not args.no_graph:
                try:
                    gk = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gk):
                        lk.forward(xk, out=yk)
                    gk.replay()
                    torch.cuda.synchronize(dev)
                    a_ev.record(stream)
                    for _ in range(reps):
                        gk.replay()
                    b_ev.record(stream)
                    torch.cuda.synchronize(dev)
                    ms_graph = a_ev.elapsed_time(b_ev) / reps
                    del gk
                except Exception as exc:  # reported, the eager number stands
                    ms_graph = f"capture failed: {exc!r}"[:200]
            v32 = vanilla_ms(xk, lk.weight, (kk - 1) // 2, False)
            ksweep[kname] = {"k": kk, "ms_per_layer": ms_k, "ms_per_layer_graph": ms_graph,
                             "gpu_Gbinop_s": binops(Nk, Ck, Hk, Wk, Ok, kk) / (ms_k * 1e-3) / 1e9,
                             "vanilla_fp32_ms": v32, "speedup_vs_vanilla_fp32": v32 / ms_k}
            del xk, yk, lk

    result = None
    if rank == 0:
        peaks, peaks_src = read_peaks()
        f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        props = torch.cuda.get_device_properties(dev)
        sms = props.multi_processor_count
        peak_probe = None
        peak_alt = None
        if kernel == "umma":
            # MEASURED_PEAKS has no int8 entry, so the stated peak is our own measured
            # tcgen05 kind::i8 rate (tools/microbench/umma_probe.cu: 7874 MAC/clk/SM,
            # back-to-back M128 N256 K32 MMAs from resident smem) at sm_max_mhz, x 2
            # binops per MAC: 4580 Tbinop/s.  Beside it: B200_PROFILING.md's nominal dense
            # fp8/int8 4.5 POPS and 2 x the driver-measured bf16 burst.
            bf16 = peaks.get("bf16_tflops")
            peak_probe = 2 * UMMA_I8_MAC_PER_CLK_SM * sms * f_max / 1e12
            peak_tbinops = peak_probe
            basis = (f"measured: tcgen05.mma kind::i8 probe {UMMA_I8_MAC_PER_CLK_SM} MAC/clk/SM "
                     f"(profiles/umma_probe_r1.jsonl) x {sms} SMs x {f_max / 1e6:.0f} MHz x 2 binops/MAC")
            peak_alt = {"nominal_B200_PROFILING_int8_4.5POPS": 4500.0,
                        "2x_measured_bf16_burst": 2.0 * float(bf16) if bf16 else None}
            bound = "tensor"
        else:
            peak_tbinops = 2 * POPC_LANES_PER_CLK_SM * 32 * sms * f_max / 1e12
            bound, basis = "popc", (f"{POPC_LANES_PER_CLK_SM} POPC lanes/clk/SM (measured microbench) x 32 "
                                    f"bit-MACs x 2 binops x {sms} SMs x {f_max / 1e6:.0f} MHz "
                                    f"(sm_max_mhz, {peaks_src})")
        conv_ms = per_kernel["xnor_conv"]
        achieved = bops_rank / (conv_ms * 1e-3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", f"ncu_{cfg_name}_conv_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        packed = N * H * W * 4 * ops.words(C)
        pack_bytes = 4.0 * N * C * H * W + packed + 4.0 * N * H * W
        result = {
            "metric": METRIC, "value": value, "unit": "Gbinop/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": ("u8 x s8 -> s32 (tcgen05 kind::i8 over 1-bit signs: d = [x < 0] bytes x +-1 filter "
                      "signs, exact) + f32 K/alpha" if kernel == "umma" else
                      "u32 (1-bit signs, XOR + POPC into int32 accumulators) + f32 K/alpha"),
            "data": "synthetic U(-1,1) float32 activations and weights, seeded",
            "config": {"workload": CONFIG_TEXT[cfg_name], "name": cfg_name, "batch_per_gpu": N,
                       "global_batch": N * ws, "C_in": C, "C_out": Oc, "H": H, "W": W, "k": k, "pad": pad,
                       "parallelism": f"batch-sharded x{ws}, per-rank weight replicas, no collective",
                       "variant": args.variant, "conv_kernel": kernel,
                       "l2": "inputs 4*N*C*H*W bytes > 126 MB L2; no flush needed"},
            "images_per_s": imgs,
            "kernel_ms": per_kernel,
            "gpu_launches": 3 * args.steps,
            "roofline": {"bound": bound, "kernel": f"xnor_conv (K3+K4, {kernel})", "achieved": achieved,
                         "peak": peak_tbinops, "unit": "Tbinop/s", "frac": achieved / peak_tbinops,
                         "traffic": traffic,
                         "peak_basis": basis,
                         "peak_alternatives_Tbinop_s": peak_alt,
                         "frac_of_nominal_4500": (achieved / 4500.0) if peak_probe else None},
            "pack_roofline": {"bound": "hbm", "achieved": pack_bytes / (per_kernel["pack_input"] * 1e-3) / 1e9,
                              "peak": float(peaks.get("hbm_gbs", 6650.0)), "unit": "GB/s",
                              "frac": pack_bytes / (per_kernel["pack_input"] * 1e-3) / 1e9 /
                                      float(peaks.get("hbm_gbs", 6650.0))},
            "e2e": e2e,
            "clocks": clk.summary(),
            "ksweep": ksweep,
            "vanilla_gpu": vanilla,
            "gpu": props.name,
            "comm": comm_info(),
        }
    if ws > 1:
        torch.distributed.barrier()
    return result


def run_network(args, cfg_name):
    """C4 / C5: full XNOR-Net AlexNet forward.  Binary layers through XnorConv2d
    (tcgen05 / popc kernels), conv1 / pools / fc8 full precision via torch.
    C5 shards a global batch of 2048 contiguously over the ranks (strong scaling,
    per-rank weight replicas from the same seed, no collective on the hot path)."""
    import torch
    from paper_2007_14178_b200.network import BINARY_MACS_PER_IMAGE, XnorNetAlexNet
    from paper_2007_14178_b200.shard import shard_bounds

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    init_dist(dev)
    gb = NETWORK_CONFIGS[cfg_name] if cfg_name == "C5" else NETWORK_CONFIGS[cfg_name] * ws
    a, b = shard_bounds(gb, ws, rank)
    N = b - a
    g = torch.Generator().manual_seed(1000 + rank)
    x_host = (torch.rand((N, 3, 224, 224), generator=g) * 2 - 1).pin_memory()
    x = x_host.to(dev)
    net = XnorNetAlexNet(dev, seed=7, variant=args.variant)
    stream = torch.cuda.current_stream(dev)
    # the forward as one CUDA graph (same kernels; removes the per-layer host launches)
    graph, logits = net.capture(x) if not args.no_graph else (None, None)
    step = graph.replay if graph is not None else (lambda: net(x))
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            out = step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if graph is None:
        logits = out
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws, dev)
    # e2e: host images in (pinned -> the graph's input buffer), host logits out, copies timed
    logits_host = torch.empty(tuple(logits.shape), dtype=torch.float32).pin_memory()
    e0.record(stream)
    for _ in range(max(2, min(args.steps, 5))):
        if graph is not None:
            x.copy_(x_host, non_blocking=True)
            graph.replay()
            logits_host.copy_(logits, non_blocking=True)
        else:
            logits_host.copy_(net(x_host.to(dev, non_blocking=True)), non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / max(2, min(args.steps, 5)), ws, dev)
    bops = 2.0 * BINARY_MACS_PER_IMAGE * gb
    per_step = count_own_kernels(lambda: net(x)) if rank == 0 else None  # eager: same kernels as the graph
    res = None
    if rank == 0:
        res = {"metric": METRIC, "value": bops / (ms * 1e-3) / 1e9, "unit": "Gbinop/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "strong" if cfg_name == "C5" else "weak", "vs_baseline": None,
               "dtype": ("1-bit signs (binary layers); conv1 f32 in / TF32 multiply on our tcgen05 kernel; fc8 cuBLAS TF32"
                         if net.conv1 == "tcgen05" else
                         "1-bit signs (binary layers); conv1 / fc8 full precision on cuDNN / cuBLAS with TF32"),
               "data": "synthetic U(-1,1), random-init weights",
               "config": {"workload": CONFIG_TEXT[cfg_name], "name": cfg_name, "global_batch": gb,
                          "batch_per_gpu": N, "variant": args.variant,
                          "binary_kernels": net.binary_kernels(N),
                          "execution": "CUDA graph of the forward" if graph is not None else "eager",
                          "parallelism": f"batch-sharded x{ws}, per-rank weight replicas, no collective"},
               "images_per_s": gb / (ms * 1e-3),
               "binops_per_image": 2.0 * BINARY_MACS_PER_IMAGE,
               "gpu_launches": None if per_step is None else per_step * args.steps,
               "gpu_launches_note": "our (xnc::) kernels per forward, counted with torch.profiler on one extra "
                                    "forward outside the timed region, x steps; cuDNN / cuBLAS / torch kernels "
                                    "(conv1, fc8, zero-fill) not counted",
               "e2e": {"value": bops / (e2e_ms * 1e-3) / 1e9, "unit": "Gbinop/s",
                       "h2d_bytes_per_step": x_host.numel() * 4 * ws, "d2h_bytes_per_step": logits_host.numel() * 4 * ws,
                       "ms_per_step": e2e_ms, "api": "XnorNetAlexNet.forward"},
               "clocks": clk.summary(), "comm": comm_info()}
    if ws > 1:
        torch.distributed.barrier()
    return res


def binary_stack_summary(steps=10, warmup=3):
    """C3 as one layer of a stack of binary layers (its input already in K1 form, the
    next layer's batch norm folded in): the float epilogue followed by the next
    layer's K1 pass, vs the sign-emitting epilogue that writes the next layer's K1
    output directly (north star item 4).  Inputs resident; CUDA events."""
    import torch
    from paper_2007_14178_b200 import XnorConv2d, ops
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.rand((256, 256, 56, 56), device=dev, generator=g) * 2 - 1
    w = torch.rand((256, 256, 3, 3), device=dev, generator=g) * 2 - 1
    bn = (torch.rand(256, device=dev, generator=g) + 0.5, torch.rand(256, device=dev, generator=g) - 0.5)
    layer = XnorConv2d(w, pad=1, variant="auto", out_affine=bn)
    bits, A = ops.pack_input(x)
    p = ops.PackedInput(bits, A, 256)

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / steps

    f_ms = timed(lambda: ops.pack_input(layer.forward(p)))
    e_ms = timed(lambda: layer.forward(p, emit_signs=True))
    bops = 2.0 * 256 * 256 * 56 * 56 * 256 * 9
    return {"workload": "C3 layer inside a stack of binary layers (input and output in K1 form, BN folded)",
            "ms_per_layer_float_epilogue_then_next_k1": f_ms, "ms_per_layer_sign_emitting_epilogue": e_ms,
            "Gbinop_s_sign_emitting": bops / (e_ms * 1e-3) / 1e9, "speedup": f_ms / e_ms}


def count_own_kernels(fn) -> int | None:
    """Number of this library's kernels (names in namespace xnc::) one call of fn
    launches, from a torch.profiler trace of one extra call (None if CUPTI is not
    available)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        return sum(1 for n in names if "xnc::" in n)
    except Exception:
        return None


def network_summary(variant="auto", batch=256, steps=5, warmup=3):
    """A short XNOR-Net AlexNet forward timing (BASELINE config 4) for the default
    bench line: images/s at batch 256 on this GPU, inputs resident."""
    import torch
    from paper_2007_14178_b200.network import BINARY_MACS_PER_IMAGE, XnorNetAlexNet
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator().manual_seed(11)
    x = ((torch.rand((batch, 3, 224, 224), generator=g) * 2 - 1)).to(dev)
    net = XnorNetAlexNet(dev, seed=7, variant=variant)
    graph, _ = net.capture(x)
    for _ in range(warmup):
        graph.replay()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    return {"workload": CONFIG_TEXT["C4"], "ms_per_step": ms, "images_per_s": batch / (ms * 1e-3),
            "Gbinop_s": 2.0 * BINARY_MACS_PER_IMAGE * batch / (ms * 1e-3) / 1e9,
            "binary_kernels": net.binary_kernels(batch), "note": "full numbers: bench.py --config C4"}


def cpu_model() -> str:
    """The host CPU model (lscpu's 'Model name', from /proc/cpuinfo)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def cpu_baseline_fields(cfg_name, budget_s, ksweep=None):
    """The reference's fused kernel on this host: all threads (the headline CPU row)
    and threads=1 (the race-free path at every k);
    medians of 5 sub-samples each."""
    cfg = CONFIGS[cfg_name]
    rr = RefRunner(cfg)
    N, C, H, W, Oc, k = cfg
    bops_pair = binops(1, C, H, W, 1, k)
    samples, pairs = rr.pair_rates(budget_s)
    s_pair = statistics.median(samples)
    s1, pairs1 = rr.pair_rates(max(2.0, budget_s / 3), threads=1)
    s1_pair = statistics.median(s1)
    out = {"value": bops_pair / s_pair / 1e9, "unit": "Gbinop/s", "cores": rr.threads, "kind": "reference",
           "sample": f"{pairs} (image, filter) pairs of {cfg_name} through the reference's fused "
                     f"xnor_reconstruct (oracle/_ref, -march={rr.march}), threads={rr.threads}, median of 5",
           "ms_per_pair": s_pair * 1e3, "ms_per_pair_mean": statistics.mean(samples) * 1e3,
           "cpu_model": cpu_model(),
           "threads_1": {"value": bops_pair / s1_pair / 1e9, "unit": "Gbinop/s", "cores": 1,
                         "ms_per_pair": s1_pair * 1e3, "pairs": pairs1,
                         "note": "race-free single-thread fused path (the parity oracle's protocol)"}}
    if ksweep:
        for kname, row in ksweep.items():
            rk = RefRunner(CONFIGS[kname])
            sp_all, _ = rk.pair_rates(max(2.0, budget_s / 4))
            sp1, _ = rk.pair_rates(max(1.5, budget_s / 6), threads=1)
            sp, sp_1 = statistics.median(sp_all), statistics.median(sp1)
            _, Ck, Hk, Wk, _, kk = CONFIGS[kname]
            bk = binops(1, Ck, Hk, Wk, 1, kk)
            row["cpu_Gbinop_s"] = bk / sp / 1e9
            row["cpu_threads"] = rk.threads
            row["cpu_note"] = ("reference fused path, threads>1: output nondeterministic (reference "
                               "race, SURVEY.md section 0 item 6)" if CONFIGS[kname][5] != 3 else
                               "reference fused path")
            row["speedup_vs_cpu"] = row["gpu_Gbinop_s"] / row["cpu_Gbinop_s"]
            row["cpu_threads_1_Gbinop_s"] = bk / sp_1 / 1e9
            row["speedup_vs_cpu_threads_1"] = row["gpu_Gbinop_s"] / row["cpu_threads_1_Gbinop_s"]
    return out


def run_reference(args, cfg_name):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    rr = RefRunner(CONFIGS[cfg_name])
    N, C, H, W, Oc, k = CONFIGS[cfg_name]
    bops_pair = binops(1, C, H, W, 1, k)
    per_step_budget = max(0.5, min(10.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        rr.pair_rate(per_step_budget / 4)
    rates = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s_pair, pairs = rr.pair_rate(per_step_budget)
        rates.append(bops_pair / s_pair / 1e9)
    el = time.perf_counter() - t0
    value = statistics.median(rates)
    return {"metric": METRIC, "value": value, "value_mean": statistics.mean(rates), "unit": "Gbinop/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 tile words + f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": CONFIG_TEXT[cfg_name], "name": cfg_name, "C_in": C, "C_out": Oc,
                       "H": H, "W": W, "k": k, "batch_per_gpu": N},
            "cpu_baseline": {"value": value, "unit": "Gbinop/s", "cores": rr.threads, "kind": "reference",
                             "sample": f"each step ~{per_step_budget:.1f}s of (image, filter) pairs of "
                                       f"{cfg_name} through xnor_reconstruct (oracle/_ref, -march={rr.march})"},
            "e2e": {"value": value, "unit": "Gbinop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run directly (no torchrun around it): re-launch this same
    command line as N ranks under torch.distributed.run on 127.0.0.1, one process
    per GPU.  Rank 0's stdout (the JSON line) passes straight through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))).returncode


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo on CPU) -- rendezvous,
    per-rank batch shards of C5, a rank-local stand-in step on each shard with no
    collective, the barrier + max-over-ranks timing, and rank 0's one JSON line.
    Exercised by tests/test_bench_spawn.py."""
    import torch
    import torch.distributed as dist
    from paper_2007_14178_b200.shard import shard_bounds
    ws, rank, _ = dist_env()
    init_dist(None)
    gb = NETWORK_CONFIGS["C5"]
    a, b = shard_bounds(gb, ws, rank)
    x = torch.arange(a, b, dtype=torch.float64)
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    acc = 0.0
    for _ in range(args.steps):
        acc += float(x.sum())  # this rank's shard only
    ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / max(1, args.steps), ws, None)
    shards = [None] * ws
    if ws > 1:
        dist.all_gather_object(shards, (rank, a, b, acc / max(1, args.steps)))
    else:
        shards = [(rank, a, b, acc / max(1, args.steps))]
    res = None
    if rank == 0:
        covered = sorted((a_, b_) for _, a_, b_, _ in shards)
        res = {"metric": METRIC, "dry_run": True, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": ms, "config": {"workload": CONFIG_TEXT["C5"], "global_batch": gb},
               "shards": [[a_, b_] for a_, b_ in covered],
               "shards_cover_batch": covered[0][0] == 0 and covered[-1][1] == gb and
                                     all(covered[i][1] == covered[i + 1][0] for i in range(len(covered) - 1)),
               "shard_sums_ok": all(abs(s_ - (a_ + b_ - 1) * (b_ - a_) / 2) < 1e-6 for _, a_, b_, s_ in shards),
               "comm": comm_info()}
    if ws > 1:
        dist.barrier()
    return res


def strong_scaling_c5(args):
    """C5 beside the default C3 line: the XNOR-Net forward over a fixed global batch
    of 2048 split across the ranks (strong scaling), so one bench run records both
    curves; the driver's scaling efficiency is computed from `value` (C3, weak)."""
    import copy
    a2 = copy.copy(args)
    a2.steps, a2.warmup = max(5, min(args.steps, 10)), max(3, args.warmup)
    r = run_network(a2, "C5")
    if r is None:
        return None
    return {k: r.get(k) for k in ("value", "unit", "images_per_s", "ms_per_step", "n_gpus", "scaling", "config",
                                  "clocks")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + sorted(NETWORK_CONFIGS), default="C3")
    ap.add_argument("--variant", choices=["popc", "b1mma", "umma", "auto"], default="auto")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-ksweep", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="C4/C5: eager forward instead of the CUDA graph")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU reference work")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only, on CPU with gloo (no GPU): spawn, shards, timing, JSON line")
    ap.add_argument("--no-strong", action="store_true", help="skip the C5 strong-scaling extra")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws_env = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and ws_env == 0:
        sys.exit(spawn_ranks(args.gpus))
    if ws_env and ws_env != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws_env} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.dry_run:
        res = run_dry(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if args.impl == "reference":
        res = run_reference(args, args.config if args.config in CONFIGS else "C3")
    elif args.config in NETWORK_CONFIGS:
        res = run_network(args, args.config)
    else:
        res = run_ours(args, args.config)
        ws, rank, _ = dist_env()
        if args.config == "C3" and not args.no_strong and not args.no_ksweep:
            try:  # every rank runs it (collective timing); rank 0 reports
                c5 = strong_scaling_c5(args)
            except Exception as exc:
                c5 = {"error": repr(exc)}
            if res is not None:
                res["strong_scaling_C5"] = c5
        if res is not None and rank == 0 and ws == 1 and not args.no_ksweep:
            for key, fn in (("network_C4", lambda: network_summary(args.variant)),
                            ("binary_stack_C3", binary_stack_summary)):
                try:  # extras: report a failure, never lose the main line
                    res[key] = fn()
                except Exception as exc:
                    res[key] = {"error": repr(exc)}
        if res is not None and rank == 0 and ws == 1 and not args.no_cpu:
            try:
                res["cpu_baseline"] = cpu_baseline_fields(args.config, args.cpu_budget, res.get("ksweep"))
                res["speedup_vs_cpu_reference"] = res["value"] / res["cpu_baseline"]["value"]
            except Exception as exc:  # report, never fake
                res["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if res is not None:
        print(json.dumps(res), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
