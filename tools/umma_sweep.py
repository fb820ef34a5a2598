"""Profiling sweep of the tcgen05 conv kernel (K3) over env knobs.

Each setting runs in its own process because the library reads XNC_UMMA_DEBUG /
XNC_UMMA_TILE once per process.  Prints one JSON line per (setting, config) with
the conv kernel's average time over `reps` launches (CUDA events, inputs resident).
Debug bits change the results (profiling only): 1 = skip epilogue stores,
2 = load B once, 4 = load the input rows once, 8 = no B barrier protocol,
16 = no tcgen05 fence after B waits.

Usage (on a B200): python tools/umma_sweep.py [--debug 0,1,2,4] [--tile 2,128 1,256]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHAPES = {
    "C3": (256, 256, 56, 56, 256, 3),
    "C2k3": (64, 128, 64, 64, 128, 3),
    "C2k5": (64, 128, 64, 64, 128, 5),
    "C2k7": (64, 128, 64, 64, 128, 7),
    # XNOR-Net AlexNet's binary layers at batch 256 (C4)
    "conv2": (256, 96, 27, 27, 256, 5),
    "conv3": (256, 256, 13, 13, 384, 3),
    "conv4": (256, 384, 13, 13, 384, 3),
    "conv5": (256, 384, 13, 13, 256, 3),
    # fc6 / fc7 at batch 256 as the network runs them: one 1 x 256 image, 1 x 1 taps
    "fc6": (1, 9216, 1, 256, 4096, 1),
    "fc7": (1, 4096, 1, 256, 4096, 1),
}


def child(cfg: str, reps: int) -> None:
    sys.path.insert(0, ROOT)
    import torch
    from paper_2007_14178_b200 import ops

    N, C, H, W, O, k = SHAPES[cfg]
    pad = (k - 1) // 2
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((N, C, H, W), device="cuda", generator=g) * 2 - 1
    w = torch.rand((O, C, k, k), device="cuda", generator=g) * 2 - 1
    filt = ops.pack_weights(w)
    ops.attach_umma_weights(filt, w)
    d, A = ops.pack_input(x)
    K = ops.scale_map(A, k, k, pad)
    y = torch.empty((N, O, H + 2 * pad - k + 1, W + 2 * pad - k + 1), device="cuda")
    for _ in range(3):
        ops.xnor_conv(d, filt, K, pad, variant="umma", y=y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        ops.xnor_conv(d, filt, K, pad, variant="umma", y=y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    prof = None
    if int(os.environ.get("XNC_UMMA_DEBUG", "0")) & 64:
        import ctypes
        import numpy as np
        from paper_2007_14178_b200._lib import lib
        buf = np.zeros((1024, 16), dtype=np.uint64)
        lib().xnc_umma_profile(buf.ctypes.data_as(ctypes.c_void_p), 1024)
        tr = buf[512:].reshape(-1, 2).astype(np.int64)
        tr = tr[: int(np.argmax(tr[1:, 0] == 0)) + 1] if (tr[1:, 0] == 0).any() else tr
        np.save(os.path.join(ROOT, "gpurun_out", f"trace_{cfg}.npy"), tr)
        gaps = np.diff(tr[:, 0])
        print(json.dumps({"trace_chunks": int(len(tr)), "gap_mean": float(gaps.mean()),
                          "gap_p50": float(np.median(gaps)), "gap_p90": float(np.percentile(gaps, 90)),
                          "gap_max": float(gaps.max()), "wait_mean": float(tr[:, 1].mean()),
                          "wait_p90": float(np.percentile(tr[:, 1], 90))}), flush=True)
    if int(os.environ.get("XNC_UMMA_DEBUG", "0")) & 128:
        import ctypes
        import numpy as np
        from paper_2007_14178_b200._lib import lib
        buf = np.zeros((148, 16), dtype=np.uint64)
        lib().xnc_umma_profile(buf.ctypes.data_as(ctypes.c_void_p), 148)
        buf[:, 9] = 0
        tot = buf[:, 0].astype(np.float64)
        names = ["issuer_total", "wait_t_empty", "wait_a_full", "wait_b_full", "mmas", "epi_total",
                 "epi_wait_t_full", "bprod_wait_b_empty", "aprod_wait_a_empty", "issue_blocks", "epi_ld",
                 "epi_store"]
        lead = buf[0::2]  # CTA pairs: the MMA issuer runs on the even (leader) CTA
        prof = {n: round(float(buf[:, i].astype(np.float64).mean()), 0) for i, n in enumerate(names)}
        for i in (0, 1, 2, 3, 4):
            prof[names[i]] = round(float(lead[:, i].astype(np.float64).mean()), 0)
        prof["issuer_total_max"] = float(tot.max())
        prof["cycles_per_mma"] = round(float((lead[:, 0] / np.maximum(lead[:, 4], 1)).mean()), 2)
    macs = N * O * (H + 2 * pad - k + 1) * (W + 2 * pad - k + 1) * C * k * k
    print(json.dumps({"cfg": cfg, "debug": os.environ.get("XNC_UMMA_DEBUG", "0"),
                      "tile": os.environ.get("XNC_UMMA_TILE", "default"), "ms": round(ms, 4),
                      "Tbinop_s": round(2 * macs / ms / 1e9, 1), "prof": prof}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--child", default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--debug", default="0")
    ap.add_argument("--tile", nargs="*", default=["default"])
    ap.add_argument("--cfgs", default="C3")
    a = ap.parse_args()
    if a.child:
        child(a.child, a.reps)
        return
    for tile in a.tile:
        for dbg in a.debug.split(","):
            for cfg in a.cfgs.split(","):
                env = dict(os.environ, XNC_UMMA_DEBUG=dbg)
                if tile != "default":
                    env["XNC_UMMA_TILE"] = tile
                try:
                    subprocess.run([sys.executable, __file__, "--child", cfg, "--reps", str(a.reps)],
                                   env=env, check=False, timeout=60)
                except subprocess.TimeoutExpired:
                    print(json.dumps({"cfg": cfg, "debug": dbg, "tile": tile, "error": "timeout"}), flush=True)


if __name__ == "__main__":
    main()
