"""Per-stage CUDA-event timing of the XNOR-Net AlexNet forward (BASELINE config 4)
at batch 256: front end (conv1 s2d + ReLU + pool), each binary layer, pools, fc8.
Profiling aid only; prints one JSON line.  Usage (on a B200): python tools/c4_stages.py [batch]"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2007_14178_b200.network import BINARY_LAYERS, XnorNetAlexNet, _tf32_full_precision_layers  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    net = XnorNetAlexNet("cuda", seed=7)
    x = torch.rand((batch, 3, 224, 224), device="cuda") * 2 - 1
    for _ in range(3):
        net(x)
    torch.cuda.synchronize()
    reps = 10
    names = ["front_end"] + [n for n, *_ in BINARY_LAYERS] + ["fc8"]  # pools run inside conv3 / fc6
    acc = {n: 0.0 for n in names}
    with torch.no_grad(), _tf32_full_precision_layers():
        for _ in range(reps):
            ev = []

            def mark(name):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))
            mark("start")
            h = net.front_end(x)
            mark("front_end")
            for name, *_ in BINARY_LAYERS:
                h = net.binary[name](h.contiguous())
                mark(name)
            F.linear(h.flatten(1), net.fc8_w, net.fc8_b)
            mark("fc8")
            torch.cuda.synchronize()
            for (_, a), (n, b) in zip(ev, ev[1:]):
                acc[n] += a.elapsed_time(b)
    out = {n: round(v / reps, 4) for n, v in acc.items()}
    out["total"] = round(sum(out.values()), 4)
    out["kernels"] = net.binary_kernels(batch)
    print(json.dumps({"bench": "c4_stages", "batch": batch, "ms": out}))


if __name__ == "__main__":
    main()
