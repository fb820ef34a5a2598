"""K1 / K2 / conv split of the XNOR-Net binary conv layers at batch 256 (inputs
resident, CUDA events).  Profiling aid; JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2007_14178_b200 import XnorConv2d, ops  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4)


for name, (C, S, O, k, pad) in {"conv2": (96, 27, 256, 5, 2), "conv3": (256, 13, 384, 3, 1),
                                "conv4": (384, 13, 384, 3, 1), "conv5": (384, 13, 256, 3, 1)}.items():
    x = torch.rand((256, C, S, S), device="cuda") * 2 - 1
    w = torch.rand((O, C, k, k), device="cuda") * 2 - 1
    layer = XnorConv2d(w, pad=pad, variant="auto")
    bits, A = ops.pack_input(x)
    K = ops.scale_map(A, k, k, pad)
    r = {"layer": t(lambda: layer.forward(x)), "k1": t(lambda: ops.pack_input(x)),
         "k2": t(lambda: ops.scale_map(A, k, k, pad)),
         "conv": t(lambda: ops.xnor_conv(bits, layer.filters, K, pad, variant="umma"))}
    print(json.dumps({"layer": name, "ms": r}), flush=True)
