"""C3 layer step through XnorConv2d (device input): the fused launch vs the three
launches (XNC_FUSED=0), CUDA events, 20 reps.  One JSON line per process."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2007_14178_b200 import XnorConv2d  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
N, C, H, W, O, k = {"C3": (256, 256, 56, 56, 256, 3), "C2k3": (64, 128, 64, 64, 128, 3)}[cfg]
x = torch.rand((N, C, H, W), device="cuda") * 2 - 1
layer = XnorConv2d(torch.rand((O, C, k, k), device="cuda") - 0.5, pad=(k - 1) // 2)
y = layer(x)
for _ in range(3):
    layer(x, out=y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    layer(x, out=y)
e.record()
torch.cuda.synchronize()
print(json.dumps({"cfg": cfg, "fused": os.environ.get("XNC_FUSED", "1"), "ms": round(s.elapsed_time(e) / 20, 4)}))
