"""Time K1 (xnc_pack_input) at C3 for alternative builds of the library (XNC_LIB)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2007_14178_b200 import ops  # noqa: E402

N, C, H, W = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 256, 56, 56))]
x = torch.rand((N, C, H, W), device="cuda") * 2 - 1
for _ in range(3):
    ops.pack_input(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    ops.pack_input(x)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
nbytes = 4 * N * C * H * W + 4 * N * H * W * ((C + 31) // 32) + 4 * N * H * W
print(json.dumps({"lib": os.environ.get("XNC_LIB", "default"), "ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1)}))
