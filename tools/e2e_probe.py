"""C3 through host buffers (XnorConv2d.forward_host) for several chunk sizes, and the
raw PCIe rates for one direction / both directions.  Profiling aid; JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2007_14178_b200 import XnorConv2d  # noqa: E402

N, C, H, W, O = 256, 256, 56, 56, 256
g = torch.Generator().manual_seed(0)
x = (torch.rand((N, C, H, W), generator=g) * 2 - 1).pin_memory()
w = (torch.rand((O, C, 3, 3), generator=g) * 2 - 1).cuda()
layer = XnorConv2d(w, pad=1, variant="auto")
out = torch.empty((N, O, H, W), dtype=torch.float32).pin_memory()
for chunk in (4, 8, 12, 16, 32):
    for _ in range(2):
        layer.forward_host(x, out=out, chunk=chunk)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        layer.forward_host(x, out=out, chunk=chunk)
    e.record()
    torch.cuda.synchronize()
    print(json.dumps({"chunk": chunk, "ms": round(s.elapsed_time(e) / 3, 3)}), flush=True)
