"""Per-kernel device time of one C4 forward (CUDA graph replay) at batch 256, from a
torch.profiler (CUPTI) trace.  Profiling aid; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2007_14178_b200.network import XnorNetAlexNet  # noqa: E402

net = XnorNetAlexNet("cuda", seed=7)
x = torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1
graph, _ = net.capture(x)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name[:90]
    rows.setdefault(k, []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
out = sorted(((sum(v) / 5.0, len(v) // 5, k) for k, v in rows.items()), reverse=True)
print(json.dumps({"bench": "c4_kernels", "us_per_forward": [[round(t, 1), n, k] for t, n, k in out],
                  "total_us": round(sum(t for t, _, _ in out), 1)}))
