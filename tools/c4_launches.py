"""Every kernel of one C4 forward (CUDA graph replay) in launch order with its
device time, from a torch.profiler trace; batch from argv (default 256).
Profiling aid; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2007_14178_b200.network import XnorNetAlexNet  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
net = XnorNetAlexNet("cuda", seed=7)
x = torch.rand((batch, 3, 224, 224), device="cuda") * 2 - 1
graph, _ = net.capture(x)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    graph.replay()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
rows = [[round(e.time_range.start, 1), round(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total, 1),
         e.name[:70]] for e in ev]
print(json.dumps({"bench": "c4_launches", "batch": batch, "launches": rows,
                  "total_us": round(sum(r[1] for r in rows), 1)}))
