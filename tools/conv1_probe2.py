"""Time the tcgen05 TF32 conv1 at batch 256 (CUDA events, 20 reps) under the
XNC_CONV1_DEBUG switches; one JSON line per process (the switch is read once)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2007_14178_b200 import ops  # noqa: E402

x = torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1
wq = ops.conv1_pack_weights(torch.rand((96, 3, 11, 11), device="cuda") - 0.5)
y = ops.conv1_forward(x, wq)
for _ in range(3):
    ops.conv1_forward(x, wq, out=y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    ops.conv1_forward(x, wq, out=y)
e.record()
torch.cuda.synchronize()
print(json.dumps({"debug": os.environ.get("XNC_CONV1_DEBUG", "0"), "ms": round(s.elapsed_time(e) / 20, 4)}))
