"""Split the C4 front end (conv1 as space-to-depth 3x3 on cuDNN TF32, ReLU, max-pool
3/2) into its pieces at batch 256.  Profiling aid; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2007_14178_b200 import ops  # noqa: E402
from paper_2007_14178_b200.network import XnorNetAlexNet, _tf32_full_precision_layers  # noqa: E402


def t(fn, reps=10):
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


net = XnorNetAlexNet("cuda", seed=7)
x = torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1
r = {}
with torch.no_grad(), _tf32_full_precision_layers():
    xs = F.pixel_unshuffle(F.pad(x, (2, 2, 2, 2)), 4)
    r["torch_pad_s2d"] = t(lambda: F.pixel_unshuffle(F.pad(x, (2, 2, 2, 2)), 4))
    r["our_pad_s2d"] = t(lambda: ops.pad_space_to_depth(x, 2, 4))
    r["conv"] = t(lambda: F.conv2d(xs, net.conv1_w_s2d, net.conv1_b))
    h = F.conv2d(xs, net.conv1_w_s2d, net.conv1_b)
    r["relu"] = t(lambda: F.relu(h))
    hr = F.relu(h)
    r["torch_pool"] = t(lambda: F.max_pool2d(hr, 3, 2))
    r["our_pool"] = t(lambda: ops.max_pool(hr, 3, 2))
    r["our_relu_pool"] = t(lambda: ops.max_pool(h, 3, 2, relu=True))
    r["front_end"] = t(lambda: net.front_end(x))
print(json.dumps({"bench": "front_probe", "ms": r, "conv_out": list(h.shape)}))
