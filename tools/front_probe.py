"""Split the C4 front end (conv1 as space-to-depth 3x3 on cuDNN TF32, ReLU, max-pool
3/2, then conv2's K1) into its pieces at batch 256, NCHW vs channels-last.
Profiling aid; prints one JSON line."""
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
bn2 = net.bn["conv2"]
with torch.no_grad(), _tf32_full_precision_layers():
    for fmt in ("nchw", "nhwc"):
        cl = fmt == "nhwc"
        w = net.conv1_w_s2d.contiguous(memory_format=torch.channels_last) if cl else net.conv1_w_s2d
        r[f"{fmt}_s2d"] = t(lambda: ops.pad_space_to_depth(x, 2, 4, channels_last=cl))
        xs = ops.pad_space_to_depth(x, 2, 4, channels_last=cl)
        r[f"{fmt}_conv"] = t(lambda: F.conv2d(xs, w, net.conv1_b))
        h = F.conv2d(xs, w, net.conv1_b)
        r[f"{fmt}_conv_out_cl"] = h.is_contiguous(memory_format=torch.channels_last) and not h.is_contiguous()
        r[f"{fmt}_relu_pool"] = t(lambda: ops.max_pool(h, 3, 2, relu=True))
        p = ops.max_pool(h, 3, 2, relu=True)
        r[f"{fmt}_conv2_k1"] = t(lambda: ops.pack_input(p, in_affine=bn2))
    r["torch_pad_s2d"] = t(lambda: F.pixel_unshuffle(F.pad(x, (2, 2, 2, 2)), 4))
    r["front_end"] = t(lambda: net.front_end(x))
print(json.dumps({"bench": "front_probe", "ms": r}))
