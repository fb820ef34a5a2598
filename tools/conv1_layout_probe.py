import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, torch.nn.functional as F
from paper_2007_14178_b200.network import XnorNetAlexNet, _tf32_full_precision_layers
from paper_2007_14178_b200 import ops
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4)
net = XnorNetAlexNet("cuda", seed=7)
x = torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1
r = {}
with torch.no_grad(), _tf32_full_precision_layers():
    xs = ops.pad_space_to_depth(x, 2, 4)
    w = net.conv1_w_s2d
    r["nchw"] = t(lambda: F.conv2d(xs, w, net.conv1_b))
    xl = xs.contiguous(memory_format=torch.channels_last); wl = w.contiguous(memory_format=torch.channels_last)
    r["nhwc"] = t(lambda: F.conv2d(xl, wl, net.conv1_b))
    hl = F.conv2d(xl, wl, net.conv1_b)
    r["nhwc_out_is_cl"] = hl.is_contiguous(memory_format=torch.channels_last)
    r["to_cl"] = t(lambda: xs.contiguous(memory_format=torch.channels_last))
    r["bf16_nhwc"] = t(lambda: F.conv2d(xl.bfloat16(), wl.bfloat16(), net.conv1_b.bfloat16()))
    # as a GEMM via unfold? skip
print(json.dumps(r))
