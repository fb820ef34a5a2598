import sys, json, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2007_14178_b200 import XnorConv2d, ops
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4)
for (N, C, S, O, k) in [(256, 256, 6, 4096, 6), (256, 4096, 1, 4096, 1)]:
    x = torch.rand((N, C, S, S), device="cuda") * 2 - 1
    w = torch.rand((O, C, k, k), device="cuda") * 2 - 1
    layer = XnorConv2d(w, pad=0, variant="auto")
    r = {"shape": [N, C, S, O, k], "kernel": layer.kernel_for(x.shape)}
    r["layer"] = t(lambda: layer.forward(x))
    bits, A = ops.pack_input(x)
    r["pack"] = t(lambda: ops.pack_input(x))
    K = ops.scale_map(A, k, k, 0)
    r["scale"] = t(lambda: ops.scale_map(A, k, k, 0))
    fcf = layer._fc_filters(umma=True)
    b2 = bits.view(1, 1, N, S * S * ops.words(C)); K2 = K.view(1, 1, N)
    r["conv"] = t(lambda: ops.xnor_conv(b2, fcf, K2, 0, variant="umma"))
    print(json.dumps(r))
