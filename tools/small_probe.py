import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2007_14178_b200 import XnorConv2d
def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps * 1000, 1)
out = {}
for name, (N, C, H, O, k) in {"C1": (1, 64, 32, 64, 3), "N8_C64_32": (8, 64, 32, 64, 3), "N1_C256_14": (1, 256, 14, 256, 3),
                              "N4_C128_28": (4, 128, 28, 128, 3), "N16_C128_28": (16, 128, 28, 128, 3)}.items():
    x = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    w = torch.rand((O, C, k, k), device="cuda") * 2 - 1
    r = {}
    for v in ("umma", "popc"):
        layer = XnorConv2d(w, pad=1, variant=v)
        r[v + "_us"] = t(lambda: layer.forward(x))
    out[name] = r
print(json.dumps(out))
