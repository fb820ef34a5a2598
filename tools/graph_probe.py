import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2007_14178_b200.network import XnorNetAlexNet
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4)
net = XnorNetAlexNet("cuda", seed=7)
x = torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1
r = {"eager": t(lambda: net(x))}
ref = net(x)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3): net(x)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out = net(x)
g.replay(); torch.cuda.synchronize()
r["graph_equal"] = bool(torch.equal(out, ref))
r["graph"] = t(lambda: g.replay())
print(json.dumps(r))
