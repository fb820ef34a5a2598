import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2007_14178_b200 import ops
x = torch.rand((256, 384, 13, 13), device="cuda") * 2 - 1
for _ in range(5): ops.pack_input(x)
torch.cuda.synchronize()
