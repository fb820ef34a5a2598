"""A C3 layer inside a stack of binary layers (its input already in K1 form): the
float epilogue + the next layer's K1 pass vs the sign-emitting epilogue.  Profiling
aid; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2007_14178_b200 import XnorConv2d, ops  # noqa: E402


def t(fn, reps=20):
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


N, C, H, W, O = 256, 256, 56, 56, 256
x = torch.rand((N, C, H, W), device="cuda") * 2 - 1
w = torch.rand((O, C, 3, 3), device="cuda") * 2 - 1
bn = (torch.rand(O, device="cuda") + 0.5, torch.rand(O, device="cuda") - 0.5)
layer = XnorConv2d(w, pad=1, variant="auto", out_affine=bn)
bits, A = ops.pack_input(x)
p = ops.PackedInput(bits, A, C)
r = {
    "float_epilogue_then_next_k1": t(lambda: ops.pack_input(layer.forward(p))),
    "float_epilogue_only": t(lambda: layer.forward(p)),
    "sign_emitting_epilogue": t(lambda: layer.forward(p, emit_signs=True)),
}
print(json.dumps({"bench": "chain_probe", "config": "C3 layer with its input in K1 form", "ms": r}))
