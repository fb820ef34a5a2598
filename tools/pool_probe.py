"""Device time of the network's pooled-K1 passes at batch 256 (C4), per kernel path:
conv3's input (NCHW 256 x 27 x 27 -> 13 x 13), fc6's (256 x 13 x 13 -> 6 x 6), and the
front end (conv1's channels-last 96 x 55 x 55 map: pool + bias + ReLU, then conv2's K1
with its BN) as two passes or fused.  Usage: python tools/pool_probe.py [batch]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_14178_b200 import ops  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.rand(s, device="cuda", generator=g) * 2 - 1
    aff = lambda c: (r(c) * 0.5 + 1.0, r(c) * 0.1)
    x3, x6 = r(N, 256, 27, 27), r(N, 256, 13, 13)
    h1 = r(N, 96, 55, 55).contiguous(memory_format=torch.channels_last)
    a3, a6, a2, b1 = aff(256), aff(256), aff(96), r(96) * 0.1
    res = {"batch": N}
    res["conv3_in_us"] = timed(lambda: ops.pack_input(x3, in_affine=a3, in_pool=(3, 2)))
    res["fc6_in_us"] = timed(lambda: ops.pack_input(x6, in_affine=a6, in_pool=(3, 2)))
    res["front_two_pass_us"] = timed(lambda: ops.pack_input(ops.max_pool(h1, 3, 2, relu=True, bias=b1), in_affine=a2))
    res["front_pool_only_us"] = timed(lambda: ops.max_pool(h1, 3, 2, relu=True, bias=b1))
    res["front_fused_us"] = timed(lambda: ops.pack_input(h1, in_affine=a2, in_pool=(3, 2), pool_relu=True, pool_bias=b1))
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)


if __name__ == "__main__":
    main()
