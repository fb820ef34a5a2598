"""Time XNOR-Net AlexNet's full-precision front end (conv1 11x11/4 + bias + ReLU +
pool 3/2) at batch 256 under different layouts, to pick the network's path."""
import json
import torch
import torch.nn.functional as F

torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
torch.backends.cudnn.benchmark = True
dev = "cuda"
x = torch.rand((256, 3, 224, 224), device=dev) * 2 - 1
w = torch.rand((96, 3, 11, 11), device=dev) * 0.1
b = torch.rand(96, device=dev) * 0.1


def nchw():
    h = F.conv2d(x, w, b, stride=4, padding=2)
    return F.max_pool2d(F.relu(h), 3, 2)


xl = x.contiguous(memory_format=torch.channels_last)
wl = w.contiguous(memory_format=torch.channels_last)


def nhwc_in():  # input already NHWC
    h = F.conv2d(xl, wl, b, stride=4, padding=2)
    h = F.max_pool2d(F.relu_(h), 3, 2)
    return h.contiguous()


def nhwc_convert():  # NCHW input converted on device
    h = F.conv2d(x.contiguous(memory_format=torch.channels_last), wl, b, stride=4, padding=2)
    h = F.max_pool2d(F.relu_(h), 3, 2)
    return h.contiguous()


def nhwc_keep():  # leave the pooled map NHWC
    h = F.conv2d(xl, wl, b, stride=4, padding=2)
    return F.max_pool2d(F.relu_(h), 3, 2)


ref = nchw()
for name, fn in [("nchw", nchw), ("nhwc_in", nhwc_in), ("nhwc_convert", nhwc_convert), ("nhwc_keep", nhwc_keep)]:
    for _ in range(5):
        y = fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        y = fn()
    e.record()
    torch.cuda.synchronize()
    err = float((y.float() - ref).abs().max())
    print(json.dumps({"variant": name, "ms": round(s.elapsed_time(e) / 20, 4), "max_abs_diff_vs_nchw": err}))


# space-to-depth: the 11x11/4 conv (kernel zero-padded to 12x12) == a 3x3/1 conv
# over pixel_unshuffle(x_pad, 4) with 48 channels
w12 = F.pad(w, (0, 1, 0, 1))                                     # [96, 3, 12, 12]
ws2d = w12.view(96, 3, 3, 4, 3, 4).permute(0, 1, 3, 5, 2, 4).reshape(96, 48, 3, 3).contiguous()
wsl = ws2d.contiguous(memory_format=torch.channels_last)


def s2d_nchw():
    xp = F.pad(x, (2, 2, 2, 2))
    h = F.conv2d(F.pixel_unshuffle(xp, 4), ws2d, b)
    return F.max_pool2d(F.relu_(h), 3, 2)


def s2d_nhwc():
    xp = F.pad(x, (2, 2, 2, 2))
    s = F.pixel_unshuffle(xp, 4).contiguous(memory_format=torch.channels_last)
    h = F.conv2d(s, wsl, b)
    return F.max_pool2d(F.relu_(h), 3, 2).contiguous()


def s2d_bf16():
    xp = F.pad(x, (2, 2, 2, 2))
    s = F.pixel_unshuffle(xp, 4).contiguous(memory_format=torch.channels_last).bfloat16()
    h = F.conv2d(s, wsl.bfloat16(), b.bfloat16())
    return F.max_pool2d(F.relu_(h), 3, 2).float().contiguous()


for name, fn in [("s2d_nchw", s2d_nchw), ("s2d_nhwc", s2d_nhwc), ("s2d_bf16_nhwc", s2d_bf16)]:
    for _ in range(5):
        y = fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        y = fn()
    e.record()
    torch.cuda.synchronize()
    err = float((y.float() - ref).abs().max())
    print(json.dumps({"variant": name, "ms": round(s.elapsed_time(e) / 20, 4), "max_abs_diff_vs_nchw": err}))


# space-to-depth straight into NHWC (one gather), conv/ReLU/pool in channels_last
def s2d_direct_nhwc(contig=True):
    xp = F.pad(x, (2, 2, 2, 2))                                   # [N, 3, 228, 228]
    s = xp.view(256, 3, 57, 4, 57, 4).permute(0, 2, 4, 1, 3, 5).reshape(256, 57, 57, 48)
    s = s.permute(0, 3, 1, 2)                                      # NCHW view, NHWC memory
    h = F.conv2d(s, wsl, b)
    h = F.max_pool2d(F.relu_(h), 3, 2)
    return h.contiguous() if contig else h


for name, fn in [("s2d_direct_nhwc", s2d_direct_nhwc), ("s2d_direct_nhwc_keep", lambda: s2d_direct_nhwc(False))]:
    for _ in range(5):
        y = fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        y = fn()
    e.record()
    torch.cuda.synchronize()
    err = float((y.float() - ref).abs().max())
    print(json.dumps({"variant": name, "ms": round(s.elapsed_time(e) / 20, 4), "max_abs_diff_vs_nchw": err,
                      "out_channels_last": bool(y.is_contiguous(memory_format=torch.channels_last))}))
