"""One small launch of every kernel family in libxnorb200.so, for compute-sanitizer
(tools/sanitize.sh).  Each case is checked against the CPU oracle or a second
kernel, so a run that the tool slows down still proves the results.

    compute-sanitizer --tool racecheck --kernel-name regex=xnc python tools/sanitize_cases.py [group ...]
groups: pack scale popc b1mma umma umma_bulk umma_emit umma_split fc_nhwc pack_wide pool_k1 network conv1 interop verify (default: all)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2007_14178_b200 import XnorConv2d, ops  # noqa: E402


def _layer(x, w, pad, variant, **kw):
    layer = XnorConv2d(torch.from_numpy(w).cuda(), pad=pad, variant=variant, **kw)
    return layer, torch.from_numpy(x).cuda()


def case_pack(rng):
    for shape in ((2, 40, 9, 12), (1, 300, 5, 5), (3, 64, 16, 16)):
        x = O.f32_exact(rng, shape)
        bits, A = ops.pack_input(torch.from_numpy(x).cuda())
        N, C, H, W = shape
        sgn = np.zeros((N, H, W, (C + 31) // 32 * 32), dtype=np.uint64)
        sgn[..., :C] = (x >= 0).transpose(0, 2, 3, 1)
        want = (sgn.reshape(N, H, W, -1, 32) << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)
        torch.cuda.synchronize()
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), want)


def _check_conv(x, w, pad, variant, **kw):
    layer, xd = _layer(x, w, pad, variant, **kw)
    y, acc = layer.forward(xd, want_acc=True)
    want, ints = O.conv_layer(x, w, pad, want_ints=True)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), ints), variant
    assert np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32)), variant


def case_scale(rng):
    x = O.f32_exact(rng, (2, 8, 13, 11))
    _, A = ops.pack_input(torch.from_numpy(x).cuda())
    for k, pad in ((3, 1), (5, 2), (7, 0)):
        ops.scale_map(A, k, k, pad)
    torch.cuda.synchronize()


def case_popc(rng):
    _check_conv(O.f32_exact(rng, (2, 70, 9, 10)), O.f32_exact(rng, (5, 70, 3, 3)), 1, "popc")


def case_b1mma(rng):
    _check_conv(O.f32_exact(rng, (2, 64, 9, 10)), O.f32_exact(rng, (8, 64, 3, 3)), 1, "b1mma")


def case_umma(rng):
    # acc requested: the general epilogue (STG)
    _check_conv(O.f32_exact(rng, (2, 128, 10, 12)), O.f32_exact(rng, (64, 128, 3, 3)), 1, "umma")
    _check_conv(O.f32_exact(rng, (1, 160, 7, 9)), O.f32_exact(rng, (300, 160, 3, 3)), 1, "umma")


def case_umma_bulk(rng):
    # float output only (the plain fast epilogue), MH = 2 and MH = 1
    for (N, C, H, W, O_, k) in ((2, 128, 12, 32, 128, 3), (1, 256, 8, 36, 256, 3)):
        x, w = O.f32_exact(rng, (N, C, H, W)), O.f32_exact(rng, (O_, C, k, k))
        layer, xd = _layer(x, w, 1, "umma")
        y = layer.forward(xd)
        want = O.conv_layer(x, w, 1)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32))


def case_umma_emit(rng):
    x, w = O.f32_exact(rng, (2, 96, 9, 9)), O.f32_exact(rng, (384, 96, 3, 3))
    layer, xd = _layer(x, w, 1, "umma")
    p = layer.forward(xd, emit_signs=True)
    y = layer.forward(xd)
    bits, A = ops.pack_input(y)
    torch.cuda.synchronize()
    assert torch.equal(p.bits, bits) and torch.equal(p.A, A)


def case_umma_split(rng):
    x, w = O.f32_exact(rng, (96, 256, 3, 3)), O.f32_exact(rng, (512, 256, 3, 3))  # fc: kernel == input
    layer, xd = _layer(x, w, 0, "auto")
    y = layer.forward(xd)
    want = O.conv_layer(x, w, 0)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().reshape(want.shape).view(np.uint32), want.view(np.uint32))


def case_fc_nhwc(rng):
    # fully connected layer on the tcgen05 kernel: K split + pixel-major finalize, and the
    # unsplit channels-last epilogue (out_channels_last)
    x, w = O.f32_exact(rng, (96, 256, 3, 3)), O.f32_exact(rng, (512, 256, 3, 3))
    layer, xd = _layer(x, w, 0, "auto")
    assert layer.kernel_for(x.shape) == "umma-fc"
    y = layer.forward(xd)
    want = O.conv_layer(x, w, 0)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().reshape(want.shape).view(np.uint32), want.view(np.uint32))
    # the fused finalize handing fc7 its K1 input (split) and its unsplit form
    for (n_img, n_out) in ((96, 512), (2560, 1024)):
        xe = torch.from_numpy(O.f32_exact(rng, (n_img, 64, 1, 1))).cuda()
        le = XnorConv2d(torch.from_numpy(O.f32_exact(rng, (n_out, 64, 1, 1))).cuda(), pad=0)
        ye = le.forward(xe)
        wb, wa = ops.pack_input(ye.contiguous())
        pe = le.forward(ops.PackedInput(*ops.pack_input(xe), 64), emit_signs=True)
        torch.cuda.synchronize()
        assert torch.equal(pe.bits.view(-1), wb.view(-1)) and torch.equal(pe.A.view(-1), wa.view(-1))
    x2, w2 = O.f32_exact(rng, (2, 64, 9, 11)), O.f32_exact(rng, (132, 64, 3, 3))
    a = XnorConv2d(torch.from_numpy(w2).cuda(), pad=1)(torch.from_numpy(x2).cuda())
    b = XnorConv2d(torch.from_numpy(w2).cuda(), pad=1, out_channels_last=True)(torch.from_numpy(x2).cuda())
    torch.cuda.synchronize()
    assert torch.equal(a, b.contiguous())


def case_pack_wide(rng):
    # K1 of 1 x 1 images with 4096 channels (fc7's input): ballot words + overlapped chain
    x = O.f32_exact(rng, (5, 4096, 1, 1))
    bits, A = ops.pack_input(torch.from_numpy(x).cuda())
    A_ref, _ = O.scale_map_f32(x[0], 1, 1, 0)
    torch.cuda.synchronize()
    assert np.array_equal(A[0].cpu().numpy().view(np.uint32), A_ref.view(np.uint32))


def case_pool_k1(rng):
    # max-pool fused into K1: conv3 / fc6-like inputs, a 33-wide map, and the
    # channels-last front end with bias + ReLU
    for shape in ((2, 96, 27, 27), (2, 64, 13, 13), (1, 40, 11, 33)):
        x = torch.from_numpy(O.f32_exact(rng, shape)).cuda()
        b1, a1 = ops.pack_input(x, in_pool=(3, 2))
        b2, a2 = ops.pack_input(ops.max_pool(x, 3, 2))
        torch.cuda.synchronize()
        assert torch.equal(b1, b2) and torch.equal(a1, a2)
    x = torch.from_numpy(O.f32_exact(rng, (2, 96, 13, 13))).cuda().contiguous(memory_format=torch.channels_last)
    bias = torch.from_numpy(O.f32_exact(rng, (96,))).cuda()
    b1, a1 = ops.pack_input(x, in_pool=(3, 2), pool_relu=True, pool_bias=bias)
    b2, a2 = ops.pack_input(ops.max_pool(x, 3, 2, relu=True, bias=bias))
    torch.cuda.synchronize()
    assert torch.equal(b1, b2) and torch.equal(a1, a2)


def case_network(rng):
    x = torch.from_numpy(O.f32_exact(rng, (2, 7, 11, 13))).cuda()
    ops.max_pool(x, 3, 2, relu=True)
    ops.pad_space_to_depth(x[:, :3, :8, :8].contiguous(), 2, 4)
    xc = x.contiguous(memory_format=torch.channels_last)
    ops.max_pool(xc, 3, 2)
    ops.pack_input(xc)
    torch.cuda.synchronize()


def case_conv1(rng):
    # the network's TF32 conv1 on the tensor cores vs an fp64 conv (TF32 tolerance)
    import torch.nn.functional as F
    x = torch.from_numpy(O.f32_exact(rng, (3, 3, 224, 224))).cuda()
    w = torch.from_numpy(O.f32_exact(rng, (96, 3, 11, 11)) * 0.05).cuda()
    y = ops.conv1_forward(x, ops.conv1_pack_weights(w))
    ref = F.conv2d(x.double(), w.double(), stride=4, padding=2)
    assert ((y.double() - ref).abs().max() / ref.abs().max()).item() < 2e-3


def case_interop(rng):
    import paper_2007_14178_b200 as xc
    t = xc.Tensor3(O.f32_exact(rng, (3, 11, 12)).astype(np.float64))
    w = xc.Tensor3(O.f32_exact(rng, (3, 3, 3)).astype(np.float64))
    for two_stream in (False, True):
        ws = xc.ConvWorkspace(3, 11, 12, 3, 3, 1)
        ws.set_weights(w)
        ws.load_input(t)
        ws.run(two_stream=two_stream)
        ws.int_plane()
        ws.grids()
    geom = xc.TileGeometry(64, 3, 3)
    grid = xc.pack(xc.sign_plane(xc.Tensor2(t.data[0])), geom)
    xc.unpack(grid, 11, 12)
    xc.input_scaling_field(t, 3, 3, 1, 0.5)
    xc.channel_abs_mean(xc.Tensor3(t.data[:, :1, :1].copy()))


def case_verify(rng):
    from paper_2007_14178_b200.verify import run_verification
    assert run_verification(6, 4, kernels=(1, 3, 5)).ok


CASES = {n[5:]: f for n, f in globals().items() if n.startswith("case_")}


def main():
    groups = sys.argv[1:] or list(CASES)
    rng = np.random.default_rng(0)
    for g in groups:
        CASES[g](rng)
        print(f"case {g}: ok", flush=True)


if __name__ == "__main__":
    main()
