"""XNOR-Net AlexNet forward (BASELINE configs 4/5): every binary layer of the
network, on the network's own intermediate activations, matches the oracle on
sampled (image, filter) pairs; the forward is deterministic."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch", [3, 256])
def test_network_binary_layers_match_oracle(batch):
    """batch 256 is BASELINE config 4 (C4): the tile counts, K splits and tails of the
    benched forward, sampled at the first, middle and last image."""
    from paper_2007_14178_b200.network import BINARY_LAYERS, XnorNetAlexNet
    torch.manual_seed(0)
    net = XnorNetAlexNet("cuda", seed=3)
    x = torch.rand((batch, 3, 224, 224), device="cuda") * 2 - 1
    logits, feats = net.forward(x, return_features=True)
    logits2 = net.forward(x)
    torch.cuda.synchronize()
    assert logits.shape == (batch, 1000) and torch.isfinite(logits).all()
    assert torch.equal(logits, logits2)
    # layer inputs: conv1 -> relu -> pool for conv2; pooled / raw previous outputs after
    with torch.no_grad():
        h = net.front_end(x)
        # the space-to-depth front end is the 11x11/4 conv (TF32 on both sides)
        ref = F.max_pool2d(F.relu(F.conv2d(x, net.conv1_w, net.conv1_b, stride=4, padding=2)), 3, 2)
    assert torch.allclose(h, ref, rtol=1e-2, atol=1e-2)
    inputs = {}
    for name, *_ in BINARY_LAYERS:
        inputs[name] = h
        h = feats[name]
        if name in ("conv2", "conv5"):
            h = F.max_pool2d(h, 3, 2)
    n_idx = [0, 1] if batch <= 3 else [0, batch // 2, batch - 1]
    for name, cin, cout, k, pad in BINARY_LAYERS:
        layer = net.binary[name]
        xin = inputs[name][n_idx].contiguous()
        if layer.in_affine is not None:  # the folded BN K1 applies: x*scale + shift, two roundings
            sc, sh = layer.in_affine
            xin = xin * sc.view(1, -1, 1, 1) + sh.view(1, -1, 1, 1)
        xi = xin.cpu().numpy()
        o_idx = [0, cout // 2, cout - 1]
        wi = layer.weight[o_idx].cpu().numpy()
        want = O.conv_layer(xi, wi, pad)
        if layer.out_affine is not None:  # the next layer's BN, fused into this epilogue
            sc, sh = (t[o_idx].cpu().numpy() for t in layer.out_affine)
            want = (want * sc.reshape(1, -1, 1, 1)).astype(np.float32)
            want = (want + sh.reshape(1, -1, 1, 1)).astype(np.float32)
        got = feats[name][n_idx][:, o_idx].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), name


def test_network_kernel_selection():
    from paper_2007_14178_b200.network import XnorNetAlexNet
    net = XnorNetAlexNet("cuda", seed=1)
    ks = net.binary_kernels(256)
    assert ks["fc7"] in ("popc-fc", "umma-fc") and ks["fc6"] in ("popc-fc", "umma-fc")
    assert all(v in ("umma", "popc", "popc-fc", "umma-fc") for v in ks.values())


@pytest.mark.parametrize("shape,pad,r", [((2, 3, 224, 224), 2, 4), ((3, 5, 10, 14), 1, 4), ((1, 2, 6, 6), 0, 2),
                                         ((2, 3, 12, 20), 2, 4), ((1, 3, 6, 10), 3, 4)])
def test_pad_space_to_depth_matches_torch(shape, pad, r):
    from paper_2007_14178_b200 import ops
    x = torch.randn(shape, device="cuda")
    want = F.pixel_unshuffle(F.pad(x, (pad,) * 4), r)
    assert torch.equal(ops.pad_space_to_depth(x, pad, r), want)
    cl = ops.pad_space_to_depth(x, pad, r, channels_last=True)
    assert cl.is_contiguous(memory_format=torch.channels_last) and torch.equal(cl, want)


@pytest.mark.parametrize("shape,k,s", [((2, 96, 55, 55), 3, 2), ((3, 7, 9, 12), 2, 2), ((1, 4, 11, 11), 5, 3),
                                       ((2, 256, 27, 27), 3, 2), ((3, 40, 13, 13), 3, 2), ((1, 5, 39, 39), 3, 1)])
def test_relu_max_pool_matches_torch(shape, k, s):
    from paper_2007_14178_b200 import ops
    x = torch.randn(shape, device="cuda")
    x[0, 0, :3, :3] = -1.0  # an all-negative window: relu -> 0
    want = F.max_pool2d(F.relu(x), k, s)
    assert torch.equal(ops.max_pool(x, k, s, relu=True), want)
    assert torch.equal(ops.max_pool(x, k, s), F.max_pool2d(x, k, s))
    xl = x.contiguous(memory_format=torch.channels_last)  # channels-last in, channels-last out
    got = ops.max_pool(xl, k, s, relu=True)
    assert got.is_contiguous(memory_format=torch.channels_last) and torch.equal(got, want)
    b = torch.randn(shape[1], device="cuda")  # a conv bias folded into the pool: exact
    want_b = F.max_pool2d(F.relu(x + b.view(1, -1, 1, 1)), k, s)
    assert torch.equal(ops.max_pool(x, k, s, relu=True, bias=b), want_b)
    assert torch.equal(ops.max_pool(xl, k, s, relu=True, bias=b), want_b)


@pytest.mark.parametrize("shape", [(3, 96, 27, 27), (2, 70, 5, 7), (2, 33, 4, 4)])
def test_pack_input_channels_last_matches_nchw(shape):
    """K1 on a channels-last map (the front end's output) == K1 on the NCHW copy:
    bits and A identical, with and without the folded BN."""
    from paper_2007_14178_b200 import ops
    x = torch.randn(shape, device="cuda")
    x[0, 0, 0, 0] = 0.0
    x[0, 1, 0, 0] = -0.0
    xl = x.contiguous(memory_format=torch.channels_last)
    C = shape[1]
    for aff in (None, (torch.rand(C, device="cuda") + 0.5, torch.rand(C, device="cuda") - 0.5)):
        b1, a1 = ops.pack_input(xl, in_affine=aff)
        b2, a2 = ops.pack_input(x, in_affine=aff)
        assert torch.equal(b1, b2)
        assert torch.equal(a1.view(torch.int32), a2.view(torch.int32))


def test_network_cuda_graph_matches_eager():
    """The captured forward (bench.py's C4 step) recomputes the eager logits exactly,
    also after new images are copied into its input buffer."""
    from paper_2007_14178_b200.network import XnorNetAlexNet
    net = XnorNetAlexNet("cuda", seed=2)
    x = torch.rand((4, 3, 224, 224), device="cuda") * 2 - 1
    graph, logits = net.capture(x)
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(logits, net.forward(x))
        x.copy_(torch.rand_like(x) * 2 - 1)


@pytest.mark.parametrize("batch", [3, 256])
def test_network_emitted_signs_match_float_chain(batch):
    """conv3 -> conv4 -> conv5 through the sign-emitting epilogue (the default forward)
    give exactly the logits of the float-feature-map chain."""
    from paper_2007_14178_b200.network import XnorNetAlexNet
    a = XnorNetAlexNet("cuda", seed=5)
    b = XnorNetAlexNet("cuda", seed=5, emit_signs=False)
    x = torch.rand((batch, 3, 224, 224), device="cuda") * 2 - 1
    assert torch.equal(a.forward(x), b.forward(x))


@pytest.mark.parametrize("batch", [1, 5, 37])
def test_conv1_tcgen05_tf32_matches_fp64(batch):
    """conv1 on our kind::tf32 tensor-core kernel (csrc/xnc_conv1.cu) vs an fp64
    conv: TF32-rounded operands, f32 accumulation over 363 terms.  Tolerance: 2e-3
    max-norm relative (TF32 keeps 10 mantissa bits; measured ~3e-4), and no worse
    than 2x cuDNN's own TF32 error on the same data.  Batches 5 / 37 put pair tiles
    across image boundaries (tiles are linear over the batch)."""
    from paper_2007_14178_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(batch)
    x = torch.rand((batch, 3, 224, 224), device="cuda", generator=g) * 2 - 1
    w = (torch.rand((96, 3, 11, 11), device="cuda", generator=g) * 2 - 1) * (3 * 121) ** -0.5
    y = ops.conv1_forward(x, ops.conv1_pack_weights(w))
    assert y.is_contiguous(memory_format=torch.channels_last) and y.shape == (batch, 96, 55, 55)
    ref = F.conv2d(x.double(), w.double(), stride=4, padding=2)
    err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    saved = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = True
    try:
        cud = F.conv2d(x, w, stride=4, padding=2)
    finally:
        torch.backends.cudnn.allow_tf32 = saved
    err_cudnn = ((cud.double() - ref).abs().max() / ref.abs().max()).item()
    assert err <= 2e-3 and err <= 2 * err_cudnn + 1e-6, (err, err_cudnn)


def test_network_front_end_engines_agree():
    """front_end on the tcgen05 conv1 vs the s2d + cuDNN path: both TF32, same layer."""
    from paper_2007_14178_b200.network import XnorNetAlexNet
    torch.manual_seed(1)
    x = torch.rand((4, 3, 224, 224), device="cuda") * 2 - 1
    a = XnorNetAlexNet("cuda", seed=2, conv1="tcgen05").front_end(x)
    b = XnorNetAlexNet("cuda", seed=2, conv1="cudnn").front_end(x)
    assert a.shape == b.shape == (4, 96, 27, 27)
    assert ((a - b).abs().max() / b.abs().max()).item() <= 4e-3
