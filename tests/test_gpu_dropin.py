"""The drop-in operator API (paper_2007_14178_b200 mirrors xnorconv's names)
on the GPU: the reference's own test cases (test_pack.py, test_binarize.py,
test_reference.py, verify.py, SPEC.md examples) re-run against the device
implementation, plus the reference-generated golden vectors, plus the C-ABI
kernel seam (xnc_pack_plane ... xnc_xnor_reconstruct)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import golden_io

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xc():
    import paper_2007_14178_b200 as m
    return m


def f32_tensor(rng, shape, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, shape).astype(np.float32).astype(np.float64)


# ---------------------------------------------------------------- binarize (test_binarize.py)
def test_alpha_kat_and_zero(xc):
    a = xc.sign_binarize(xc.Tensor3(np.array([[[3.0, -7.0], [5.0, -5.0]]])))
    assert a.scale == 5.0
    z = xc.sign_binarize(xc.Tensor3(np.zeros((2, 3, 3))))
    assert z.scale == 0.0 and all((p.signs == 1).all() for p in z.signs)


def test_alpha_matches_sequential_loop(xc):
    rng = np.random.default_rng(3)
    w = rng.uniform(-2, 2, (5, 3, 3))
    assert xc.sign_binarize(xc.Tensor3(w)).scale == O.alpha(w)


def test_sign_of_zero_is_plus_one(xc):
    p = xc.sign_plane(xc.Tensor2(np.array([[0.0, -0.0, -1e-300, 2.0]])))
    assert p.signs.tolist() == [[1, 1, -1, 1]]


# ---------------------------------------------------------------- pack (test_pack.py)
def test_pack_word_kats(xc):
    g64 = xc.TileGeometry(64, 3, 3)
    assert xc.pack(xc.SignPlane(np.ones((8, 8))), g64).words[0, 0] == 0xFFFF_FFFF_FFFF_FFFF
    p = -np.ones((8, 8)); p[0, 0] = 1
    assert xc.pack(xc.SignPlane(p), g64).words[0, 0] == 1
    p = -np.ones((8, 8)); p[2, 5] = 1
    assert xc.pack(xc.SignPlane(p), g64).words[0, 0] == 1 << 21
    p = -np.ones((8, 4)); p[1, 3] = 1
    assert xc.pack(xc.SignPlane(p), xc.TileGeometry(32, 3, 3)).words[0, 0] == 1 << 7


def test_grid_shape_kats(xc):
    assert xc.tile_grid_shape(xc.TileGeometry(64, 3, 3), 14, 14) == (3, 3)
    assert xc.tile_grid_shape(xc.TileGeometry(64, 3, 3), 4, 4) == (1, 1)
    with pytest.raises(ValueError):
        xc.TileGeometry(32, 3, 5)


@pytest.mark.parametrize("case", golden_io.pack_cases(), ids=lambda c: c["name"])
def test_pack_matches_reference_golden(xc, case):
    geom = xc.TileGeometry(case["word_bits"], case["kh"], case["kw"])
    grid = xc.pack(xc.sign_plane(xc.Tensor2(case["plane"])), geom)
    assert np.array_equal(grid.words, case["words"])
    back = xc.unpack(grid, case["h"], case["w"])
    assert np.array_equal(back.signs, O.signs(case["plane"]))


def test_unpack_detects_corrupt_overlap(xc):
    geom = xc.TileGeometry(64, 3, 3)
    rng = np.random.default_rng(5)
    grid = xc.pack(xc.SignPlane(np.where(rng.random((14, 14)) < 0.5, 1, -1)), geom)
    words = grid.words.copy()
    words[0, 0] ^= np.uint64(1 << 7)  # (0,7): shared with tile (0,1)
    with pytest.raises(xc.OverlapMismatchError):
        xc.unpack(xc.PackedTileGrid(geom, words), 14, 14)


# ---------------------------------------------------------------- engine (SPEC.md xnor examples)
def test_xnor_tile_kats(xc):
    geom = xc.TileGeometry(64, 3, 3)
    filt = xc.build_filter(xc.Tensor3(np.ones((1, 3, 3))), geom)
    assert (xc.xnor_tile(0xFFFF_FFFF_FFFF_FFFF, filt, geom) == 9).all()
    assert (xc.xnor_tile(0, filt, geom) == -9).all()
    assert xc.popcount_to_signed(5, 9) == 1


def test_engine_instances_like_verify(xc):
    """verify.check_engine_instances (verify.py:42-79) with k in {1,3,5,7}: exact."""
    rng = np.random.default_rng(0)
    for i in range(60):
        wb = (64, 32)[i % 2]
        k = int(rng.choice([1, 3] if wb == 32 else [1, 3, 5, 7]))
        geom = xc.TileGeometry(wb, k, k)
        c = int(rng.integers(1, 5))
        h, w = int(rng.integers(max(8, k), 40)), int(rng.integers(max(8, k), 40))
        planes = f32_tensor(rng, (c, h, w))
        wts = f32_tensor(rng, (c, k, k))
        filt = xc.build_filter(xc.Tensor3(wts), geom)
        grids = [xc.pack(xc.sign_plane(xc.Tensor2(p)), geom) for p in planes]
        got = xc.xnor_conv_multichannel(grids, filt, h - k + 1, w - k + 1)
        want = O.sign_conv2d_int(planes, wts, 0)
        assert np.array_equal(got.values, want)
        one = xc.xnor_conv2d(grids[0], filt, h - k + 1, w - k + 1, channel=0)
        assert np.array_equal(one.values, O.sign_conv2d_int(planes[:1], wts[:1], 0))


def test_geometry_mismatch_errors(xc):
    geom = xc.TileGeometry(64, 3, 3)
    filt = xc.build_filter(xc.Tensor3(np.ones((2, 3, 3))), geom)
    grid = xc.pack(xc.SignPlane(np.ones((10, 10))), geom)
    with pytest.raises(xc.GeometryMismatchError):
        xc.xnor_conv_multichannel([grid], filt, 8, 8)
    with pytest.raises(xc.GeometryMismatchError):
        xc.build_filter(xc.Tensor3(np.ones((2, 5, 5))), geom)


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 1, 1), (8, 1, 1), (9, 1, 1), (129, 1, 1), (1000, 1, 1),
                                   (3001, 1, 1), (13, 1, 5), (13, 5, 1), (200, 3, 3)])
def test_channel_abs_mean_is_numpys(xc, shape):
    # the reference's own formula (tensor.py:103-105); (C,1,1) takes numpy's pairwise order
    rng = np.random.default_rng(shape[0])
    x = rng.standard_normal(shape) * 37.0
    assert np.array_equal(xc.channel_abs_mean(xc.Tensor3(x)).data, np.abs(x).mean(axis=0))


# ---------------------------------------------------------------- scaling (float64 operator API)
@pytest.mark.parametrize("case", golden_io.scale_cases(), ids=lambda c: c["name"])
def test_float64_scale_path_matches_reference_golden(xc, case):
    t = xc.Tensor3(case["x"])
    k, pad = case["k"], case["pad"]
    A = xc.channel_abs_mean(t)
    assert np.array_equal(A.data, case["A"])
    K = xc.input_scale_map(A, k, k, pad)
    assert np.array_equal(K.data, case["K"])
    geom = xc.TileGeometry(64, k, k)
    filt = xc.build_filter(xc.Tensor3(case["w"]), geom)
    assert np.array_equal(filt.weight_words, case["weight_words"]) and filt.scale == case["alpha"][0]
    grids = [xc.pack(xc.sign_plane(xc.Tensor2(ch)), geom) for ch in xc.zero_pad(t, pad).data]
    ints = xc.xnor_conv_multichannel(grids, filt, K.height, K.width)
    assert np.array_equal(ints.values, case["ints"])
    y = xc.apply_scaling(ints, xc.input_scaling_field(t, k, k, pad, filt.scale))
    assert np.array_equal(y.data, case["y"])


def test_scale_kats(xc):
    K = xc.input_scale_map(xc.Tensor2(np.full((6, 6), 2.0)), 3, 3, 1)
    assert K.data[2, 2] == pytest.approx(2.0) and K.data[0, 0] == pytest.approx(8 / 9)
    ints = xc.IntOutputPlane(np.full((2, 2), 9))
    y = xc.apply_scaling(ints, xc.ScalingField(xc.Tensor2(np.ones((2, 2))), 0.5))
    assert (y.data == 4.5).all()


# ---------------------------------------------------------------- pipeline (ConvWorkspace / xnor_conv)
@pytest.mark.parametrize("variant", ["auto", "popc", "umma"])
@pytest.mark.parametrize("case", [c for c in golden_io.layer_cases() if c["N"] * c["O"] <= 16],
                         ids=lambda c: c["name"])
def test_workspace_matches_reference_golden(xc, case, variant):
    from paper_2007_14178_b200 import ops
    N, C, H, W, Oc = case["N"], case["C"], case["H"], case["W"], case["O"]
    if variant == "umma" and not ops.umma_supported(1, C, H, W, 1, case["kh"], case["kw"], case["pad"]):
        pytest.skip("shape outside the tcgen05 kernel's smem plan")
    ws = xc.ConvWorkspace(C, H, W, case["kh"], case["kw"], case["pad"], case["word_bits"])
    ws.variant = variant
    for n in range(N):
        ws.load_input(xc.Tensor3(case["x"][n].astype(np.float64)))
        for o in range(Oc):
            ws.set_weights(xc.Tensor3(case["w"][o].astype(np.float64)))
            if variant != "popc":
                assert ws.kernel == "umma" or variant == "auto"
            out = ws.run(threads=4)
            assert np.array_equal(out.view(np.uint32), case["out"][n, o].view(np.uint32))
            assert np.array_equal(ws.int_plane().values, case["ints"][n, o])
            assert ws.filter.scale == case["alpha"][o]
    ws.close()


def test_xnor_conv_one_shot_and_grids(xc):
    rng = np.random.default_rng(11)
    x = f32_tensor(rng, (5, 12, 13))
    w = f32_tensor(rng, (5, 3, 3))
    got = xc.xnor_conv(xc.Tensor3(x), xc.Tensor3(w))
    want = O.conv_layer(x[None].astype(np.float32), w[None].astype(np.float32), 1)[0, 0]
    assert np.array_equal(got.data, want.astype(np.float64))
    ws = xc.ConvWorkspace(5, 12, 13, 3, 3, 1)
    ws.load_input(xc.Tensor3(x))
    grids = ws.grids()
    padded = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    for c in range(5):
        assert np.array_equal(grids[c].words, O.pack_plane(padded[c].astype(np.float32), 64, 3, 3))


def test_pipeline_instances_like_verify(xc):
    """verify.check_pipeline_instances (verify.py:82-130), k in {1,3,5,7}, <= 1e-5."""
    rng = np.random.default_rng(1)
    for i in range(20):
        k = int(rng.choice([1, 3, 5, 7]))
        pad = (k - 1) // 2
        c, h, w = int(rng.integers(1, 4)), int(rng.integers(8, 33)), int(rng.integers(8, 33))
        inp = rng.uniform(-1, 1, (c, h, w))
        wts = rng.uniform(-1, 1, (c, k, k))
        ws = xc.ConvWorkspace(c, h, w, k, k, pad, 64)
        ws.set_weights(xc.Tensor3(wts))
        ws.load_input(xc.Tensor3(inp))
        got = ws.run().copy()
        ints = O.sign_conv2d_int(np.pad(inp, ((0, 0), (pad, pad), (pad, pad))), wts, 0)
        K = O.box_mean_f64(np.pad(O.channel_abs_mean_f64(inp), pad), k, k)
        want = ints * K * O.alpha(wts)
        assert np.abs(got - want).max() / max(np.abs(want).max(), 1e-30) <= 1e-5


def test_workspace_errors(xc):
    with pytest.raises(ValueError):
        xc.ConvWorkspace(2, 8, 8, 3, 3, -1)
    with pytest.raises(ValueError):
        xc.ConvWorkspace(2, 2, 2, 7, 7, 0)
    ws = xc.ConvWorkspace(2, 8, 8, 3, 3, 1)
    with pytest.raises(RuntimeError):
        ws.run()
    with pytest.raises(ValueError):
        ws.set_weights(xc.Tensor3(np.ones((3, 3, 3))))
    with pytest.raises(ValueError):
        xc.xnor_conv(xc.Tensor3(np.ones((2, 8, 8))), xc.Tensor3(np.ones((2, 2, 2))))  # no default pad
    with pytest.raises(ValueError):
        xc.ConvWorkspace(2, 8, 8, 3, 3, 1, backend="python")


# ---------------------------------------------------------------- the C-ABI kernel seam
def _seam_reconstruct(xc, padded, filt_words, mask, geom, kh, kw, alpha):
    from paper_2007_14178_b200 import _dev
    from paper_2007_14178_b200._lib import check, DTYPE_F32
    C, ph, pw = padded.shape
    p = _dev.to_dev(padded.astype(np.float32))
    out = _dev.empty((ph - kh + 1, pw - kw + 1), np.float32)
    ww = _dev.to_dev(np.ascontiguousarray(filt_words, dtype=np.uint64))
    check(_dev.L().xnc_xnor_reconstruct(ww.data_ptr(), mask, geom.tile_h, geom.tile_w, geom.stride_y,
                                        geom.stride_x, kh * kw, p.data_ptr(), DTYPE_F32, C, ph, pw, kh,
                                        kw, 1.0 / (kh * kw), alpha, out.data_ptr(), _dev.stream()),
          "xnc_xnor_reconstruct")
    return _dev.to_host(out)


@pytest.mark.parametrize("case", [c for c in golden_io.layer_cases() if c["N"] * c["O"] <= 8],
                         ids=lambda c: c["name"])
def test_seam_xnor_reconstruct_matches_reference_fused(xc, case):
    geom = xc.TileGeometry(case["word_bits"], case["kh"], case["kw"])
    pad = case["pad"]
    for n in range(case["N"]):
        padded = np.pad(case["x"][n], ((0, 0), (pad, pad), (pad, pad)))
        for o in range(case["O"]):
            f = xc.build_filter(xc.Tensor3(case["w"][o].astype(np.float64)), geom)
            got = _seam_reconstruct(xc, padded, f.weight_words, f.base_mask, geom, case["kh"],
                                    case["kw"], f.scale)
            assert np.array_equal(got.view(np.uint32), case["out"][n, o].view(np.uint32))
