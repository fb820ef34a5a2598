"""Pin the CPU oracle (oracle/xnor_oracle.c + oracle/oracle.py) to the reference:
golden vectors produced by the reference itself (tests/golden/make_golden.py)
and the reference's own known-answer tests (test_pack.py, test_binarize.py,
test_reference.py, SPEC.md worked examples).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import golden_io


@pytest.mark.parametrize("case", golden_io.layer_cases(), ids=lambda c: c["name"])
def test_oracle_layer_matches_reference_bit_exact(case):
    out, ints = O.conv_layer(case["x"], case["w"], case["pad"], word_bits=case["word_bits"], want_ints=True)
    assert np.array_equal(ints, case["ints"])
    assert np.array_equal(out.view(np.uint32), case["out"].view(np.uint32))  # bit-exact f32


@pytest.mark.parametrize("case", golden_io.layer_cases(), ids=lambda c: c["name"])
def test_oracle_alpha_and_naive_ints(case):
    for o in range(case["w"].shape[0]):
        assert O.alpha(case["w"][o]) == case["alpha"][o]
        assert O.build_filter(case["w"][o])[2] == case["alpha"][o]
    if case["C"] * case["H"] * case["W"] <= 4096:
        for n in range(case["x"].shape[0]):
            for o in range(case["w"].shape[0]):
                assert np.array_equal(O.sign_conv2d_int(case["x"][n], case["w"][o], case["pad"]),
                                      case["ints"][n, o])


@pytest.mark.parametrize("case", golden_io.pack_cases(), ids=lambda c: c["name"])
def test_oracle_pack_words(case):
    words = O.pack_plane(O.signs(case["plane"]), case["word_bits"], case["kh"], case["kw"])
    assert np.array_equal(words, case["words"])
    words_f = O.pack_plane(case["plane"].astype(np.float32), case["word_bits"], case["kh"], case["kw"])
    assert np.array_equal(words_f, case["words"])


@pytest.mark.parametrize("case", golden_io.scale_cases(), ids=lambda c: c["name"])
def test_oracle_float64_operator_api(case):
    A = O.channel_abs_mean_f64(case["x"])
    assert np.array_equal(A, case["A"])
    k, pad = case["k"], case["pad"]
    K = O.box_mean_f64(np.pad(A, pad), k, k)
    assert np.array_equal(K, case["K"])
    words, mask, a = O.build_filter(case["w"])
    assert np.array_equal(words, case["weight_words"]) and mask == int(case["base_mask"][0])
    assert a == case["alpha"][0]
    y = case["ints"] * K * a  # apply_scaling (scaling.py:98), float64
    assert np.array_equal(y, case["y"])


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 1, 1), (8, 1, 1), (9, 1, 1), (129, 1, 1), (1000, 1, 1),
                                   (3001, 1, 1), (13, 1, 5), (13, 5, 1), (200, 3, 3)])
def test_oracle_channel_abs_mean_is_numpys(shape):
    # tensor.py:103-105 is np.abs(x).mean(axis=0): pairwise when axis 0 is the lone
    # axis (C,1,1), sequential per pixel otherwise -- bit-exact either way
    rng = np.random.default_rng(shape[0])
    x = rng.standard_normal(shape) * 37.0
    assert np.array_equal(O.channel_abs_mean_f64(x), np.abs(x).mean(axis=0))


# ---- the reference's own KATs -------------------------------------------------------

def test_kat_padding_is_plus_one():
    # test_reference.py:69-75: all -1 image, all +1 3x3 filter, pad 1: corner +1, interior -9
    x = -np.ones((1, 4, 4), np.float32)
    w = np.ones((1, 3, 3), np.float32)
    ints = O.sign_conv2d_int(x, w, 1)
    assert ints[0, 0] == 1 and ints[1, 1] == -9
    _, oi = O.conv_layer(x[None], w[None], 1, want_ints=True)
    assert np.array_equal(oi[0, 0], ints)


def test_kat_sign_zero_is_plus_one():
    # test_binarize.py:78-82
    assert list(O.signs(np.array([0.0, -0.0, -1e-30, 1.0]))) == [1, 1, -1, 1]


def test_kat_alpha():
    # test_binarize.py:16-27: alpha of [[3,-7]] style KAT = mean |w|; all-zero -> 0
    assert O.alpha(np.array([[[3.0, -7.0], [5.0, -5.0]]])) == 5.0
    assert O.alpha(np.zeros((2, 3, 3))) == 0.0


def test_kat_pack_words():
    # test_pack.py:77-100
    assert O.pack_plane(np.ones((8, 8), np.int8), 64, 3, 3)[0, 0] == 0xFFFF_FFFF_FFFF_FFFF
    p = -np.ones((8, 8), np.int8); p[0, 0] = 1
    assert O.pack_plane(p, 64, 3, 3)[0, 0] == 1
    p = -np.ones((8, 8), np.int8); p[2, 5] = 1
    assert O.pack_plane(p, 64, 3, 3)[0, 0] == 1 << 21
    p = -np.ones((8, 4), np.int8); p[1, 3] = 1
    assert O.pack_plane(p, 32, 3, 3)[0, 0] == 1 << 7


def test_kat_xnor_uniform_and_single_pixel():
    # SPEC.md xnor_conv2d examples: 16x16 all +1 -> +9 everywhere; a single -1 pixel -> 9 windows at +7
    x = np.ones((1, 1, 16, 16), np.float32)
    w = np.ones((1, 1, 3, 3), np.float32)
    _, ints = O.conv_layer(x, w, 1, want_ints=True)
    assert (ints == 9).all()
    x[0, 0, 7, 7] = -1
    _, ints = O.conv_layer(x, w, 1, want_ints=True)
    assert (ints == 7).sum() == 9 and (ints == 9).sum() == 16 * 16 - 9


def test_kat_scale_map_constant_and_corner():
    # SPEC.md compute_K: constant A = 2.0, k=3, pad 1 -> interior 2.0, corner 8/9
    x = np.full((1, 6, 6), 2.0, np.float32)
    _, K = O.scale_map_f32(x, 3, 3, 1)
    assert K[2, 2] == pytest.approx(2.0, rel=1e-6) and K[0, 0] == pytest.approx(8 / 9, rel=1e-6)
