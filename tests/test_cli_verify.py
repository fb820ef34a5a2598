"""The reference's CLI (cli.py:30-137), verify (verify.py:22-145), naive
reference loops (reference.py:30-122) and bench harness (bench.py:44-297),
re-run against this package's device implementations.

CPU tests: argument handling, config validation, report formatting.
GPU tests: verification (k in {1,3,5,7} included), the naive device kernels
against Python loops / the C oracle, and the three subcommands end to end."""
import numpy as np
import pytest

from oracle import oracle as O


# ---------------------------------------------------------------- CPU
def test_cli_refuses_python_backend(capsys):
    from paper_2007_14178_b200.cli import main
    assert main(["verify", "--backend", "python"]) == 2
    assert "CPU fallback" in capsys.readouterr().err


def test_cli_parser_matches_reference_options():
    from paper_2007_14178_b200.cli import build_parser
    p = build_parser()
    a = p.parse_args(["bench", "--sizes", "64,128", "--kernel", "5", "--format", "csv", "--word-bits", "32"])
    assert a.sizes == (64, 128) and a.kernel == 5 and a.format == "csv" and a.word_bits == 32
    assert a.repeats == 100 and a.warmup == 10 and a.threads == "all"
    a = p.parse_args(["conv", "--input", "i", "--weights", "w", "--output", "o"])
    assert a.pad is None and a.word_bits == 64
    a = p.parse_args(["verify", "--kernels", "1,3,5,7"])
    assert a.kernels == (1, 3, 5, 7) and a.engine_instances == 200 and a.pipeline_instances == 25
    with pytest.raises(SystemExit):
        p.parse_args(["bench", "--sizes", "a,b"])


@pytest.mark.parametrize("kw,msg", [(dict(sizes=()), "non-empty"), (dict(sizes=(2,), kernel=3), ">= the kernel"),
                                    (dict(kernel=4), "odd"), (dict(channels=0), "channels"),
                                    (dict(repeats=0), "repeats"), (dict(warmup=-1), "warmup"),
                                    (dict(word_bits=16), "word_bits"), (dict(fmt="xml"), "format"),
                                    (dict(threads=0), "threads")])
def test_bench_config_validation(kw, msg):
    from paper_2007_14178_b200.bench import BenchConfig
    with pytest.raises(ValueError, match=msg):
        BenchConfig(**kw)


def test_cli_bench_bad_config_exit_code(capsys):
    from paper_2007_14178_b200.cli import main
    assert main(["bench", "--kernel", "4"]) == 2
    assert "error:" in capsys.readouterr().err


def test_bench_report_csv_round_trip_and_table():
    from paper_2007_14178_b200.bench import BenchReport, BenchRow, emit_report, parse_csv
    rep = BenchReport([BenchRow("vanilla", 256, 1.25, 0.5, 1.0), BenchRow("xnor", 256, 0.1, 0.01, 12.5)])
    assert parse_csv(emit_report(rep, "csv")).rows == rep.rows
    table = emit_report(rep, "table")
    assert "speed-up" in table and "12.50x" in table
    with pytest.raises(ValueError):
        parse_csv("nope")
    with pytest.raises(ValueError):
        emit_report(rep, "xml")


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_run_verification_reference_instances():
    from paper_2007_14178_b200.verify import run_verification
    res = run_verification()
    assert res.ok, res.failures
    assert res.engine_checked == 200 and res.pipeline_checked == 25


@pytest.mark.gpu
def test_run_verification_k1357():
    from paper_2007_14178_b200.verify import run_verification
    res = run_verification(120, 40, seed=5, kernels=(1, 3, 5, 7))
    assert res.ok, res.failures


@pytest.mark.gpu
def test_naive_sign_conv_matches_oracle():
    from paper_2007_14178_b200 import SignPlane, reference
    rng = np.random.default_rng(2)
    for k, pad in ((1, 0), (3, 1), (5, 2), (7, 0), (3, 4)):
        x = O.f32_exact(rng, (3, 13, 11))
        w = O.f32_exact(rng, (3, k, k))
        got = reference.sign_conv2d_int([SignPlane(s) for s in O.signs(x)], [SignPlane(s) for s in O.signs(w)], pad)
        assert np.array_equal(got.values, O.sign_conv2d_int(x, w, pad))


def _loop_conv(x, w, pad, bwn=False, scale=1.0):
    """reference.py:30-54 / 93-122, as plain Python loops (small shapes)."""
    c, h, wd = x.shape
    kh, kw = w.shape[1:]
    oh, ow = h + 2 * pad - kh + 1, wd + 2 * pad - kw + 1
    out = np.empty((oh, ow))
    for y in range(oh):
        for xo in range(ow):
            acc = 0.0
            for ch in range(c):
                for ky in range(kh):
                    iy = y + ky - pad
                    if not 0 <= iy < h:
                        continue
                    for kx in range(kw):
                        ix = xo + kx - pad
                        if 0 <= ix < wd:
                            v = float(x[ch, iy, ix])
                            if bwn:
                                acc = acc + v if w[ch, ky, kx] > 0 else acc - v
                            else:
                                acc += v * float(w[ch, ky, kx])
            out[y, xo] = acc * scale if bwn else acc
    return out


@pytest.mark.gpu
def test_naive_float_convs_match_python_loops():
    from paper_2007_14178_b200 import Tensor3, reference, sign_binarize
    rng = np.random.default_rng(3)
    for k, pad in ((1, 0), (3, 1), (5, 2), (3, 0)):
        x = rng.uniform(-1, 1, (2, 9, 10))
        w = rng.uniform(-1, 1, (2, k, k))
        got = reference.conv2d_float(Tensor3(x), Tensor3(w), pad).data
        assert np.array_equal(got, _loop_conv(x, w, pad))
        ap = sign_binarize(Tensor3(w))
        got = reference.bwn_conv(Tensor3(x), ap, pad).data
        ws = np.stack([p.signs for p in ap.signs]).astype(np.float64)
        assert np.array_equal(got, _loop_conv(x, ws, pad, bwn=True, scale=ap.scale))
    with pytest.raises(ValueError, match="weight channels"):
        reference.conv2d_float(Tensor3(np.ones((2, 4, 4))), Tensor3(np.ones((3, 3, 3))))
    with pytest.raises(ValueError, match="larger than padded"):
        reference.conv2d_float(Tensor3(np.ones((1, 2, 2))), Tensor3(np.ones((1, 3, 3))))


@pytest.mark.gpu
def test_cli_verify_and_conv(tmp_path, capsys):
    from paper_2007_14178_b200 import Tensor3, load_tensor, save_tensor
    from paper_2007_14178_b200.cli import main
    assert main(["verify", "--engine-instances", "30", "--pipeline-instances", "10", "--kernels", "1,3,5,7"]) == 0
    assert "all checks passed" in capsys.readouterr().out
    rng = np.random.default_rng(9)
    x = O.f32_exact(rng, (4, 17, 15))
    w = O.f32_exact(rng, (4, 5, 5))
    save_tensor(Tensor3(x.astype(np.float64)), tmp_path / "x.btsr")
    save_tensor(Tensor3(w.astype(np.float64)), tmp_path / "w.btsr")
    assert main(["conv", "--input", str(tmp_path / "x.btsr"), "--weights", str(tmp_path / "w.btsr"),
                 "--output", str(tmp_path / "y.btsr")]) == 0
    assert "wrote 17x15 output" in capsys.readouterr().out
    y = load_tensor(tmp_path / "y.btsr").data[0]
    want = O.conv_layer(x[None], w[None], 2)[0, 0]
    assert np.array_equal(y.astype(np.float32).view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
def test_cli_bench_csv(capsys):
    from paper_2007_14178_b200.bench import parse_csv
    from paper_2007_14178_b200.cli import main
    assert main(["bench", "--sizes", "48,96", "--channels", "3", "--repeats", "3", "--warmup", "1",
                 "--format", "csv"]) == 0
    rep = parse_csv(capsys.readouterr().out)
    assert [(r.impl, r.size) for r in rep.rows] == [("vanilla", 48), ("xnor", 48), ("vanilla", 96), ("xnor", 96)]
    assert all(r.mean_ms > 0 for r in rep.rows)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_vanilla_conv_kernel_matches_numpy_order(dtype):
    """xnc_vanilla_conv == the reference's _kernels_py.vanilla_conv order (products
    rounded then accumulated in (ch, ky, kx) order from 0)."""
    import torch
    from paper_2007_14178_b200._lib import check, lib
    rng = np.random.default_rng(6)
    p = rng.uniform(-1, 1, (3, 12, 14)).astype(dtype)
    w = rng.uniform(-1, 1, (3, 3, 5)).astype(dtype)
    want = np.zeros((10, 10), dtype=dtype)
    for ch in range(3):
        for ky in range(3):
            for kx in range(5):
                want += p[ch, ky:ky + 10, kx:kx + 10] * w[ch, ky, kx]
    pd, wd = torch.from_numpy(p).cuda(), torch.from_numpy(w).cuda()
    out = torch.empty((10, 10), dtype=pd.dtype, device="cuda")
    check(lib().xnc_vanilla_conv(pd.data_ptr(), 0 if dtype == np.float32 else 1, 3, 12, 14, wd.data_ptr(), 3, 5,
                                 out.data_ptr(), None), "xnc_vanilla_conv")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
