"""The reference package itself, running on libxnorb200.so.

A scratch copy of the UNMODIFIED reference `xnorconv` (pip-installed into
baseline/_ref) gets the b200 backend the way a
maintainer would add it (integration/reference_backend: `_kernels_b200.py` +
the `_backend.get_kernels` edit of INTEGRATION.md section 1, reference
_backend.py:28-41).  Then the reference's own code -- ConvWorkspace.run /
int_plane / grids, pack, xnor_conv_multichannel, input_scale_map and
verify.run_verification -- runs with backend="b200" and is checked against the
reference-generated golden vectors and against the reference's own compiled
backend in the same process.

CPU tests: the edit applies and the patched package imports and routes
get_kernels("b200") to the ctypes module (no device call).  GPU tests: the
numbers."""
import importlib
import os
import shutil
import sys

import numpy as np
import pytest

from tests import golden_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "xnorconv")
LIB = os.path.join(ROOT, "paper_2007_14178_b200", "libxnorb200.so")

needs_ref = pytest.mark.skipif(not os.path.isdir(REF_PKG),
                               reason="reference not installed in baseline/_ref (DESIGN.md: Reference install)")


@pytest.fixture(scope="module")
def xnorconv(tmp_path_factory):
    """The reference package with the b200 backend installed, imported as `xnorconv`."""
    if not os.path.isdir(REF_PKG):
        pytest.skip("reference not installed in baseline/_ref")
    from paper_2007_14178_b200._build import build_library
    build_library()  # the in-tree .so the binding loads (no-op when fresh)
    sys.path.insert(0, os.path.join(ROOT, "integration", "reference_backend"))
    import install
    dst = tmp_path_factory.mktemp("refpkg")
    shutil.copytree(REF_PKG, dst / "xnorconv", ignore=shutil.ignore_patterns("__pycache__"))
    install.install(str(dst / "xnorconv"))
    os.environ["XNORB200_LIB"] = LIB
    saved = {k: v for k, v in sys.modules.items() if k == "xnorconv" or k.startswith("xnorconv.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, str(dst))
    try:
        mod = importlib.import_module("xnorconv")
        assert os.path.dirname(mod.__file__) == str(dst / "xnorconv")
        yield mod
    finally:
        sys.path.remove(str(dst))
        for k in [k for k in sys.modules if k == "xnorconv" or k.startswith("xnorconv.")]:
            del sys.modules[k]
        sys.modules.update(saved)


# ---------------------------------------------------------------- CPU: the plumbing
@needs_ref
def test_backend_edit_applies_to_the_installed_reference():
    sys.path.insert(0, os.path.join(ROOT, "integration", "reference_backend"))
    import install
    with open(os.path.join(REF_PKG, "_backend.py")) as fh:
        src = fh.read()
    out = install.patch_backend_source(src)
    assert "_kernels_b200" in out and '"b200"' in out
    assert install.patch_backend_source(out) == out  # idempotent
    with pytest.raises(ValueError):
        install.patch_backend_source("BACKENDS = ()\n")


@needs_ref
def test_patched_reference_routes_b200(xnorconv):
    from xnorconv import _backend
    k = _backend.get_kernels("b200")
    assert k.__name__ == "xnorconv._kernels_b200"
    for name in ("pack_plane", "xnor_accumulate", "box_mean", "scale_rows", "scale_join",
                 "xnor_reconstruct", "vanilla_conv"):
        assert callable(getattr(k, name))
    assert _backend.get_kernels("python").__name__ == "xnorconv._kernels_py"
    with pytest.raises(ValueError):
        k.pack_plane(np.zeros((4, 4), np.float32)[:, ::2], 1, 1, 8, 8, 6, 6, np.zeros((1, 1), np.uint64), 1)
    with pytest.raises(ValueError):
        k.pack_plane(np.zeros((4, 4), np.float32), 1, 1, 8, 8, 6, 6, np.zeros((1, 1), np.int64), 1)


# ---------------------------------------------------------------- GPU: the numbers
@pytest.mark.gpu
@needs_ref
def test_reference_run_verification_on_b200(xnorconv):
    """verify.run_verification (verify.py:133-145): 200 engine + 25 pipeline instances,
    exact ints and <= 1e-5 floats, all through the b200 kernels."""
    from xnorconv.verify import run_verification
    res = run_verification(200, 25, seed=0, backend="b200")
    assert res.ok, res.failures
    assert res.engine_checked == 200 and res.pipeline_checked == 25


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("two_stream", [False, True])
@pytest.mark.parametrize("case", [c for c in golden_io.layer_cases() if c["N"] * c["O"] <= 8],
                         ids=lambda c: c["name"])
def test_reference_workspace_on_b200_matches_golden(xnorconv, case, two_stream):
    """The reference's own ConvWorkspace (pipeline.py:40-173) with backend='b200':
    run() (fused xnor_reconstruct, or the two-stream split path) and int_plane()
    bit-exact to the golden vectors the reference's compiled backend produced."""
    N, C, H, W, Oc = case["N"], case["C"], case["H"], case["W"], case["O"]
    ws = xnorconv.ConvWorkspace(C, H, W, case["kh"], case["kw"], case["pad"], case["word_bits"],
                                backend="b200")
    for n in range(N):
        ws.load_input(xnorconv.Tensor3(case["x"][n].astype(np.float64)))
        for o in range(Oc):
            ws.set_weights(xnorconv.Tensor3(case["w"][o].astype(np.float64)))
            out = ws.run(threads=4, two_stream=two_stream)
            assert np.array_equal(out.view(np.uint32), case["out"][n, o].view(np.uint32))
            assert np.array_equal(ws.int_plane().values, case["ints"][n, o])
    ws.close()


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("case", golden_io.pack_cases(), ids=lambda c: c["name"])
def test_reference_pack_on_b200_matches_golden(xnorconv, case):
    """pack.pack (pack.py:105-120) with backend='b200', and unpack of its words."""
    geom = xnorconv.TileGeometry(case["word_bits"], case["kh"], case["kw"])
    signs = xnorconv.sign_plane(xnorconv.Tensor2(case["plane"].astype(np.float64)))
    grid = xnorconv.pack(signs, geom, backend="b200")
    assert np.array_equal(grid.words, case["words"])
    back = xnorconv.unpack(grid, signs.height, signs.width)
    assert np.array_equal(back.signs, signs.signs)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("k", [1, 3, 5, 7])
@pytest.mark.parametrize("word_bits", [64, 32])
def test_reference_b200_equals_reference_compiled(xnorconv, k, word_bits):
    """Same reference code, two backends, same inputs: the b200 kernels and the
    reference's compiled kernels (threads=1, its race-free path) agree bit for bit
    -- fused run, int plane, engine path and the float64 scale map."""
    if word_bits == 32 and k > 4:
        pytest.skip("k > tile width 4 of 32-bit words (pack.py:45-53)")
    from xnorconv import _backend
    if not _backend.HAVE_COMPILED:
        pytest.skip("reference compiled backend not built")
    rng = np.random.default_rng(100 + k)
    C, H, W = 9, 23, 30
    x = rng.uniform(-1, 1, (C, H, W)).astype(np.float32).astype(np.float64)
    w = rng.uniform(-1, 1, (C, k, k)).astype(np.float32).astype(np.float64)
    pad = (k - 1) // 2
    outs = {}
    for be in ("compiled", "b200"):
        ws = xnorconv.ConvWorkspace(C, H, W, k, k, pad, word_bits, backend=be)
        ws.load_input(xnorconv.Tensor3(x))
        ws.set_weights(xnorconv.Tensor3(w))
        y = ws.run(threads=1).copy()
        ints = ws.int_plane().values
        geom = xnorconv.TileGeometry(word_bits, k, k)
        grids = [xnorconv.pack(xnorconv.sign_plane(xnorconv.Tensor2(ch)), geom, backend=be)
                 for ch in xnorconv.zero_pad(xnorconv.Tensor3(x), pad).data]
        filt = xnorconv.build_filter(xnorconv.Tensor3(w), geom)
        eng = xnorconv.xnor_conv_multichannel(grids, filt, ints.shape[0], ints.shape[1], backend=be).values
        K = xnorconv.input_scale_map(xnorconv.channel_abs_mean(xnorconv.Tensor3(x)), k, k, pad, backend=be).data
        outs[be] = (y, ints, eng, K)
    for a, b in zip(outs["compiled"], outs["b200"]):
        assert a.dtype == b.dtype and np.array_equal(a, b)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_reference_vanilla_conv_b200_equals_python(xnorconv, dtype):
    """vanilla_conv (_kernels_py.py:90-108 order: products rounded, then added, in
    (ch, ky, kx) order) -- the b200 kernel and the reference's numpy fallback agree bit for bit."""
    from xnorconv import _backend
    rng = np.random.default_rng(4)
    padded = rng.uniform(-1, 1, (5, 21, 19)).astype(dtype)
    w = rng.uniform(-1, 1, (5, 3, 3)).astype(dtype)
    outs = []
    for be in ("python", "b200"):
        out = np.empty((19, 17), dtype=dtype)
        _backend.get_kernels(be).vanilla_conv(padded, w, out, 1)
        outs.append(out)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.gpu
@needs_ref
def test_reference_bench_harness_on_b200(xnorconv):
    """The reference's own bench (bench.py:223-260) with backend='b200': its
    pre-timing gates (exact ints vs the naive loops, decomposition <= 1e-5, bwn
    and vanilla interior checks, thread-count invariance) all pass on our kernels."""
    from xnorconv.bench import BenchConfig, emit_report, parse_csv, run_bench
    cfg = BenchConfig(sizes=(48, 64), kernel=3, channels=2, repeats=2, warmup=1, threads=2, backend="b200")
    report = run_bench(cfg)
    assert {r.impl for r in report.rows} == {"vanilla-1t", "vanilla-mt", "xnor-1t", "xnor-mt"}
    assert parse_csv(emit_report(report, "csv")).rows == report.rows
