"""Generate golden vectors by running the REFERENCE itself (xnorconv, imported
from /root/reference/pkg/src) in this container.  /root/reference does not
exist on the GPU box, so the outputs are committed as tests/golden/golden_v1.npz
and this script is kept beside them.

Backend: the reference's own compiled kernels (oracle/_ref/_kernels_cy*.so,
built from the reference .pyx by oracle/build_ref.sh), injected as
xnorconv._kernels_cy before the package import -- i.e. the stock compiled
path, at threads=1 (the race-free configuration).
Falls back to the reference's numpy backend (bit-identical, SURVEY.md section 0
item 5) only if the compiled module is missing.

Run:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import glob
import importlib.util
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")


def import_reference():
    so = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_kernels_cy*.so"))
    if so:
        spec = importlib.util.spec_from_file_location("xnorconv._kernels_cy", so[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["xnorconv._kernels_cy"] = mod
    sys.path.insert(0, REF_SRC)
    import xnorconv  # noqa: E402
    return xnorconv


def main():
    xc = import_reference()
    backend = "compiled" if xc.compiled_available() else "python"
    from xnorconv.reference import sign_conv2d_int
    arrays: dict[str, np.ndarray] = {}
    manifest = {"generator": "tests/golden/make_golden.py", "reference_backend": backend,
                "reference": "xnorconv 0.1.0 (/root/reference/pkg)", "layer_cases": [], "pack_cases": [],
                "scale_cases": []}

    def f32(rng, shape, lo=-1.0, hi=1.0):
        return rng.uniform(lo, hi, shape).astype(np.float32)

    # ---------------------------------------------------------------- layer cases
    # (name, N, C, H, W, O, kh, kw, pad, word_bits, distribution)
    cases = [
        ("c1_slice", 1, 64, 32, 32, 8, 3, 3, 1, 64, "uniform"),   # BASELINE config 1 shape, 8 of 64 filters
        ("k1_c3", 2, 3, 9, 13, 3, 1, 1, 0, 64, "uniform"),
        ("k1_pad2", 1, 2, 7, 6, 2, 1, 1, 2, 32, "uniform"),
        ("k3_c1", 1, 1, 16, 16, 2, 3, 3, 1, 64, "uniform"),
        ("k3_c31", 2, 31, 11, 10, 4, 3, 3, 1, 64, "uniform"),
        ("k3_c33", 1, 33, 12, 9, 3, 3, 3, 1, 32, "uniform"),
        ("k3_pad0", 1, 5, 10, 14, 2, 3, 3, 0, 64, "uniform"),
        ("k3_pad3", 1, 4, 6, 7, 2, 3, 3, 3, 64, "uniform"),
        ("k5_c7", 2, 7, 13, 12, 3, 5, 5, 2, 64, "uniform"),
        ("k5_c64", 1, 64, 9, 11, 2, 5, 5, 2, 64, "uniform"),
        ("k7_c3", 1, 3, 15, 17, 3, 7, 7, 3, 64, "uniform"),
        ("k7_c96", 1, 96, 8, 8, 2, 7, 7, 3, 64, "uniform"),
        ("k7_pad1", 1, 6, 12, 12, 2, 7, 7, 1, 64, "uniform"),
        ("k3x5_rect", 1, 9, 10, 12, 2, 3, 5, 2, 64, "uniform"),
        ("k5x3_rect", 1, 9, 12, 10, 2, 5, 3, 1, 64, "uniform"),
        ("k3x1_w32", 1, 4, 9, 9, 2, 3, 1, 1, 32, "uniform"),
        ("zeros_negzeros", 1, 8, 10, 10, 3, 3, 3, 1, 64, "zeros"),
        ("all_negative", 1, 5, 8, 9, 2, 3, 3, 1, 64, "negative"),
        ("sign_dominated", 1, 6, 12, 12, 2, 3, 3, 1, 64, "dominated"),
        ("tiny_1x1_image", 1, 2, 1, 1, 2, 3, 3, 1, 64, "uniform"),
        ("c257_tail", 1, 257, 5, 6, 2, 3, 3, 1, 64, "uniform"),
    ]
    for (name, N, C, H, W, O, kh, kw, pad, wb, dist) in cases:
        rng = np.random.default_rng([ord(ch) for ch in name])
        if dist == "uniform":
            x = f32(rng, (N, C, H, W)); w = f32(rng, (O, C, kh, kw))
        elif dist == "zeros":
            x = f32(rng, (N, C, H, W)); w = f32(rng, (O, C, kh, kw))
            m = rng.integers(0, 3, x.shape)
            x[m == 0] = 0.0; x[m == 1] = -0.0
            wm = rng.integers(0, 3, w.shape)
            w[wm == 0] = 0.0; w[wm == 1] = -0.0
        elif dist == "negative":
            x = -np.abs(f32(rng, (N, C, H, W))) - np.float32(0.01); w = f32(rng, (O, C, kh, kw))
        else:  # bench.py:111-117 sign-dominated
            x = ((rng.integers(0, 2, (N, C, H, W)) * 2 - 1) * 0.75).astype(np.float32)
            w = ((rng.integers(0, 2, (O, C, kh, kw)) * 2 - 1) * 0.5).astype(np.float32)
        oh, ow = H + 2 * pad - kh + 1, W + 2 * pad - kw + 1
        out = np.zeros((N, O, oh, ow), np.float32)
        ints = np.zeros((N, O, oh, ow), np.int32)
        alphas = np.zeros(O, np.float64)
        for n in range(N):
            ws = xc.ConvWorkspace(C, H, W, kh, kw, pad, wb, backend)
            ws.load_input(xc.Tensor3(x[n].astype(np.float64)))
            for o in range(O):
                ws.set_weights(xc.Tensor3(w[o].astype(np.float64)))
                out[n, o] = ws.run(threads=1)
                ints[n, o] = ws.int_plane().values
                alphas[o] = ws.filter.scale
                # cross-check the integer truth tier on the way (reference.py:58-90)
                if C * H * W * O <= 20000:
                    pz = xc.zero_pad(xc.Tensor3(x[n].astype(np.float64)), pad)
                    want = sign_conv2d_int([xc.sign_plane(xc.Tensor2(ch)) for ch in pz.data],
                                           xc.sign_binarize(xc.Tensor3(w[o].astype(np.float64))).signs)
                    assert np.array_equal(want.values, ints[n, o]), name
            ws.close()
            # the one-shot wrapper must agree with the workspace path
            one = xc.xnor_conv(xc.Tensor3(x[n].astype(np.float64)), xc.Tensor3(w[0].astype(np.float64)),
                               pad=pad, word_bits=wb, backend=backend)
            assert np.array_equal(one.data.astype(np.float32), out[n, 0]), name
        for key, arr in (("x", x), ("w", w), ("out", out), ("ints", ints), ("alpha", alphas)):
            arrays[f"layer/{name}/{key}"] = arr
        manifest["layer_cases"].append({"name": name, "N": N, "C": C, "H": H, "W": W, "O": O, "kh": kh,
                                        "kw": kw, "pad": pad, "word_bits": wb, "dist": dist})

    # ---------------------------------------------------------------- pack cases (pack.py:105-120)
    for (name, h, w, kh, kw, wb) in [("p64_k3", 18, 21, 3, 3, 64), ("p32_k3", 14, 13, 3, 3, 32),
                                     ("p64_k7", 16, 16, 7, 7, 64), ("p64_k1", 9, 9, 1, 1, 64),
                                     ("p32_k1x4", 11, 10, 1, 4, 32)]:
        rng = np.random.default_rng([ord(ch) for ch in name])
        plane = f32(rng, (h, w)).astype(np.float64)
        geom = xc.TileGeometry(wb, kh, kw)
        grid = xc.pack(xc.sign_plane(xc.Tensor2(plane)), geom, backend)
        arrays[f"pack/{name}/plane"] = plane
        arrays[f"pack/{name}/words"] = grid.words.copy()
        manifest["pack_cases"].append({"name": name, "h": h, "w": w, "kh": kh, "kw": kw, "word_bits": wb})

    # ---------------------------------------------------------------- float64 operator API
    # channel_abs_mean -> input_scale_map -> apply_scaling (scaling.py:32-98), sign_binarize
    for (name, C, H, W, k, pad) in [("s_k3", 5, 11, 13, 3, 1), ("s_k5", 3, 9, 8, 5, 2), ("s_k1", 2, 6, 7, 1, 0),
                                    ("s_k3_pad0", 4, 10, 10, 3, 0), ("s_c64_k3", 64, 12, 12, 3, 1)]:
        rng = np.random.default_rng([ord(ch) for ch in name])
        x = f32(rng, (C, H, W)).astype(np.float64)
        w = f32(rng, (C, k, k)).astype(np.float64)
        t = xc.Tensor3(x)
        A = xc.channel_abs_mean(t)
        approx = xc.sign_binarize(xc.Tensor3(w))
        field = xc.input_scaling_field(t, k, k, pad, approx.scale, backend)
        K = xc.input_scale_map(A, k, k, pad, backend)
        pz = xc.zero_pad(t, pad)
        geom = xc.TileGeometry(64, k, k)
        grids = [xc.pack(xc.sign_plane(xc.Tensor2(ch)), geom, backend) for ch in pz.data]
        filt = xc.build_filter(xc.Tensor3(w), geom)
        oh, ow = H + 2 * pad - k + 1, W + 2 * pad - k + 1
        ints = xc.xnor_conv_multichannel(grids, filt, oh, ow, backend)
        y = xc.apply_scaling(ints, field)
        for key, arr in (("x", x), ("w", w), ("A", A.data), ("K", K.data), ("ints", ints.values),
                         ("y", y.data), ("weight_words", filt.weight_words),
                         ("alpha", np.array([approx.scale])), ("base_mask", np.array([filt.base_mask], np.uint64))):
            arrays[f"scale/{name}/{key}"] = np.asarray(arr)
        manifest["scale_cases"].append({"name": name, "C": C, "H": H, "W": W, "k": k, "pad": pad})

    np.savez_compressed(OUT, **arrays)
    with open(OUT.replace(".npz", ".json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB), backend={backend}")


if __name__ == "__main__":
    main()
