"""Loader for the committed golden vectors (tests/golden/golden_v1.npz,
generated from the reference by tests/golden/make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_CACHE = {}


def load():
    if "g" not in _CACHE:
        _CACHE["g"] = dict(np.load(os.path.join(HERE, "golden_v1.npz")))
        with open(os.path.join(HERE, "golden_v1.json")) as fh:
            _CACHE["m"] = json.load(fh)
    return _CACHE["g"], _CACHE["m"]


def layer_cases():
    g, m = load()
    out = []
    for c in m["layer_cases"]:
        p = f"layer/{c['name']}/"
        out.append(dict(c, **{k: g[p + k] for k in ("x", "w", "out", "ints", "alpha")}))
    return out


def pack_cases():
    g, m = load()
    return [dict(c, plane=g[f"pack/{c['name']}/plane"], words=g[f"pack/{c['name']}/words"]) for c in m["pack_cases"]]


def scale_cases():
    g, m = load()
    keys = ("x", "w", "A", "K", "ints", "y", "weight_words", "alpha", "base_mask")
    return [dict(c, **{k: g[f"scale/{c['name']}/{k}"] for k in keys}) for c in m["scale_cases"]]
