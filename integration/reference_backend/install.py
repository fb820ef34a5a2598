"""Add the b200 backend to a copy of the reference `xnorconv` package.

`install(pkg_dir)` copies `_kernels_b200.py` into `pkg_dir` (a directory laid out
like /root/reference/pkg/src/xnorconv) and applies the two edits of
INTEGRATION.md section 1 to its `_backend.py` (_backend.py:13-41): import the
module when libxnorb200.so loads, and answer `get_kernels("b200")` with it.
Nothing else in the reference changes.  Used by tests/test_gpu_reference_backend.py
on a scratch copy of baseline/_ref/xnorconv (the reference as pip installed).

    python integration/reference_backend/install.py <path to xnorconv package dir>
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

_IMPORT_ANCHOR = "HAVE_COMPILED = _kernels_cy is not None\n"
_IMPORT_EDIT = (
    "try:\n"
    "    from . import _kernels_b200\n"
    "except OSError:  # libxnorb200.so or the CUDA runtime is not loadable\n"
    "    _kernels_b200 = None\n"
    "\n"
)
_GET_ANCHOR = '    if backend == "python":\n        return _kernels_py\n'
_GET_EDIT = (
    '    if backend == "b200":\n'
    "        if _kernels_b200 is None:\n"
    '            raise RuntimeError("b200 kernels are not available: libxnorb200.so did not load")\n'
    "        return _kernels_b200\n"
)
_BACKENDS_OLD = 'BACKENDS = ("compiled", "python")'
_BACKENDS_NEW = 'BACKENDS = ("compiled", "python", "b200")'


def patch_backend_source(src: str) -> str:
    """The _backend.py edit, applied to its source text (fails loudly on drift)."""
    if "_kernels_b200" in src:
        return src
    for anchor in (_IMPORT_ANCHOR, _GET_ANCHOR, _BACKENDS_OLD):
        if anchor not in src:
            raise ValueError(f"_backend.py does not look like the reference's: missing {anchor!r}")
    src = src.replace(_IMPORT_ANCHOR, _IMPORT_EDIT + _IMPORT_ANCHOR, 1)
    src = src.replace(_GET_ANCHOR, _GET_EDIT + _GET_ANCHOR, 1)
    return src.replace(_BACKENDS_OLD, _BACKENDS_NEW, 1)


def install(pkg_dir: str) -> None:
    shutil.copy(os.path.join(HERE, "_kernels_b200.py"), os.path.join(pkg_dir, "_kernels_b200.py"))
    be = os.path.join(pkg_dir, "_backend.py")
    with open(be) as fh:
        src = fh.read()
    with open(be, "w") as fh:
        fh.write(patch_backend_source(src))


if __name__ == "__main__":
    install(sys.argv[1])
