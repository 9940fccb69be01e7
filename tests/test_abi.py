"""The C-ABI library builds, loads without a GPU, and exports every symbol
the public headers declare; error paths that need no device behave."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT, have_gpu

HEADERS = sorted(os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))
                 if h.endswith(".h"))


def declared_functions():
    names = []
    for h in HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(spmmm_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_headers_declare_the_boundary():
    names = declared_functions()
    for required in ("spmmm_multiply", "spmmm_product_download", "spmmm_estimate_nnz",
                     "spmmm_context_create", "spmmm_last_error", "spmmm_gen_random_k"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1303_1651_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    assert set(declared_functions()) == set(_lib.EXPORTS)


def test_abi_version_and_error_string():
    from paper_1303_1651_b200 import _lib

    assert _lib.lib().spmmm_abi_version() == 1
    assert isinstance(_lib.last_error(), str)


def test_null_arguments_are_rejected_without_a_device():
    from paper_1303_1651_b200 import _lib

    lib = _lib.lib()
    assert lib.spmmm_device_count(None) == _lib.ERR_INVALID
    assert "NULL" in _lib.last_error()
    assert lib.spmmm_multiply(None, None, None, 6, 0, None) == _lib.ERR_INVALID
    assert lib.spmmm_product_shape(None, None, None, None, None) == _lib.ERR_INVALID
    assert lib.spmmm_product_destroy(None) == _lib.OK
    assert lib.spmmm_context_destroy(None) == _lib.OK


@pytest.mark.skipif(have_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly_not_silently():
    """Without a CUDA device the product path raises; it never falls back."""
    from paper_1303_1651_b200 import _lib
    from paper_1303_1651_b200.genmat import gen_fd
    from paper_1303_1651_b200.kernels import multiply_rowmajor

    a = gen_fd(4)
    with pytest.raises(RuntimeError):
        multiply_rowmajor(a, a)
    with pytest.raises(RuntimeError):
        _lib.Context(0)


def test_built_for_sm_100a():
    import subprocess

    from paper_1303_1651_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_row_classes_are_reported_without_a_device():
    """spmmm_row_classes (bench.py attributes a skewed input's products to the
    kernels that compute them): the split-mode limits, consistent with each
    other, and NULL is rejected."""
    import ctypes

    from paper_1303_1651_b200 import _lib

    lib = _lib.lib()
    assert lib.spmmm_row_classes(None) == _lib.ERR_INVALID
    lim = (ctypes.c_uint32 * 5)()
    assert lib.spmmm_row_classes(lim) == _lib.OK
    warp_limit, part_limit, rcap, minrun, half = (int(x) for x in lim)
    assert 32 < warp_limit < part_limit      # warp rows, then block rows, then parts
    assert 0 < rcap <= warp_limit            # the others are sorted by one warp
    assert minrun >= 32 and half in (0, 1)
