"""Shared fixtures. GPU tests are marked `gpu` (run on a B200 via gpurun);
everything else runs on the CPU-only build container.

The golden fixtures under tests/golden/ were produced by the reference
package itself (tests/golden/make_golden.py); nothing here reads
/root/reference at run time.
"""

from __future__ import annotations

import json
import os
import sys
from functools import lru_cache

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_1303_1651_b200.formats import CsrMatrix  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: full-size configs (tens of seconds)")


@lru_cache(maxsize=1)
def _small():
    return np.load(os.path.join(GOLDEN, "small_cases.npz"))


def golden_names():
    return [str(n) for n in _small()["_names"]]


def golden_case(name):
    """(a, b, c_ref, mults, row_choices) for one reference-computed case."""
    z = _small()

    def m(tag):
        rows, cols = (int(x) for x in z[f"{name}/{tag}_shape"])
        return CsrMatrix(rows, cols, z[f"{name}/{tag}_rp"].copy(), z[f"{name}/{tag}_ci"].copy(),
                         z[f"{name}/{tag}_v"].copy())

    return (m("a"), m("b"), m("c"), int(z[f"{name}/mults"][0]),
            z[f"{name}/row_choices"].copy())


def golden_splitmix(seed):
    return _small()[f"splitmix64/{seed}"]


@lru_cache(maxsize=1)
def fingerprints():
    path = os.path.join(GOLDEN, "fingerprints.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        return json.load(f)


def assert_csr_bitwise_equal(got, ref, label=""):
    assert (got.rows, got.cols) == (ref.rows, ref.cols), label
    assert np.asarray(got.row_ptr, np.uint64).tobytes() == np.asarray(ref.row_ptr, np.uint64).tobytes(), \
        f"{label}: row_ptr differs"
    assert np.asarray(got.col_idx, np.uint64).tobytes() == np.asarray(ref.col_idx, np.uint64).tobytes(), \
        f"{label}: col_idx differs"
    gv = np.asarray(got.values, np.float64)
    rv = np.asarray(ref.values, np.float64)
    if gv.tobytes() != rv.tobytes():
        # parity bar (north_star): values within 1e-12 relative to the reference
        assert np.allclose(gv, rv, rtol=1e-12, atol=0.0), f"{label}: values beyond 1e-12"
        pytest.fail(f"{label}: values within 1e-12 but not bit-identical "
                    f"({int(np.sum(gv != rv))} differ); the accumulation order drifted")


def have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
