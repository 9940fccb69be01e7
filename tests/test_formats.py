"""Storage orders: the CPU oracle's transpose and
column-major product pinned against the reference's own outputs
(tests/golden/formats_cases.npz, made by make_golden.py formats), and the
GPU path (multiply_colmajor / multiply_mixed / csr_to_csc / csc_to_csr /
estimate_nnz_csc) against the same fixtures and the oracle."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from conftest import have_gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats_cases.npz")


def _load():
    return np.load(GOLDEN)


def _names():
    return [str(n) for n in _load()["_names"]]


class _M:
    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def nnz(self):
        return int(self.values.size)


def _mat(z, prefix, csc):
    rows, cols = (int(x) for x in z[f"{prefix}_shape"])
    ptr, idx, v = z[f"{prefix}_ptr"], z[f"{prefix}_idx"], z[f"{prefix}_v"]
    if csc:
        return _M(rows=rows, cols=cols, col_ptr=ptr, row_idx=idx, values=v)
    return _M(rows=rows, cols=cols, row_ptr=ptr, col_idx=idx, values=v)


def _same(x, y, what):
    x, y = np.asarray(x), np.asarray(y)
    assert x.dtype == y.dtype and x.shape == y.shape, what
    assert x.tobytes() == y.tobytes(), what


@pytest.mark.parametrize("name", _names())
def test_oracle_transpose_matches_reference(name):
    z = _load()
    a = _mat(z, f"{name}/a", False)
    ref = _mat(z, f"{name}/a_csc", True)
    ptr, idx, v = oracle.transpose(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    _same(ptr, ref.col_ptr, "col_ptr")
    _same(idx, ref.row_idx, "row_idx")
    _same(v, ref.values, "values")


@pytest.mark.parametrize("name", _names())
def test_oracle_colmajor_matches_reference(name):
    z = _load()
    a, b = _mat(z, f"{name}/a_csc", True), _mat(z, f"{name}/b_csc", True)
    ref = _mat(z, f"{name}/col", True)
    r = oracle.multiply_colmajor(a, b, row_choices=True)
    _same(r.row_ptr, ref.col_ptr, "col_ptr")
    _same(r.col_idx, ref.row_idx, "row_idx")
    _same(r.values, ref.values, "values")
    assert r.multiplications == int(z[f"{name}/col_mults"][0])
    if b.cols:  # zero-row results: the reference's sentinel quirk, checked on the GPU path
        if a.rows:
            np.testing.assert_array_equal(r.row_choices, z[f"{name}/col_choices"])


# ---------------------------------------------------------------------------
# GPU path (through libspmmm.so)

gpu = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]


def _choices(stats, n):
    out = np.full(n, -1, np.int8)
    for r, ch in stats.row_choices:
        out[r] = 0 if ch.value == "minmax" else 1
    return out


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", _names())
def test_gpu_storage_orders_match_reference(name):
    from paper_1303_1651_b200 import (KernelStats, StrategyKind, csc_to_csr, csr_to_csc,
                                      estimate_nnz_csc, multiply_colmajor, multiply_mixed)
    from paper_1303_1651_b200.formats import CscMatrix, CsrMatrix

    z = _load()
    a = CsrMatrix.from_arrays(*z[f"{name}/a_shape"], z[f"{name}/a_ptr"], z[f"{name}/a_idx"],
                              z[f"{name}/a_v"])
    b = CsrMatrix.from_arrays(*z[f"{name}/b_shape"], z[f"{name}/b_ptr"], z[f"{name}/b_idx"],
                              z[f"{name}/b_v"])
    # conversions
    a_csc = csr_to_csc(a)
    ref = _mat(z, f"{name}/a_csc", True)
    _same(a_csc.col_ptr, ref.col_ptr, "csr_to_csc ptr")
    _same(a_csc.row_idx, ref.row_idx, "csr_to_csc idx")
    _same(a_csc.values, ref.values, "csr_to_csc values")
    back = csc_to_csr(a_csc)
    _same(back.row_ptr, a.row_ptr, "round trip ptr")
    _same(back.col_idx, a.col_idx, "round trip idx")
    _same(back.values, a.values, "round trip values")
    b_csc = csr_to_csc(b)
    assert estimate_nnz_csc(a_csc, b_csc) == int(z[f"{name}/estimate_csc"][0])
    # column-major product
    st = KernelStats()
    c = multiply_colmajor(a_csc, b_csc, StrategyKind.COMBINED, st)
    assert isinstance(c, CscMatrix)
    ref = _mat(z, f"{name}/col", True)
    _same(c.col_ptr, ref.col_ptr, "colmajor ptr")
    _same(c.row_idx, ref.row_idx, "colmajor idx")
    _same(c.values, ref.values, "colmajor values")
    assert st.multiplications == int(z[f"{name}/col_mults"][0])
    np.testing.assert_array_equal(_choices(st, b.cols), z[f"{name}/col_choices"])
    # mixed: CSR x CSC -> CSR (B converted), CSC x CSR -> CSC (B converted)
    for tag, lhs, rhs, out_cls, n_major in (("mix_rc", a, b_csc, CsrMatrix, a.rows),
                                            ("mix_cr", a_csc, b, CscMatrix, b.cols)):
        st = KernelStats()
        c = multiply_mixed(lhs, rhs, StrategyKind.COMBINED, st)
        assert isinstance(c, out_cls), tag
        ref = _mat(z, f"{name}/{tag}", out_cls is CscMatrix)
        ptr, idx = ((c.col_ptr, c.row_idx) if out_cls is CscMatrix else (c.row_ptr, c.col_idx))
        rptr, ridx = ((ref.col_ptr, ref.row_idx) if out_cls is CscMatrix
                      else (ref.row_ptr, ref.col_idx))
        _same(ptr, rptr, f"{tag} ptr")
        _same(idx, ridx, f"{tag} idx")
        _same(c.values, ref.values, f"{tag} values")
        assert st.multiplications == int(z[f"{name}/{tag}_mults"][0]), tag
        assert st.conversions == int(z[f"{name}/{tag}_conv"][0]), tag
        np.testing.assert_array_equal(_choices(st, n_major), z[f"{name}/{tag}_choices"])
    # same-order pairs dispatch without conversions
    st = KernelStats()
    multiply_mixed(a_csc, b_csc, StrategyKind.COMBINED, st)
    multiply_mixed(a, b, StrategyKind.COMBINED, st)
    assert st.conversions == 0


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("seed,shape", [(1, (3000, 2500, 2000, 12, 9)),
                                        (2, (400, 3000, 5000, 300, 40)),    # long rows
                                        (3, (20000, 20000, 20000, 5, 5))])  # ELL path
def test_gpu_colmajor_larger_vs_oracle(seed, shape):
    from paper_1303_1651_b200 import csr_to_csc, multiply_colmajor, multiply_mixed
    from paper_1303_1651_b200.formats import CsrMatrix

    rows, inner, cols, amax, bmax = shape
    rng = np.random.default_rng(seed)

    def rand(r, c, m):
        lens = np.minimum(rng.integers(0, m + 1, size=r), c)
        rp = np.zeros(r + 1, np.uint64)
        rp[1:] = np.cumsum(lens)
        ci = np.concatenate([np.sort(rng.choice(c, n, replace=False)) for n in lens]
                            ).astype(np.uint64) if rp[-1] else np.zeros(0, np.uint64)
        return CsrMatrix(r, c, rp, ci, rng.uniform(-1, 1, ci.size))

    a, b = rand(rows, inner, amax), rand(inner, cols, bmax)
    a_csc, b_csc = csr_to_csc(a), csr_to_csc(b)
    r = oracle.multiply_colmajor(a_csc, b_csc)
    c = multiply_colmajor(a_csc, b_csc)
    _same(c.col_ptr, r.row_ptr, "ptr")
    _same(c.row_idx, r.col_idx, "idx")
    _same(c.values, r.values, "values")
    c2 = multiply_mixed(a_csc, b)
    _same(c2.col_ptr, r.row_ptr, "mixed ptr")
    _same(c2.values, r.values, "mixed values")
