"""Host-side logic of the drop-in that runs before (or around) the C ABI:
argument validation with the reference's exceptions, the Combined rule,
CSR helpers, row partitioning, block concatenation, and the install hook."""

from __future__ import annotations

import sys
import types

import numpy as np
import pytest

import oracle
from conftest import golden_case
from paper_1303_1651_b200.distributed import concat_row_blocks, partition_rows, row_block_host
from paper_1303_1651_b200.formats import CsrMatrix, make_like, validate_csr
from paper_1303_1651_b200.kernels import (KernelStats, StrategyKind, combined_select,
                                          multiply_rowmajor)
from paper_1303_1651_b200.perfmodel import bytes_alg, inner_loop_balance, roofline


def test_dimension_mismatch_raises_before_the_abi():
    a = CsrMatrix.from_dense(np.ones((2, 3)))
    b = CsrMatrix.from_dense(np.ones((2, 2)))
    with pytest.raises(ValueError, match=r"dimension mismatch: 3 \(cols of a\) != 2 \(rows of b\)"):
        multiply_rowmajor(a, b)


def test_unknown_strategy_raises_value_error():
    a = CsrMatrix.from_dense(np.eye(2))
    with pytest.raises(ValueError):
        multiply_rowmajor(a, a, "quicksort")


def test_strategy_enum_matches_reference_values():
    assert [s.value for s in StrategyKind] == [
        "bfdouble", "bfbool", "bfchar", "minmax", "minmaxchar", "sort", "combined"]


@pytest.mark.parametrize("rng_len,nnz,expected", [
    (10, 6, StrategyKind.MIN_MAX), (12, 6, StrategyKind.SORT), (1, 1, StrategyKind.MIN_MAX)])
def test_combined_select_rule(rng_len, nnz, expected):
    # test_kernels.py:302-313
    assert combined_select(rng_len, nnz) is expected


def test_formats_roundtrip_and_freeze():
    d = np.array([[0.0, 2.0, 0.0], [1.0, 0.0, -3.0]])
    m = CsrMatrix.from_dense(d)
    assert m.row_ptr.tolist() == [0, 1, 3]
    assert m.col_idx.tolist() == [1, 0, 2]
    assert np.array_equal(m.to_dense(), d)
    validate_csr(m)
    with pytest.raises(ValueError):
        m.values[0] = 1.0
    bad = CsrMatrix(1, 3, np.array([0, 2], np.uint64), np.array([2, 1], np.uint64), np.ones(2))
    with pytest.raises(ValueError):
        validate_csr(bad)


def test_result_takes_the_left_operands_class():
    class Other:
        def __init__(self, rows, cols, row_ptr, col_idx, values):
            self.rows, self.cols = rows, cols
            self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values

    z = np.zeros(0, np.uint64)
    r = make_like(Other(1, 1, z, z, z), 1, 1, np.zeros(2, np.uint64), z, np.zeros(0))
    assert isinstance(r, Other)


def test_partition_rows_balances_products():
    rng = np.random.default_rng(0)
    prod = rng.zipf(2.0, size=100_000).clip(1, 4096).astype(np.uint64)
    prefix = np.zeros(prod.size + 1, np.uint64)
    np.cumsum(prod, out=prefix[1:])
    for parts in (1, 2, 3, 8):
        b = partition_rows(prefix, parts)
        assert b[0] == 0 and b[-1] == prod.size and np.all(np.diff(b) >= 0)
        loads = np.diff(prefix[b].astype(np.int64))
        assert loads.sum() == int(prefix[-1])
        assert loads.max() - loads.min() <= 2 * int(prod.max())


def test_partition_rows_edge_cases():
    assert partition_rows(np.array([0], np.uint64), 4).tolist() == [0, 0, 0, 0, 0]
    assert partition_rows(np.array([0, 0, 0], np.uint64), 2).tolist()[-1] == 2
    with pytest.raises(ValueError):
        partition_rows(np.array([0, 1], np.uint64), 0)


def test_row_blocks_concatenate_to_the_full_product():
    """SURVEY.md §4 recommendation 1: C's rows depend only on A's rows, so
    products of A row blocks stack to the full product, byte for byte."""
    a, b, c_ref, _, _ = golden_case("signed_k40")
    prefix = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    bounds = partition_rows(prefix, 5)
    blocks = []
    for g in range(5):
        r = oracle.multiply_rowmajor(row_block_host(a, int(bounds[g]), int(bounds[g + 1])), b)
        blocks.append((r.row_ptr, r.col_idx, r.values))
    c = concat_row_blocks(blocks, b.cols)
    assert c.row_ptr.tobytes() == c_ref.row_ptr.tobytes()
    assert c.col_idx.tobytes() == c_ref.col_idx.tobytes()
    assert c.values.tobytes() == c_ref.values.tobytes()


def test_install_patches_every_reference_name():
    from paper_1303_1651_b200 import install

    pkg = types.ModuleType("fakesparsemm")
    kern = types.ModuleType("fakesparsemm.kernels")
    bench = types.ModuleType("fakesparsemm.bench")
    orig = object()
    for m in (pkg, kern, bench):
        m.multiply_rowmajor = orig
    kern.multiply_colmajor = kern.multiply_mixed = orig
    pkg.multiply_mixed = orig
    sys.modules.update({"fakesparsemm": pkg, "fakesparsemm.kernels": kern,
                        "fakesparsemm.bench": bench})
    from paper_1303_1651_b200 import multiply_colmajor, multiply_mixed
    try:
        with install(pkg):
            assert kern.multiply_rowmajor is multiply_rowmajor
            assert bench.multiply_rowmajor is multiply_rowmajor
            assert pkg.multiply_rowmajor is multiply_rowmajor
            assert kern.multiply_colmajor is multiply_colmajor
            assert kern.multiply_mixed is multiply_mixed and pkg.multiply_mixed is multiply_mixed
            assert not hasattr(bench, "multiply_mixed")
        assert kern.multiply_rowmajor is orig and bench.multiply_rowmajor is orig
        assert kern.multiply_colmajor is orig and kern.multiply_mixed is orig
    finally:
        for n in ("fakesparsemm", "fakesparsemm.kernels", "fakesparsemm.bench"):
            sys.modules.pop(n, None)


def test_stats_defaults():
    s = KernelStats()
    assert s.multiplications == 0 and s.conversions == 0 and s.row_choices == []


def test_perfmodel_numbers():
    # PAPER.md:342-365 / perfmodel tests: 16 B/F; 18.24 GB/s / 16 = 1140 MFlop/s
    assert inner_loop_balance().bytes_per_flop == 16.0
    assert roofline(7.6e9, 18.24e9, 16.0) == pytest.approx(1.14e9)
    assert roofline(3.8e9, 1e12, 16.0) == 3.8e9
    # SURVEY.md §8d bytes_alg table
    assert bytes_alg(10_000, 49_600, 246_408, 128_004) == 11_680_336
    assert bytes_alg(4_194_304, 20_963_328, 104_783_880, 54_484_996) == 4_962_779_472
    assert bytes_alg(2_000_000, 10_000_000, 50_000_000, 49_999_743) == 2_751_995_904
    assert bytes_alg(1_000_000, 26_463_592, 704_969_000, 120_553_784) == 25_350_703_504
