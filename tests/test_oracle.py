"""Pin the CPU oracle (oracle/spmmm_oracle.c) to the reference package:
every golden case the reference computed (tests/golden/make_golden.py) must
come out byte-identical, with the same multiplication count and the same
per-row Combined choices. Full-size configs are pinned through the
reference's sha256 fingerprints."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import (assert_csr_bitwise_equal, fingerprints, golden_case, golden_names)
from paper_1303_1651_b200.formats import CsrMatrix, validate_csr


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_golden(name):
    a, b, c_ref, mults, choices = golden_case(name)
    got = oracle.multiply_rowmajor(a, b, row_choices=True)
    c = CsrMatrix(got.rows, got.cols, got.row_ptr, got.col_idx, got.values)
    assert_csr_bitwise_equal(c, c_ref, name)
    assert got.multiplications == mults
    assert np.array_equal(got.row_choices, choices), name
    assert oracle.estimate_nnz(a, b) == mults
    validate_csr(c)


def test_known_answers():
    # test_kernels.py:41-47, :113-120, :122-130
    a, b, c, _, _ = golden_case("hand_2x2")
    assert np.array_equal(oracle.multiply_rowmajor(a, b).values, [7.0, 2.0, 3.0, 1.0])
    a, b, c, _, _ = golden_case("cancellation")
    r = oracle.multiply_rowmajor(a, b)
    assert r.col_idx.tolist() == [1] and r.values.tolist() == [2.0]
    a, b, c, _, _ = golden_case("transient_zero")
    r = oracle.multiply_rowmajor(a, b, row_choices=True)
    assert r.col_idx.tolist() == [0] and r.values.tolist() == [3.0]


def test_dense_oracle_agrees_on_small_cases():
    for name in ("hand_2x2", "fd_4", "random_3", "signed_dense_rows", "rect_7x13_13x5"):
        a, b, c, mults, _ = golden_case(name)
        dense, dm = oracle.dense_multiply(a.to_dense(), b.to_dense())
        got = c.to_dense()
        assert np.array_equal(got != 0.0, dense != 0.0), name
        assert np.allclose(got, dense, rtol=1e-12, atol=0.0), name
        assert dm == mults


def test_threaded_oracle_is_byte_identical():
    for name in ("signed_k40", "long_rows", "medium_rows", "fd_16", "random_7"):
        a, b, _, _, _ = golden_case(name)
        one = oracle.multiply_rowmajor(a, b)
        many = oracle.multiply_rowmajor(a, b, threads=4)
        assert one.row_ptr.tobytes() == many.row_ptr.tobytes()
        assert one.col_idx.tobytes() == many.col_idx.tobytes()
        assert one.values.tobytes() == many.values.tobytes()


def test_row_products_sum_to_estimate():
    a, b, _, mults, _ = golden_case("long_rows")
    rp = oracle.row_products(a, b)
    assert int(rp.sum()) == mults


def test_dimension_mismatch():
    a, b, _, _, _ = golden_case("rect_7x13_13x5")
    with pytest.raises(ValueError):
        oracle.multiply_rowmajor(b, b)


def _digest_match(m, ref):
    from paper_1303_1651_b200.genmat import digests  # pure hashlib/numpy

    d = digests(m)
    return all(d[k] == ref[k] for k in ("nnz", "row_ptr_sha256", "col_idx_sha256",
                                        "values_sha256", "fingerprint"))


FULL = ["C1_fd100", "C2_fd256", "C2_fd1024", "C2_fd2048", "C3_random2M", "C4_fd3_100",
        "C5_zipf2M"]


@pytest.mark.slow
@pytest.mark.parametrize("label", FULL)
def test_oracle_full_size_fingerprints(label):
    """The oracle reproduces the reference's full-size products byte for byte
    (operands from the native generators, themselves pinned in test_genmat)."""
    fp = fingerprints().get(label)
    if fp is None:
        pytest.skip(f"{label} not in tests/golden/fingerprints.json")
    pytest.importorskip("ctypes")
    from paper_1303_1651_b200 import genmat

    try:
        genmat._lib.lib()
    except RuntimeError as e:
        pytest.skip(str(e))
    if label.startswith("C1"):
        a = b = genmat.gen_fd(100)
    elif label.startswith("C2"):
        a = b = genmat.gen_fd(int(label[len("C2_fd"):]))
    elif label.startswith("C3"):
        a, b = genmat.gen_random_k(2_000_000, 5, 0), genmat.gen_random_k(2_000_000, 5, 1)
    elif label.startswith("C4"):
        a = b = genmat.gen_fd3(100)
    else:
        a, b = genmat.gen_zipf(2_000_000, 0), genmat.gen_zipf(2_000_000, 1)
    assert _digest_match(a, fp["a"]), "operand A differs from the reference's"
    assert _digest_match(b, fp["b"]), "operand B differs from the reference's"
    r = oracle.multiply_rowmajor(a, b, threads=8)
    c = CsrMatrix(r.rows, r.cols, r.row_ptr, r.col_idx, r.values)
    assert r.multiplications == fp["multiplications"]
    assert _digest_match(c, fp["c"]), f"oracle product differs from the reference on {label}"
