"""Matrix Market I/O: the native reader/writer against the
reference's own test cases (pkg/tests/test_mtx_io.py) and, where the
reference package is importable, byte-identical files and results."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from paper_1303_1651_b200.formats import CsrMatrix, validate_csr
from paper_1303_1651_b200.genmat import gen_fd, gen_random_k
from paper_1303_1651_b200.mtxio import HEADER, load_matrix_market, save_matrix_market

REF_SRC = "/root/reference/pkg/src"


def _same(a, b):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    for x, y in ((a.row_ptr, b.row_ptr), (a.col_idx, b.col_idx), (a.values, b.values)):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()


def test_round_trip_bit_identical(tmp_path):
    m = gen_random_k(32, 5, 42)
    save_matrix_market(m, tmp_path / "m.mtx")
    _same(load_matrix_market(tmp_path / "m.mtx"), m)


def test_header_and_one_based_indices(tmp_path):
    m = CsrMatrix.from_dense([[0.0, 1.5], [0.0, 0.0]])
    save_matrix_market(m, tmp_path / "m.mtx")
    lines = (tmp_path / "m.mtx").read_text().splitlines()
    assert lines[0] == HEADER and lines[1] == "2 2 1" and lines[2].split()[:2] == ["1", "2"]


def test_loads_unordered_entries(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text(HEADER + "\n2 3 3\n2 2 5.0\n1 3 2.0\n1 1 1.0\n")
    m = load_matrix_market(p)
    validate_csr(m)
    assert np.array_equal(m.to_dense(), [[1.0, 0.0, 2.0], [0.0, 5.0, 0.0]])


def test_comments_and_blank_lines_ignored(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text(HEADER + "\n% a comment\n\n1 1 1\n% another\n1 1 7.5\n")
    assert load_matrix_market(p).values.tolist() == [7.5]


@pytest.mark.parametrize("body,match", [
    ("\n2 2 2\n1 1 1.0\n1 1 2.0\n", "duplicate entry at row 1, column 1"),
    ("\n2 2 1\n3 1 1.0\n", r"entry \(3, 1\) outside 2 x 2"),
    ("\n2 2 2\n1 1 1.0\n", "size line promises 2 entries, file holds 1"),
    ("\n2 2\n", "malformed size line: '2 2'"),
    ("\n% only comments\n", "missing size line"),
])
def test_rejects_malformed(tmp_path, body, match):
    p = tmp_path / "m.mtx"
    p.write_text(HEADER + body)
    with pytest.raises(ValueError, match=match):
        load_matrix_market(p)


def test_rejects_wrong_header(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 0\n")
    with pytest.raises(ValueError, match="unsupported Matrix Market header"):
        load_matrix_market(p)


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(OSError):
        load_matrix_market(tmp_path / "nope.mtx")


def test_empty_and_stencil_round_trip(tmp_path):
    for m in (CsrMatrix.from_dense(np.zeros((3, 2))), gen_fd(4), gen_fd(100)):
        save_matrix_market(m, tmp_path / "m.mtx")
        _same(load_matrix_market(tmp_path / "m.mtx"), m)


def test_special_values_round_trip(tmp_path):
    v = np.array([np.inf, -np.inf, -0.0, 5e-324, 1.7976931348623157e308, 0.1, -1 / 3])
    m = CsrMatrix(1, v.size, np.array([0, v.size], np.uint64),
                  np.arange(v.size, dtype=np.uint64), v)
    save_matrix_market(m, tmp_path / "m.mtx")
    _same(load_matrix_market(tmp_path / "m.mtx"), m)


def test_large_parallel_paths_round_trip(tmp_path):
    m = gen_random_k(300_000, 7, 3)  # > 1 MiB body and > 65536 rows: threaded paths
    save_matrix_market(m, tmp_path / "m.mtx")
    _same(load_matrix_market(tmp_path / "m.mtx"), m)


def test_files_and_loads_match_reference(tmp_path):
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, REF_SRC)
    try:
        from sparsemm import mtxio as rm
    finally:
        sys.path.remove(REF_SRC)
    m = gen_random_k(2000, 9, 5)
    save_matrix_market(m, tmp_path / "ours.mtx")
    rm.save_matrix_market(m, tmp_path / "ref.mtx")
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()
    # shuffled entries with a comment: both loaders agree bit for bit
    lines = (tmp_path / "ref.mtx").read_text().splitlines()
    body = lines[2:]
    np.random.default_rng(0).shuffle(body)
    (tmp_path / "shuf.mtx").write_text("\n".join(lines[:2] + ["% c"] + body) + "\n")
    _same(load_matrix_market(tmp_path / "shuf.mtx"), rm.load_matrix_market(tmp_path / "shuf.mtx"))
    for bad in ("\n2 2 2\n1 1 1.0\n1 1 2.0\n", "\n2 2 1\n3 1 1.0\n", "\n2 2 2\n1 1 1.0\n",
                "\n2 2\n"):
        (tmp_path / "bad.mtx").write_text(HEADER + bad)
        with pytest.raises(ValueError) as ours:
            load_matrix_market(tmp_path / "bad.mtx")
        with pytest.raises(ValueError) as ref:
            rm.load_matrix_market(tmp_path / "bad.mtx")
        assert str(ours.value) == str(ref.value)
