"""CSR storage for the drop-in: the same layout and invariants as the
reference's `sparsemm.formats.CsrMatrix` (formats.py:15-16, 40-91).

`row_ptr` (uint64, rows+1), `col_idx` (uint64, nnz) and `values` (float64,
nnz), strictly increasing columns per row, arrays frozen on construction
(formats.py:35-37, 55-58). `multiply_rowmajor` accepts any object with
`rows, cols, row_ptr, col_idx, values` (the reference's own CsrMatrix
included) and returns an instance of the left operand's class when that
class has this constructor signature, so the result drops into reference
code unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

INDEX_DTYPE = np.uint64
VALUE_DTYPE = np.float64


def _frozen(arr: np.ndarray) -> np.ndarray:
    arr.flags.writeable = False
    return arr


@dataclass(eq=False)
class CsrMatrix:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        _frozen(self.row_ptr)
        _frozen(self.col_idx)
        _frozen(self.values)

    @property
    def nnz(self) -> int:
        return len(self.values)

    @classmethod
    def from_arrays(cls, rows, cols, row_ptr, col_idx, values) -> "CsrMatrix":
        return cls(int(rows), int(cols),
                   np.asarray(row_ptr, dtype=INDEX_DTYPE).copy(),
                   np.asarray(col_idx, dtype=INDEX_DTYPE).copy(),
                   np.asarray(values, dtype=VALUE_DTYPE).copy())

    @classmethod
    def from_dense(cls, dense) -> "CsrMatrix":
        dense = np.asarray(dense, dtype=VALUE_DTYPE)
        rows, cols = dense.shape
        mask = dense != 0.0
        r, c = np.nonzero(mask)
        row_ptr = np.zeros(rows + 1, INDEX_DTYPE)
        np.cumsum(mask.sum(axis=1), out=row_ptr[1:])
        return cls(rows, cols, row_ptr, c.astype(INDEX_DTYPE), dense[r, c].astype(VALUE_DTYPE))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), dtype=VALUE_DTYPE)
        if self.nnz:
            per_row = np.diff(self.row_ptr).astype(np.intp)
            r = np.repeat(np.arange(self.rows), per_row)
            out[r, self.col_idx.astype(np.intp)] = self.values
        return out


@dataclass(eq=False)
class CscMatrix:
    """Column-major mirror of CsrMatrix (formats.py:94-140): `col_ptr`
    (uint64, cols+1), `row_idx` (uint64, nnz), `values` (float64, nnz),
    strictly increasing rows per column, arrays frozen on construction."""

    rows: int
    cols: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        _frozen(self.col_ptr)
        _frozen(self.row_idx)
        _frozen(self.values)

    @property
    def nnz(self) -> int:
        return len(self.values)

    @classmethod
    def from_arrays(cls, rows, cols, col_ptr, row_idx, values) -> "CscMatrix":
        return cls(int(rows), int(cols),
                   np.asarray(col_ptr, dtype=INDEX_DTYPE).copy(),
                   np.asarray(row_idx, dtype=INDEX_DTYPE).copy(),
                   np.asarray(values, dtype=VALUE_DTYPE).copy())

    @classmethod
    def from_dense(cls, dense) -> "CscMatrix":
        dense = np.asarray(dense, dtype=VALUE_DTYPE)
        t = CsrMatrix.from_dense(dense.T)
        return cls(dense.shape[0], dense.shape[1], t.row_ptr, t.col_idx, t.values)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), dtype=VALUE_DTYPE)
        if self.nnz:
            per_col = np.diff(self.col_ptr).astype(np.intp)
            c = np.repeat(np.arange(self.cols), per_col)
            out[self.row_idx.astype(np.intp), c] = self.values
        return out


def is_csr(m) -> bool:
    """Row-major operand: anything with `row_ptr` (the reference's CsrMatrix,
    ours, or a compatible class); column-major: anything with `col_ptr`."""
    return hasattr(m, "row_ptr")


def csc_arrays(m):
    """(col_ptr, row_idx, values) of any CSC-like object, contiguous."""
    return (np.ascontiguousarray(m.col_ptr, dtype=INDEX_DTYPE),
            np.ascontiguousarray(m.row_idx, dtype=INDEX_DTYPE),
            np.ascontiguousarray(m.values, dtype=VALUE_DTYPE))


def _transpose_arrays(n_major, n_minor, ptr, idx, val):
    """Device transpose of the compressed (ptr, idx, val) structure with
    n_major slices over n_minor indices: the arrays of the other storage
    order, minor indices ascending within each new slice (spmmm_transpose)."""
    from . import _lib
    ctx = _lib.default_context()
    view = _lib.csr_view(n_major, n_minor, ptr, idx, val)
    with _lib.transpose_view(ctx, view) as p:
        return p.download()


def csr_to_csc(a):
    """formats.py:302-329 on the GPU (stable: rows ascend within each column)."""
    rp, ci, v = csr_arrays(a)
    cp, ri, vv = _transpose_arrays(a.rows, a.cols, rp, ci, v)
    return CscMatrix(a.rows, a.cols, cp, ri, vv)


def csc_to_csr(a):
    """formats.py:332-357 on the GPU (the mirror of csr_to_csc)."""
    cp, ri, v = csc_arrays(a)
    rp, ci, vv = _transpose_arrays(a.cols, a.rows, cp, ri, v)
    return CsrMatrix(a.rows, a.cols, rp, ci, vv)


def csr_arrays(m):
    """(row_ptr, col_idx, values) of any CSR-like object as contiguous
    uint64/uint64/float64 arrays (no copy when already in that layout)."""
    return (np.ascontiguousarray(m.row_ptr, dtype=INDEX_DTYPE),
            np.ascontiguousarray(m.col_idx, dtype=INDEX_DTYPE),
            np.ascontiguousarray(m.values, dtype=VALUE_DTYPE))


def make_like(template, rows, cols, row_ptr, col_idx, values):
    """Construct the result with the left operand's CSR class when possible."""
    cls = type(template)
    try:
        return cls(rows, cols, row_ptr, col_idx, values)
    except TypeError:
        return CsrMatrix(rows, cols, row_ptr, col_idx, values)


def validate_csr(m) -> None:
    """Vectorised check of the CsrMatrix invariants (formats.py:231-273)."""
    rp, ci, v = m.row_ptr, m.col_idx, m.values
    if rp.dtype != INDEX_DTYPE or ci.dtype != INDEX_DTYPE:
        raise ValueError("index arrays must be 64-bit unsigned integers")
    if v.dtype != VALUE_DTYPE:
        raise ValueError("values must be IEEE-754 doubles")
    if len(rp) != m.rows + 1:
        raise ValueError(f"pointer array has length {len(rp)}, expected {m.rows + 1}")
    if rp[0] != 0:
        raise ValueError("pointer array must start at 0")
    if len(ci) != len(v):
        raise ValueError("index and value arrays differ in length")
    if int(rp[-1]) != len(ci):
        raise ValueError(f"pointer array ends at {int(rp[-1])} but {len(ci)} entries are stored")
    d = np.diff(rp.astype(np.int64))
    if np.any(d < 0):
        raise ValueError("pointer array decreases")
    if len(ci):
        if int(ci.max()) >= m.cols:
            raise ValueError("column index out of range")
        same_row = np.repeat(np.arange(m.rows), d)
        inc = np.diff(ci.astype(np.int64))
        if np.any((inc <= 0) & (same_row[1:] == same_row[:-1])):
            raise ValueError("columns not strictly increasing within a row")
