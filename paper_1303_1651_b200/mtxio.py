"""Matrix Market coordinate I/O, native: libspmmm.so's
multi-threaded reader/writer (include/spmmm_mtx.h) behind the reference's
mtxio.py interface (mtxio.py:1-72): `HEADER`, `save_matrix_market(m, path)`,
`load_matrix_market(path) -> CsrMatrix`, the same accepted inputs and the
same ValueError cases and messages. Lets real matrices drive the pipeline:

    a = load_matrix_market("matrix.mtx")
    c = multiply_rowmajor(a, a)
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .formats import INDEX_DTYPE, VALUE_DTYPE, CsrMatrix, csr_arrays

HEADER = "%%MatrixMarket matrix coordinate real general"


def _raise(rc: int, what: str):
    msg = (_lib.lib().spmmm_mtx_last_error() or b"").decode()
    if rc in (1, 2):
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg}")


def save_matrix_market(m, path) -> None:
    """mtxio.py:16-26: header, `rows cols nnz`, 1-based entries in row-major
    order with %.17g values."""
    rp, ci, v = csr_arrays(m)
    view = _lib.csr_view(m.rows, m.cols, rp, ci, v)
    rc = _lib.lib().spmmm_mtx_write(os.fsencode(os.fspath(path)), ctypes.byref(view))
    if rc:
        _raise(rc, "save_matrix_market")


def load_matrix_market(path) -> CsrMatrix:
    """mtxio.py:29-72: any entry order, '%' comments and blank lines skipped;
    ValueError for an unsupported header, a missing/malformed size line, an
    entry outside the shape, a wrong entry count or a duplicate position."""
    open(os.fspath(path), "rb").close()  # the reference's OSError for a missing file
    h = ctypes.c_void_p()
    L = _lib.lib()
    rc = L.spmmm_mtx_read(os.fsencode(os.fspath(path)), ctypes.byref(h))
    if rc:
        _raise(rc, "load_matrix_market")
    try:
        rows, cols, nnz = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        L.spmmm_mtx_shape(h, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(nnz))
        rp = np.empty(rows.value + 1, INDEX_DTYPE)
        ci = np.empty(nnz.value, INDEX_DTYPE)
        v = np.empty(nnz.value, VALUE_DTYPE)
        L.spmmm_mtx_copy(h, rp.ctypes.data, ci.ctypes.data if nnz.value else None,
                         v.ctypes.data if nnz.value else None)
    finally:
        L.spmmm_mtx_free(h)
    return CsrMatrix(rows.value, cols.value, rp, ci, v)
