"""The drop-in row-major spMMM: `multiply_rowmajor(a, b, strategy, stats)`.

Mirrors `sparsemm.kernels.multiply_rowmajor` (kernels.py:302-332): same
signature, same CSR result, same errors, same `KernelStats` side effects. The
product runs on the B200 through libspmmm.so (ctypes releases the GIL for
the call). There is no CPU fallback: without the library or a GPU the call
raises RuntimeError.

Semantics reproduced exactly:
* C[r, x] = left fold over the A-row entries k in ascending column order of
  fl(A[r,k] * B[k,x]), separately rounded multiply and add (kernels.py:167-174);
* an entry is emitted iff that sum != 0.0 — exact cancellations vanish
  (kernels.py:296-298); columns strictly ascending; empty rows stay empty.
* every StrategyKind yields the same bytes (kernels.py:1-17): the argument is
  validated (ValueError for unknown values, kernels.py:77) and recorded;
* stats.multiplications += Σ products (kernels.py:330-331);
  stats.row_choices gets (r, combined_select(max-min+1, len(touched))) for
  every row that touched a column (kernels.py:255-258) — the GPU reports the
  touched range and the touched-list length, re-touches after a transient
  exact zero included (test_kernels.py:122-130).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .formats import CscMatrix, CsrMatrix, csc_arrays, csr_arrays, is_csr, make_like


class StrategyKind(str, Enum):
    """kernels.py:38-47 (same values; compares equal to the reference's)."""

    BRUTE_FORCE_DOUBLE = "bfdouble"
    BRUTE_FORCE_BOOL = "bfbool"
    BRUTE_FORCE_CHAR = "bfchar"
    MIN_MAX = "minmax"
    MIN_MAX_CHAR = "minmaxchar"
    SORT = "sort"
    COMBINED = "combined"


_STRATEGY_IDS = {s.value: i for i, s in enumerate(StrategyKind)}

# multiply_rowmajor without stats on operands of at least this many A entries
# takes the block-pipelined host path (spmmm_multiply_host), in row blocks of
# about PIPELINE_BLOCK_NNZ A entries (2..12 blocks). Below it the per-block
# fixed costs outweigh the overlap (tools/pipe_threshold.py, C2 sweep points,
# pinned operands: 1.3M entries one-shot 1.59 ms vs pipelined >= 1.59; 2.6M
# entries one-shot 3.09 vs 5 blocks 2.70; 5.2M entries 6.07 vs 10 blocks 4.68).
PIPELINE_MIN_NNZ = 1 << 21
PIPELINE_BLOCK_NNZ = 1 << 19


def pipeline_blocks(nnz_a: int) -> int:
    return max(2, min(12, nnz_a // PIPELINE_BLOCK_NNZ))


@dataclass
class KernelStats:
    """kernels.py:57-63."""

    multiplications: int = 0
    conversions: int = 0
    row_choices: list = field(default_factory=list)


def combined_select(range_len: int, row_nnz: int):
    """kernels.py:186-191: MinMax iff the touched range is smaller than twice
    the row's touched count."""
    return StrategyKind.MIN_MAX if range_len < 2 * row_nnz else StrategyKind.SORT


def _strategy_id(strategy) -> int:
    value = strategy.value if isinstance(strategy, Enum) else strategy
    if value not in _STRATEGY_IDS:
        raise ValueError(f"{strategy!r} is not a valid StrategyKind")
    return _STRATEGY_IDS[value]


def _choice_enum(strategy):
    """Row choices are reported with the caller's StrategyKind class (the
    reference's, once installed) so identity checks keep working."""
    cls = type(strategy)
    if isinstance(strategy, Enum) and hasattr(cls, "MIN_MAX") and hasattr(cls, "SORT"):
        return cls
    return StrategyKind


def choices_from_row_stats(row_stats, cols: int, a_row_ptr, row0: int = 0):
    """[(row + row0, is_minmax)] for every row that touched a column: the
    reference's combined_select(max - min + 1, len(touched)) per row
    (kernels.py:186-191, 255-258), from the GPU's per-row stats."""
    if cols == 0:
        # With zero result columns the accumulator's sentinels coincide
        # (min_idx = length = 0 = max_idx, kernels.py:82-83), so the reference
        # records combined_select(1, 0) = SORT for every non-empty A row
        # (kernels.py:255-258) although nothing was touched.
        rows = np.nonzero(np.diff(np.asarray(a_row_ptr).astype(np.int64)))[0]
        return [(int(r) + row0, False) for r in rows.tolist()]
    mn, mx, touched = row_stats
    rows = np.nonzero(touched)[0]
    if rows.size == 0:
        return []
    span = (mx[rows] - mn[rows] + np.uint64(1)).astype(np.uint64)
    use_minmax = span < np.uint64(2) * touched[rows]
    return list(zip((rows + row0).tolist(), use_minmax.tolist()))


def _record_row_choices(stats, product: _lib.Product, enum_cls, a_row_ptr) -> None:
    row_stats = product.row_stats() if product.cols else None
    mm, so = enum_cls.MIN_MAX, enum_cls.SORT
    stats.row_choices.extend(
        (r, mm if m else so) for r, m in choices_from_row_stats(row_stats, product.cols, a_row_ptr))


def multiply_rowmajor(a, b, strategy=StrategyKind.COMBINED, stats=None):
    """Row-major product of two CSR matrices on the GPU (kernels.py:302-332)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    sid = _strategy_id(strategy)
    arp, aci, av = csr_arrays(a)
    if b is a:
        brp, bci, bv = arp, aci, av
    else:
        brp, bci, bv = csr_arrays(b)
    va = _lib.csr_view(a.rows, a.cols, arp, aci, av)
    vb = _lib.csr_view(b.rows, b.cols, brp, bci, bv)
    flags = _lib.FLAG_ROW_STATS if stats is not None else 0
    ctx = _lib.default_context()
    if stats is None and len(av) >= PIPELINE_MIN_NNZ:
        # large host operands: uploads, kernels and downloads overlap in row
        # blocks (spmmm_multiply_host); the same bytes as the path below.
        # Its result reservation is page-locked host memory (8 nnz(A)
        # entries); if that cannot be had, the one-shot path below runs.
        try:
            rp, ci, v, _ = _lib.multiply_host(ctx, va, vb, sid, 0, pipeline_blocks(len(av)))
            return make_like(a, a.rows, b.cols, rp, ci, v)
        except _lib.OutOfMemory:
            pass
    with _lib.multiply_views(ctx, va, vb, sid, flags) as product:
        rp, ci, v = product.download()
        if stats is not None:
            stats.multiplications += product.multiplications
            _record_row_choices(stats, product, _choice_enum(strategy), arp)
    return make_like(a, a.rows, b.cols, rp, ci, v)


def estimate_nnz(a, b) -> int:
    """formats.py:276-289 on the GPU (the count pass): Σ over A nonzeros of the
    nonzero count of the matching B row; an upper bound of nnz(A·B)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    import ctypes

    arp, aci, av = csr_arrays(a)
    brp, bci, bv = csr_arrays(b)
    out = ctypes.c_uint64()
    ctx = _lib.default_context()
    _lib.check(_lib.lib().spmmm_estimate_nnz(
        ctx.handle, ctypes.byref(_lib.csr_view(a.rows, a.cols, arp, aci, av)),
        ctypes.byref(_lib.csr_view(b.rows, b.cols, brp, bci, bv)), ctypes.byref(out)),
        "spmmm_estimate_nnz")
    return int(out.value)


def row_products_prefix(a, b) -> np.ndarray:
    """Inclusive prefix (rows+1, leading 0) of per-row product counts — the
    input of product-balanced row partitioning (distributed.partition_rows)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    arp, aci, av = csr_arrays(a)
    brp, bci, bv = csr_arrays(b)
    out = np.zeros(a.rows + 1, np.uint64)
    import ctypes

    ctx = _lib.default_context()
    _lib.check(_lib.lib().spmmm_row_products_prefix(
        ctx.handle, ctypes.byref(_lib.csr_view(a.rows, a.cols, arp, aci, av)),
        ctypes.byref(_lib.csr_view(b.rows, b.cols, brp, bci, bv)), out.ctypes.data),
        "spmmm_row_products_prefix")
    return out


# ---------------------------------------------------------------------------
# Column-major and mixed storage orders.
#
# A CSC matrix's arrays are the CSR arrays of its transpose, and
# multiply_colmajor(A, B) (kernels.py:335-363) accumulates, for each column c
# of B, column k of A scaled by b[k, c] over B's column entries in ascending k
# order — exactly the row-major product Bᵀ·Aᵀ on the same arrays, with the
# same fold order per output entry and the same products (fp multiplication
# commutes). So the column-major product is the row-major kernel on zero-copy
# transposed views, bit for bit, with stats recorded per result column.


def _dim_check(a, b):
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")


def estimate_nnz_csc(a, b) -> int:
    """formats.py:292-299: Σ over B's entries of the nonzero count of the
    matching A column (the count pass on the transposed views)."""
    _dim_check(a, b)
    if b.nnz == 0:
        return 0
    import ctypes

    bp, bi, bv = csc_arrays(b)
    ap, ai, av = csc_arrays(a)
    out = ctypes.c_uint64()
    ctx = _lib.default_context()
    _lib.check(_lib.lib().spmmm_estimate_nnz(
        ctx.handle, ctypes.byref(_lib.csr_view(b.cols, b.rows, bp, bi, bv)),
        ctypes.byref(_lib.csr_view(a.cols, a.rows, ap, ai, av)), ctypes.byref(out)),
        "spmmm_estimate_nnz")
    return int(out.value)


def _colmajor_views(ctx, a_view, b_view, a, b, strategy, stats, b_major_ptr):
    sid = _strategy_id(strategy)
    flags = _lib.FLAG_ROW_STATS if stats is not None else 0
    # C^T = B^T · A^T: left operand = B's CSC arrays, right = A's
    with _lib.multiply_views(ctx, b_view, a_view, sid, flags) as product:
        cp, ri, v = product.download()
        if stats is not None:
            stats.multiplications += product.multiplications
            _record_row_choices(stats, product, _choice_enum(strategy), b_major_ptr)
    return make_like(a, a.rows, b.cols, cp, ri, v)


def multiply_colmajor(a, b, strategy=StrategyKind.COMBINED, stats=None):
    """Column-major mirror of multiply_rowmajor for two CSC matrices
    (kernels.py:335-363), on the GPU; returns the left operand's CSC class."""
    _dim_check(a, b)
    ap, ai, av = csc_arrays(a)
    if b is a:
        bp, bi, bv = ap, ai, av
    else:
        bp, bi, bv = csc_arrays(b)
    ctx = _lib.default_context()
    a_view = _lib.csr_view(a.cols, a.rows, ap, ai, av)
    b_view = _lib.csr_view(b.cols, b.rows, bp, bi, bv)
    return _colmajor_views(ctx, a_view, b_view, a, b, strategy, stats, bp)


def multiply_mixed(a, b, strategy=StrategyKind.COMBINED, stats=None):
    """kernels.py:417-438: same-order pairs go to the matching kernel; for a
    mixed pair the right operand is converted once (stats.conversions += 1),
    on the device, and feeds the kernel without a host round trip. The result
    is in the left operand's storage order."""
    a_csr, b_csr = is_csr(a), is_csr(b)
    if a_csr and b_csr:
        return multiply_rowmajor(a, b, strategy, stats)
    if not a_csr and not b_csr:
        return multiply_colmajor(a, b, strategy, stats)
    _dim_check(a, b)
    if stats is not None:
        stats.conversions += 1
    ctx = _lib.default_context()
    if a_csr:
        # B (CSC) -> CSR on the device: its CSC arrays are the CSR of B^T
        bp, bi, bv = csc_arrays(b)
        with _lib.transpose_view(ctx, _lib.csr_view(b.cols, b.rows, bp, bi, bv)) as b_rm:
            arp, aci, av = csr_arrays(a)
            sid = _strategy_id(strategy)
            flags = _lib.FLAG_ROW_STATS if stats is not None else 0
            with _lib.multiply_views(ctx, _lib.csr_view(a.rows, a.cols, arp, aci, av),
                                     _lib.product_view(b_rm), sid, flags) as product:
                rp, ci, v = product.download()
                if stats is not None:
                    stats.multiplications += product.multiplications
                    _record_row_choices(stats, product, _choice_enum(strategy), arp)
        return make_like(a, a.rows, b.cols, rp, ci, v)
    # A (CSC) with B (CSR): B -> CSC on the device (= the CSR of B^T), then
    # the column-major product on the views
    brp, bci, bv = csr_arrays(b)
    with _lib.transpose_view(ctx, _lib.csr_view(b.rows, b.cols, brp, bci, bv)) as b_cm:
        ap, ai, av = csc_arrays(a)
        a_view = _lib.csr_view(a.cols, a.rows, ap, ai, av)
        # (B's column pointers matter only for the zero-row quirk of stats)
        b_major_ptr = b_cm.download()[0] if stats is not None and a.rows == 0 else None
        return _colmajor_views(ctx, a_view, _lib.product_view(b_cm), a, b, strategy, stats,
                               b_major_ptr)
