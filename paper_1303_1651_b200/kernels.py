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
from .formats import csr_arrays, make_like


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


def _record_row_choices(stats, product: _lib.Product, enum_cls, a_row_ptr) -> None:
    if product.cols == 0:
        # With zero result columns the accumulator's sentinels coincide
        # (min_idx = length = 0 = max_idx, kernels.py:82-83), so the reference
        # records combined_select(1, 0) = SORT for every non-empty A row
        # (kernels.py:255-258) although nothing was touched.
        rows = np.nonzero(np.diff(a_row_ptr.astype(np.int64)))[0]
        stats.row_choices.extend((int(r), enum_cls.SORT) for r in rows.tolist())
        return
    mn, mx, touched = product.row_stats()
    rows = np.nonzero(touched)[0]
    if rows.size == 0:
        return
    span = (mx[rows] - mn[rows] + np.uint64(1)).astype(np.uint64)
    use_minmax = span < np.uint64(2) * touched[rows]
    mm, so = enum_cls.MIN_MAX, enum_cls.SORT
    stats.row_choices.extend(
        (int(r), mm if m else so) for r, m in zip(rows.tolist(), use_minmax.tolist()))


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
