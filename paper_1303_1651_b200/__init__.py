"""B200-native CSR x CSR spMMM: a drop-in for the reference package's
row-major product `sparsemm.kernels.multiply_rowmajor` (arXiv 1303.1651's
Gustavson kernel), running as hand-written sm_100a CUDA in libspmmm.so.

Public surface (mirrors the reference's names for this path):
    multiply_rowmajor, StrategyKind, KernelStats, combined_select,
    CsrMatrix, estimate_nnz, count_mults, install
and the storage-order neighbours:
    multiply_colmajor, multiply_mixed, estimate_nnz_csc, CscMatrix,
    csr_to_csc, csc_to_csr
Matrix Market I/O (native): load_matrix_market, save_matrix_market
"""

from ._lib import build as _build_lib
from .formats import (INDEX_DTYPE, VALUE_DTYPE, CscMatrix, CsrMatrix, csc_to_csr, csr_to_csc,
                      validate_csr)
from .install import install
from .mtxio import load_matrix_market, save_matrix_market
from .kernels import (
    KernelStats,
    StrategyKind,
    combined_select,
    estimate_nnz,
    estimate_nnz_csc,
    multiply_colmajor,
    multiply_mixed,
    multiply_rowmajor,
    row_products_prefix,
)
from .perfmodel import FlopCount, bytes_alg, count_mults, inner_loop_balance, roofline

__version__ = "0.1.0"


def build(verbose: bool = False) -> str:
    """Compile libspmmm.so (sm_100a) in place; returns its path."""
    return _build_lib(verbose)


__all__ = [
    "CscMatrix", "csc_to_csr", "csr_to_csc", "estimate_nnz_csc", "multiply_colmajor",
    "multiply_mixed", "CsrMatrix", "load_matrix_market", "save_matrix_market", "FlopCount", "INDEX_DTYPE", "KernelStats", "StrategyKind", "VALUE_DTYPE",
    "build", "bytes_alg", "combined_select", "count_mults", "estimate_nnz",
    "inner_loop_balance", "install", "multiply_rowmajor", "roofline", "row_products_prefix",
    "validate_csr",
]
