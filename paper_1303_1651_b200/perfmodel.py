"""Flop and traffic model of the spMMM hot path (measurement side).

* flops = 2 * multiplications, multiplications = Σ_k nnz(col k of A) *
  nnz(row k of B) (perfmodel.py:63-76), computed on the GPU
  by the count pass.
* Inner-loop code balance: 3 loads + 1 store of 8 B per 2 flops = 16 B/F
  (perfmodel.py:102-109).
* `bytes_alg` extends that per-product term with the compulsory A, pointer and
  C traffic: it is the byte count the roofline fraction in
  bench.py divides by the kernel time.
"""

from __future__ import annotations

from dataclasses import dataclass

from .kernels import estimate_nnz


@dataclass(frozen=True)
class FlopCount:
    multiplications: int

    @property
    def flops(self) -> int:
        return 2 * self.multiplications


@dataclass(frozen=True)
class InnerLoopTraffic:
    loads: int
    stores: int
    bytes_per_value: int
    flops: int

    @property
    def bytes_per_iteration(self) -> int:
        return (self.loads + self.stores) * self.bytes_per_value

    @property
    def bytes_per_flop(self) -> float:
        return self.bytes_per_iteration / self.flops


def inner_loop_balance() -> InnerLoopTraffic:
    """perfmodel.py:102-109: idx LD + value LD + temp LD + temp ST, 8 B each."""
    return InnerLoopTraffic(loads=3, stores=1, bytes_per_value=8, flops=2)


def count_mults(a, b) -> FlopCount:
    """perfmodel.py:63-76 (numerically equal to estimate_nnz)."""
    return FlopCount(estimate_nnz(a, b))


def roofline(peak_flops: float, bandwidth: float, code_balance: float) -> float:
    """perfmodel.py:95-99: min(peak, bandwidth / code balance)."""
    if peak_flops <= 0 or bandwidth <= 0 or code_balance <= 0:
        raise ValueError("all roofline parameters must be strictly positive")
    return min(peak_flops, bandwidth / code_balance)


def bytes_alg(rows_a: int, nnz_a: int, products: int, nnz_c: int) -> int:
    """Algorithmic bytes of one C = A·B:

    read A (row_ptr, col_idx, values)          8(N+1) + 16 nnz(A)
    B.row_ptr[k], B.row_ptr[k+1] per A entry   16 nnz(A)
    referenced B entries (index + value)       16 products
    accumulator load + store                   16 products
    write C                                    8(N+1) + 16 nnz(C)
    """
    return (8 * (rows_a + 1) + 16 * nnz_a + 16 * nnz_a + 16 * products + 16 * products
            + 8 * (rows_a + 1) + 16 * nnz_c)


def compulsory_bytes(rows_a: int, nnz_a: int, nnz_b: int, rows_b: int, nnz_c: int) -> int:
    """DRAM bytes if every array is touched exactly once (no accumulator
    traffic, every B row fetched once): the floor ncu traffic is compared to."""
    return (8 * (rows_a + 1) + 16 * nnz_a + 8 * (rows_b + 1) + 16 * nnz_b
            + 8 * (rows_a + 1) + 16 * nnz_c)
