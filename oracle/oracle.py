"""ctypes front end of the CPU oracle (oracle/spmmm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
CPU baseline, never as the measured product. The product package
(paper_1303_1651_b200) does not import this module.

Every function takes plain numpy CSR triples (uint64 row_ptr, uint64 col_idx,
float64 values) so it can check the CUDA library and the reference package
alike. See spmmm_oracle.c for the reference file:line each routine restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)
_i8p = ctypes.POINTER(ctypes.c_int8)


def build() -> str:
    """Compile liboracle.so in place (gcc; a few seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.oracle_estimate_nnz.restype = ctypes.c_uint64
    lib.oracle_estimate_nnz.argtypes = [ctypes.c_uint64, _u64p, _u64p, _u64p]
    lib.oracle_count_mults.restype = ctypes.c_uint64
    lib.oracle_count_mults.argtypes = [ctypes.c_uint64, _u64p, _u64p, _u64p]
    lib.oracle_row_products.restype = None
    lib.oracle_row_products.argtypes = [ctypes.c_uint64, _u64p, _u64p, _u64p, _u64p]
    lib.oracle_multiply_rowmajor.restype = ctypes.c_int
    lib.oracle_multiply_rowmajor.argtypes = (
        [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p, _f64p]
        + [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p, _f64p]
        + [_u64p, _u64p, _f64p, ctypes.c_uint64, _i8p, _u64p, _u64p]
    )
    lib.oracle_multiply_rowmajor_mt.restype = ctypes.c_int
    lib.oracle_multiply_rowmajor_mt.argtypes = (
        [ctypes.c_int]
        + [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p, _f64p]
        + [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p, _f64p]
        + [_u64p, _u64p, _f64p, ctypes.c_uint64, _u64p]
    )
    _lib = lib
    return lib


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


def _arrays(m):
    rp = np.ascontiguousarray(m.row_ptr, dtype=np.uint64)
    ci = np.ascontiguousarray(m.col_idx, dtype=np.uint64)
    v = np.ascontiguousarray(m.values, dtype=np.float64)
    if ci.size == 0:
        ci = np.zeros(1, np.uint64)
        v = np.zeros(1, np.float64)
    return rp, ci, v


@dataclass
class OracleResult:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    multiplications: int
    row_choices: np.ndarray | None  # int8 per row: -1 none, 0 MinMax, 1 Sort

    @property
    def nnz(self) -> int:
        return int(self.values.size)


def estimate_nnz(a, b) -> int:
    """formats.py:276-289."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    lib = _load()
    arp, aci, _ = _arrays(a)
    brp, _, _ = _arrays(b)
    return int(lib.oracle_estimate_nnz(a.rows, _p(arp, _u64p), _p(aci, _u64p), _p(brp, _u64p)))


def row_products(a, b) -> np.ndarray:
    lib = _load()
    arp, aci, _ = _arrays(a)
    brp, _, _ = _arrays(b)
    out = np.zeros(a.rows, np.uint64)
    lib.oracle_row_products(a.rows, _p(arp, _u64p), _p(aci, _u64p), _p(brp, _u64p),
                            _p(out, _u64p))
    return out


def multiply_rowmajor(a, b, *, row_choices: bool = False, threads: int = 1) -> OracleResult:
    """kernels.py:302-332 with StrategyKind.COMBINED (all strategies are
    bit-identical by the reference's contract, kernels.py:1-17)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    lib = _load()
    arp, aci, av = _arrays(a)
    brp, bci, bv = _arrays(b)
    cap = estimate_nnz(a, b)
    out_rp = np.zeros(a.rows + 1, np.uint64)
    out_ci = np.empty(max(cap, 1), np.uint64)
    out_v = np.empty(max(cap, 1), np.float64)
    nnz = ctypes.c_uint64(0)
    mults = ctypes.c_uint64(0)
    choice = None
    if threads > 1 and not row_choices:
        rc = lib.oracle_multiply_rowmajor_mt(
            threads, a.rows, a.cols, _p(arp, _u64p), _p(aci, _u64p), _p(av, _f64p),
            b.rows, b.cols, _p(brp, _u64p), _p(bci, _u64p), _p(bv, _f64p),
            _p(out_rp, _u64p), _p(out_ci, _u64p), _p(out_v, _f64p), cap, ctypes.byref(nnz))
        mults.value = cap
    else:
        choice = np.full(a.rows, -1, np.int8) if row_choices else None
        rc = lib.oracle_multiply_rowmajor(
            a.rows, a.cols, _p(arp, _u64p), _p(aci, _u64p), _p(av, _f64p),
            b.rows, b.cols, _p(brp, _u64p), _p(bci, _u64p), _p(bv, _f64p),
            _p(out_rp, _u64p), _p(out_ci, _u64p), _p(out_v, _f64p), cap,
            _p(choice, _i8p) if choice is not None else None,
            ctypes.byref(nnz), ctypes.byref(mults))
    if rc != 0:
        raise RuntimeError(f"oracle failed with status {rc}")
    n = int(nnz.value)
    # views into the capacity-sized buffers, as the reference's own
    # CsrBuilder.finish() returns (formats.py:189-196); untouched pages of the
    # reservation are never faulted in
    return OracleResult(a.rows, b.cols, out_rp, out_ci[:n], out_v[:n],
                        int(mults.value), choice)


def dense_multiply(a_dense, b_dense):
    """kernels.py:441-457: triple loop, k ascending, returns (C, mults)."""
    a = np.asarray(a_dense, dtype=np.float64)
    b = np.asarray(b_dense, dtype=np.float64)
    if a.shape[1] != b.shape[0]:
        raise ValueError("dimension mismatch")
    out = np.zeros((a.shape[0], b.shape[1]), np.float64)
    for k in range(a.shape[1]):
        # rank-1 update per k, ascending: every C entry is a left fold over k
        # of separately rounded products
        out += np.multiply.outer(a[:, k], b[k, :])
    mults = int(np.count_nonzero(a, axis=0) @ np.count_nonzero(b, axis=1))
    return out, mults


# ---------------------------------------------------------------------------
# Storage orders (kernels.py:335-363, 417-438; formats.py:292-357).


@dataclass
class _Csr:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.size)


def transpose(n_major, n_minor, ptr, idx, val):
    """formats.py:302-329 (csr_to_csc) / 332-357 (csc_to_csr): count per minor
    index, prefix sum, then a stable scatter of the entries in major order.
    Returns (ptr, idx, val) of the other storage order (n_minor slices)."""
    ptr = np.asarray(ptr, np.uint64)
    idx = np.asarray(idx, np.uint64)
    val = np.asarray(val, np.float64)
    counts = np.bincount(idx.astype(np.intp), minlength=n_minor)
    out_ptr = np.zeros(n_minor + 1, np.uint64)
    np.cumsum(counts, out=out_ptr[1:])
    # stable order by minor index == the reference's scatter in major order
    order = np.argsort(idx, kind="stable")
    major_of = np.repeat(np.arange(n_major, dtype=np.uint64), np.diff(ptr).astype(np.intp))
    return out_ptr, major_of[order], val[order]


def multiply_colmajor(a_csc, b_csc, *, row_choices: bool = False) -> OracleResult:
    """kernels.py:335-363: for each column c of B, its entries b[k, c] in
    ascending k scale column k of A into the accumulator. That is the
    row-major kernel with B's columns as the 'rows' and A's columns as the
    scaled slices — kernels.py:344-357 calls the same accumulate with the
    roles swapped — so it runs on the CSR views of Bᵀ and Aᵀ. Returns the CSC
    arrays of C (as row_ptr/col_idx of Cᵀ) and per-column choices."""
    if a_csc.cols != b_csc.rows:
        raise ValueError(f"dimension mismatch: {a_csc.cols} (cols of a) != {b_csc.rows} (rows of b)")
    bt = _Csr(b_csc.cols, b_csc.rows, b_csc.col_ptr, b_csc.row_idx, b_csc.values)
    at = _Csr(a_csc.cols, a_csc.rows, a_csc.col_ptr, a_csc.row_idx, a_csc.values)
    return multiply_rowmajor(bt, at, row_choices=row_choices)


# ---------------------------------------------------------------------------
# Operand generators (gen_oracle.c): the reference arm of bench.py builds its
# operands here, so it never maps the product library.

# BASELINE.json configs (labels and wording as SURVEY.md §8(d))
CONFIGS = {
    "C1": dict(family="fd", grid=100, desc="2D 5-pt Laplacian 100x100, C = A*A"),
    "C2": dict(family="fd", grid=2048,
               desc="2D 5-pt Laplacian sweep 32..2048 (grid {grid}x{grid}), C = A*A"),
    "C3": dict(family="random", n=2_000_000, k=5, seeds=(0, 1),
               desc="random 5 per row, N=2M, C = A*B"),
    "C4": dict(family="fd3", grid=100, desc="3D 27-pt stencil 100^3, C = A*A"),
    "C5": dict(family="zipf", n=2_000_000, seeds=(0, 1),
               desc="Zipf(2) rows clipped to [1,4096], N=2M, C = A*B"),
}


def _gen_lib():
    lib = _load()
    if not getattr(lib, "_gen_declared", False):
        vp = ctypes.c_void_p
        u64 = ctypes.c_uint64
        lib.oracle_splitmix64.argtypes = [u64, u64, vp]
        lib.oracle_gen_fd_size.argtypes = [u64, _u64p, _u64p]
        lib.oracle_gen_fd.argtypes = [u64, vp, vp, vp]
        lib.oracle_gen_fd3_size.argtypes = [u64, _u64p, _u64p]
        lib.oracle_gen_fd3.argtypes = [u64, vp, vp, vp]
        lib.oracle_gen_random_k.argtypes = [u64, u64, u64, vp, vp, vp]
        lib.oracle_gen_zipf.argtypes = [u64, u64, u64, _u64p, vp, vp, vp]
        for f in (lib.oracle_splitmix64, lib.oracle_gen_fd, lib.oracle_gen_fd3,
                  lib.oracle_gen_random_k, lib.oracle_gen_zipf):
            f.restype = ctypes.c_int
        lib._gen_declared = True
    return lib


def splitmix64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _gen_lib().oracle_splitmix64(seed & (2**64 - 1), n, out.ctypes.data)
    return out


def _stencil(size_fn, fill_fn, grid):
    rows, nnz = ctypes.c_uint64(), ctypes.c_uint64()
    size_fn(grid, ctypes.byref(rows), ctypes.byref(nnz))
    rp = np.empty(rows.value + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint64)
    v = np.empty(nnz.value, np.float64)
    fill_fn(grid, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    return _Csr(rows.value, rows.value, rp, ci, v)


def gen_fd(grid: int):
    lib = _gen_lib()
    return _stencil(lib.oracle_gen_fd_size, lib.oracle_gen_fd, grid)


def gen_fd3(grid: int):
    lib = _gen_lib()
    return _stencil(lib.oracle_gen_fd3_size, lib.oracle_gen_fd3, grid)


def gen_random_k(n: int, k: int, seed: int):
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(n * k, np.uint64)
    v = np.empty(n * k, np.float64)
    if _gen_lib().oracle_gen_random_k(n, k, seed, rp.ctypes.data, ci.ctypes.data, v.ctypes.data):
        raise ValueError("need 1 <= k <= n")
    return _Csr(n, n, rp, ci, v)


def gen_zipf(n: int, seed: int, lmax: int = 4096):
    lib = _gen_lib()
    nnz = ctypes.c_uint64()
    lib.oracle_gen_zipf(n, lmax, seed, ctypes.byref(nnz), None, None, None)
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint64)
    v = np.empty(nnz.value, np.float64)
    lib.oracle_gen_zipf(n, lmax, seed, ctypes.byref(nnz), rp.ctypes.data, ci.ctypes.data,
                        v.ctypes.data)
    return _Csr(n, n, rp, ci, v)


def config_operands(label: str, grid: int | None = None):
    """(a, b, desc) of a BASELINE config; b is a for the A*A configs."""
    cfg = dict(CONFIGS[label])
    if grid:
        cfg["grid"] = grid
    fam = cfg["family"]
    desc = cfg["desc"].format(**cfg)
    if fam == "fd":
        a = gen_fd(cfg["grid"])
        return a, a, desc
    if fam == "fd3":
        a = gen_fd3(cfg["grid"])
        return a, a, desc
    s0, s1 = cfg["seeds"]
    if fam == "random":
        return gen_random_k(cfg["n"], cfg["k"], s0), gen_random_k(cfg["n"], cfg["k"], s1), desc
    return gen_zipf(cfg["n"], s0), gen_zipf(cfg["n"], s1), desc
