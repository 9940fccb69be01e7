"""Seeded operand generators for the BASELINE configs (host C++ in libspmmm.so,
declared in include/spmmm_gen.h).

`gen_fd` and `gen_random_k` are bit-identical to the reference's
sparsemm.genmat.gen_fd / gen_random_k (genmat.py:79-130; pinned by
tests/test_genmat.py against fingerprints the reference produced);
`gen_fd3` (C4) and `gen_zipf` (C5) are new. All run in
native code: the 2M-row configs build in well under a second instead of the
reference's ~27 s per matrix.
"""

from __future__ import annotations

import ctypes
import hashlib

import numpy as np

from . import _lib
from .formats import CsrMatrix


def _rc(rc, what):
    if rc != 0:
        raise ValueError(f"{what}: invalid arguments (status {rc})")


def splitmix64(seed: int, n: int) -> np.ndarray:
    """genmat.py:28-39: the first n outputs of splitmix64(seed)."""
    out = np.empty(n, np.uint64)
    _rc(_lib.lib().spmmm_splitmix64(seed & (2**64 - 1), n, out.ctypes.data), "splitmix64")
    return out


def _sized(size_fn, fill_fn, *args):
    rows, nnz = ctypes.c_uint64(), ctypes.c_uint64()
    _rc(size_fn(*args, ctypes.byref(rows), ctypes.byref(nnz)), "size")
    rp = np.empty(rows.value + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint64)
    v = np.empty(nnz.value, np.float64)
    _rc(fill_fn(*args, rp.ctypes.data, ci.ctypes.data, v.ctypes.data), "fill")
    return CsrMatrix(rows.value, rows.value, rp, ci, v)


def gen_fd(grid: int) -> CsrMatrix:
    """5-point Laplacian on grid x grid (genmat.py:79-103)."""
    lib = _lib.lib()
    return _sized(lib.spmmm_gen_fd_size, lib.spmmm_gen_fd, grid)


def gen_fd3(grid: int) -> CsrMatrix:
    """27-point stencil on grid^3 (config C4): 26 on the diagonal, -1 elsewhere."""
    lib = _lib.lib()
    return _sized(lib.spmmm_gen_fd3_size, lib.spmmm_gen_fd3, grid)


def gen_random_k(n: int, k: int, seed: int) -> CsrMatrix:
    """Exactly k distinct uniform columns per row, values in (0, 1]
    (genmat.py:106-130, one splitmix64 stream, rejected repeats draw no value)."""
    if not 1 <= k <= n:
        raise ValueError("need 1 <= k <= n")
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(n * k, np.uint64)
    v = np.empty(n * k, np.float64)
    _rc(_lib.lib().spmmm_gen_random_k(n, k, seed & (2**64 - 1), rp.ctypes.data, ci.ctypes.data,
                                      v.ctypes.data), "gen_random_k")
    return CsrMatrix(n, n, rp, ci, v)


def gen_zipf(n: int, seed: int, s: float = 2.0, lmax: int = 4096) -> CsrMatrix:
    """Row lengths min(Zipf(s), lmax) by inverse CDF, distinct uniform columns,
    values uniform in [-1, 1) (config C5)."""
    lib = _lib.lib()
    nnz = ctypes.c_uint64()
    _rc(lib.spmmm_gen_zipf(n, s, lmax, seed, ctypes.byref(nnz), None, None, None), "gen_zipf")
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint64)
    v = np.empty(nnz.value, np.float64)
    _rc(lib.spmmm_gen_zipf(n, s, lmax, seed, ctypes.byref(nnz), rp.ctypes.data,
                           ci.ctypes.data, v.ctypes.data), "gen_zipf")
    return CsrMatrix(n, n, rp, ci, v)


def gen_stencil_device(family: str, grid: int, device=None):
    """The fd (5-point) or fd3 (27-point) stencil generated on the GPU
    (spmmm_gen_fd_device / spmmm_gen_fd3_device): the bytes of gen_fd /
    gen_fd3, written straight into HBM. Returns a device.DeviceCsr."""
    import torch

    from .device import DeviceCsr

    lib = _lib.lib()
    size_fn, fill_fn = {"fd": (lib.spmmm_gen_fd_size, lib.spmmm_gen_fd_device),
                        "fd3": (lib.spmmm_gen_fd3_size, lib.spmmm_gen_fd3_device)}[family]
    rows, nnz = ctypes.c_uint64(), ctypes.c_uint64()
    _rc(size_fn(grid, ctypes.byref(rows), ctypes.byref(nnz)), "size")
    device = torch.device(device or "cuda")
    rp = torch.empty(rows.value + 1, dtype=torch.int64, device=device)
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=device)
    v = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    rc = fill_fn(grid, rp.data_ptr(), ci.data_ptr(), v.data_ptr(), stream)
    if rc == 3:
        raise RuntimeError(f"gen_{family}_device: CUDA error")
    _rc(rc, f"gen_{family}_device")
    return DeviceCsr(rows.value, rows.value, rp, ci[:nnz.value], v[:nnz.value])


def matrix_fingerprint(m) -> str:
    """genmat.py:154-165: sha256 over the canonical little-endian bytes."""
    h = hashlib.sha256()
    h.update(f"csr:{m.rows}:{m.cols}:".encode())
    h.update(np.ascontiguousarray(m.row_ptr, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(m.col_idx, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(m.values, dtype="<f8").tobytes())
    return h.hexdigest()


def digests(m) -> dict:
    """Per-array digests (the layout of tests/golden/fingerprints.json)."""
    def h(arr, dt):
        return hashlib.sha256(np.ascontiguousarray(arr, dtype=dt).tobytes()).hexdigest()

    return {
        "rows": int(m.rows), "cols": int(m.cols), "nnz": int(len(m.values)),
        "fingerprint": matrix_fingerprint(m),
        "row_ptr_sha256": h(m.row_ptr, "<u8"),
        "col_idx_sha256": h(m.col_idx, "<u8"),
        "values_sha256": h(m.values, "<f8"),
    }


# BASELINE.json configs (labels as in SURVEY.md)
CONFIGS = {
    "C1": dict(desc="2D 5-pt Laplacian 100x100, C = A*A", family="fd", grid=100),
    "C2": dict(desc="2D 5-pt Laplacian 2048x2048 (top of the 32..2048 sweep), C = A*A",
               family="fd", grid=2048),
    "C3": dict(desc="random N=2,000,000, 5 distinct cols/row, seeds 0/1, C = A*B",
               family="random", n=2_000_000, k=5, seeds=(0, 1)),
    "C4": dict(desc="3D 27-pt stencil 100^3, C = A*A", family="fd3", grid=100),
    "C5": dict(desc="Zipf(2) row lengths clipped to [1,4096], N=2,000,000, seeds 0/1, C = A*B",
               family="zipf", n=2_000_000, seeds=(0, 1)),
}


def config_operands(label: str, **override):
    """(a, b, desc) for a BASELINE config; b is a when the config is A*A."""
    cfg = dict(CONFIGS[label], **override)
    fam = cfg["family"]
    if fam == "fd":
        a = gen_fd(cfg["grid"])
        return a, a, cfg["desc"]
    if fam == "fd3":
        a = gen_fd3(cfg["grid"])
        return a, a, cfg["desc"]
    if fam == "random":
        s0, s1 = cfg["seeds"]
        return gen_random_k(cfg["n"], cfg["k"], s0), gen_random_k(cfg["n"], cfg["k"], s1), cfg["desc"]
    if fam == "zipf":
        s0, s1 = cfg["seeds"]
        return gen_zipf(cfg["n"], s0), gen_zipf(cfg["n"], s1), cfg["desc"]
    raise ValueError(fam)
