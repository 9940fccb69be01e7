"""ctypes binding of libspmmm.so (the C ABI in include/spmmm.h).

The shared library is built in-tree (`paper_1303_1651_b200/libspmmm.so`) by
`build()`; there is no CPU fallback: if the library or a CUDA device is
missing, calls raise RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPMMM_LIB_PATH", os.path.join(HERE, "libspmmm.so"))
CSRC = os.path.join(HERE, "csrc")

# status codes (include/spmmm.h)
OK = 0
ERR_DIMENSION = 1
ERR_INVALID = 2
ERR_CUDA = 3
ERR_NCCL = 4
ERR_OOM = 5
ERR_UNSUPPORTED = 6

MEM_HOST = 0
MEM_DEVICE = 1

FLAG_ROW_STATS = 1
FLAG_TIMING = 2

# every symbol include/spmmm.h and include/spmmm_gen.h declare
EXPORTS = (
    "spmmm_abi_version", "spmmm_last_error", "spmmm_device_count",
    "spmmm_context_create", "spmmm_context_destroy", "spmmm_synchronize",
    "spmmm_multiply", "spmmm_multiply_host", "spmmm_product_shape", "spmmm_product_device_arrays",
    "spmmm_product_reserved_bytes", "spmmm_row_classes",
    "spmmm_product_download", "spmmm_product_copy_device", "spmmm_product_row_stats",
    "spmmm_product_destroy", "spmmm_estimate_nnz", "spmmm_row_products_prefix",
    "spmmm_transpose", "spmmm_partition_rows", "spmmm_product_download_offset",
    "spmmm_host_register", "spmmm_host_unregister",
    "spmmm_last_timings", "spmmm_last_launch_count",
    "spmmm_host_alloc", "spmmm_host_free", "spmmm_host_pool_bytes",
    "spmmm_splitmix64", "spmmm_gen_fd_size", "spmmm_gen_fd", "spmmm_gen_fd3_size",
    "spmmm_gen_fd3", "spmmm_gen_random_k", "spmmm_gen_zipf", "spmmm_gen_fd_device",
    "spmmm_gen_fd3_device",
    "spmmm_mtx_last_error", "spmmm_mtx_write", "spmmm_mtx_read", "spmmm_mtx_shape",
    "spmmm_mtx_copy", "spmmm_mtx_free",
)


class SpmmmHostCsr(ctypes.Structure):
    """spmmm_host_csr (include/spmmm.h): a result in pinned pool memory."""
    _fields_ = [
        ("rows", ctypes.c_uint64),
        ("cols", ctypes.c_uint64),
        ("nnz", ctypes.c_uint64),
        ("mults", ctypes.c_uint64),
        ("row_ptr", ctypes.c_void_p),
        ("col_idx", ctypes.c_void_p),
        ("values", ctypes.c_void_p),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
    ]


class SpmmmCsr(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_uint64),
        ("cols", ctypes.c_uint64),
        ("nnz", ctypes.c_uint64),
        ("row_ptr", ctypes.c_void_p),
        ("col_idx", ctypes.c_void_p),
        ("values", ctypes.c_void_p),
        ("memory", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib = None
_lib_lock = threading.Lock()


def build(verbose: bool = False) -> str:
    """Compile libspmmm.so for sm_100a in place (nvcc; no GPU needed)."""
    cmd = ["make", "-C", CSRC]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def _declare(lib):
    c_u64 = ctypes.c_uint64
    p_u64 = ctypes.POINTER(ctypes.c_uint64)
    vp = ctypes.c_void_p
    pp = ctypes.POINTER(ctypes.c_void_p)
    i = ctypes.c_int
    sig = {
        "spmmm_abi_version": (i, []),
        "spmmm_last_error": (ctypes.c_char_p, []),
        "spmmm_device_count": (i, [ctypes.POINTER(ctypes.c_int)]),
        "spmmm_context_create": (i, [i, vp, pp]),
        "spmmm_context_destroy": (i, [vp]),
        "spmmm_synchronize": (i, [vp]),
        "spmmm_multiply": (i, [vp, ctypes.POINTER(SpmmmCsr), ctypes.POINTER(SpmmmCsr), i,
                               ctypes.c_uint32, pp]),
        "spmmm_product_shape": (i, [vp, p_u64, p_u64, p_u64, p_u64]),
        "spmmm_product_device_arrays": (i, [vp, pp, pp, pp]),
        "spmmm_product_reserved_bytes": (i, [vp, p_u64]),
        "spmmm_row_classes": (i, [ctypes.POINTER(ctypes.c_uint32)]),
        "spmmm_product_download": (i, [vp, vp, vp, vp]),
        "spmmm_multiply_host": (i, [vp, ctypes.POINTER(SpmmmCsr), ctypes.POINTER(SpmmmCsr), i,
                                    ctypes.c_uint32, i, ctypes.POINTER(SpmmmHostCsr)]),
        "spmmm_product_copy_device": (i, [vp, vp, vp, vp]),
        "spmmm_product_row_stats": (i, [vp, vp, vp, vp]),
        "spmmm_product_destroy": (i, [vp]),
        "spmmm_estimate_nnz": (i, [vp, ctypes.POINTER(SpmmmCsr), ctypes.POINTER(SpmmmCsr), p_u64]),
        "spmmm_row_products_prefix": (i, [vp, ctypes.POINTER(SpmmmCsr), ctypes.POINTER(SpmmmCsr),
                                          vp]),
        "spmmm_transpose": (i, [vp, ctypes.POINTER(SpmmmCsr), pp]),
        "spmmm_partition_rows": (i, [vp, ctypes.POINTER(SpmmmCsr), ctypes.POINTER(SpmmmCsr), i,
                                     vp, p_u64]),
        "spmmm_product_download_offset": (i, [vp, c_u64, vp, vp, vp]),
        "spmmm_host_register": (i, [vp, c_u64]),
        "spmmm_host_unregister": (i, [vp]),
        "spmmm_last_timings": (i, [vp, ctypes.POINTER(ctypes.c_char_p),
                                   ctypes.POINTER(ctypes.c_double), i, ctypes.POINTER(i)]),
        "spmmm_last_launch_count": (i, [vp, ctypes.POINTER(i)]),
        "spmmm_host_alloc": (i, [c_u64, pp]),
        "spmmm_host_free": (i, [vp]),
        "spmmm_host_pool_bytes": (i, [p_u64, p_u64]),
        "spmmm_splitmix64": (i, [c_u64, c_u64, vp]),
        "spmmm_gen_fd_size": (i, [c_u64, p_u64, p_u64]),
        "spmmm_gen_fd": (i, [c_u64, vp, vp, vp]),
        "spmmm_gen_fd3_size": (i, [c_u64, p_u64, p_u64]),
        "spmmm_gen_fd3": (i, [c_u64, vp, vp, vp]),
        "spmmm_gen_random_k": (i, [c_u64, c_u64, c_u64, vp, vp, vp]),
        "spmmm_gen_zipf": (i, [c_u64, ctypes.c_double, c_u64, c_u64, p_u64, vp, vp, vp]),
        "spmmm_gen_fd_device": (i, [c_u64, vp, vp, vp, vp]),
        "spmmm_gen_fd3_device": (i, [c_u64, vp, vp, vp, vp]),
        "spmmm_mtx_last_error": (ctypes.c_char_p, []),
        "spmmm_mtx_write": (i, [ctypes.c_char_p, ctypes.POINTER(SpmmmCsr)]),
        "spmmm_mtx_read": (i, [ctypes.c_char_p, pp]),
        "spmmm_mtx_shape": (i, [vp, p_u64, p_u64, p_u64]),
        "spmmm_mtx_copy": (i, [vp, vp, vp, vp]),
        "spmmm_mtx_free": (i, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded library. Raises RuntimeError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import paper_1303_1651_b200 as m; m.build()'`")
            handle = ctypes.CDLL(LIB_PATH)
            _declare(handle)
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().spmmm_last_error()
    return msg.decode() if msg else ""


class OutOfMemory(RuntimeError):
    """SPMMM_ERR_OOM: a device or page-locked host allocation failed."""


def check(rc: int, what: str) -> None:
    """Map a status code to the exception the reference raises."""
    if rc == OK:
        return
    msg = last_error() or f"status {rc}"
    if rc in (ERR_DIMENSION, ERR_INVALID):
        raise ValueError(msg)
    if rc == ERR_OOM:
        raise OutOfMemory(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def csr_view(rows, cols, row_ptr, col_idx, values, memory=MEM_HOST) -> SpmmmCsr:
    """Build a spmmm_csr from numpy arrays (host) or raw device pointers."""
    v = SpmmmCsr()
    v.rows = int(rows)
    v.cols = int(cols)
    if memory == MEM_HOST:
        v.nnz = int(values.size)
        v.row_ptr = row_ptr.ctypes.data
        v.col_idx = col_idx.ctypes.data if col_idx.size else None
        v.values = values.ctypes.data if values.size else None
    else:
        # (row_ptr, col_idx, values) are device addresses; nnz passed in values' slot
        raise TypeError("use device_view() for device memory")
    v.memory = memory
    return v


def device_view(rows, cols, nnz, row_ptr_addr, col_idx_addr, values_addr) -> SpmmmCsr:
    v = SpmmmCsr()
    v.rows = int(rows)
    v.cols = int(cols)
    v.nnz = int(nnz)
    v.row_ptr = int(row_ptr_addr)
    v.col_idx = int(col_idx_addr) if nnz else None
    v.values = int(values_addr) if nnz else None
    v.memory = MEM_DEVICE
    return v


class Context:
    """One CUDA device + stream. `stream` is a raw cudaStream_t (int) or None."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._h = ctypes.c_void_p()
        check(lib().spmmm_context_create(int(device), stream, ctypes.byref(self._h)),
              "spmmm_context_create")
        self.device = device

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().spmmm_context_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(lib().spmmm_synchronize(self._h), "spmmm_synchronize")

    def last_timings(self) -> dict:
        # (buffers kept on the context: this is called once per bench step)
        if not hasattr(self, "_tbuf"):
            self._tbuf = ((ctypes.c_char_p * 16)(), (ctypes.c_double * 16)(), ctypes.c_int(0))
        names, ms, n = self._tbuf
        check(lib().spmmm_last_timings(self._h, names, ms, 16, ctypes.byref(n)), "timings")
        return {names[i].decode(): ms[i] for i in range(min(n.value, 16))}

    def last_launch_count(self) -> int:
        n = ctypes.c_int(0)
        check(lib().spmmm_last_launch_count(self._h, ctypes.byref(n)), "launch count")
        return n.value


def pinned_empty(n: int, dtype) -> np.ndarray:
    """numpy array of n elements in page-locked memory from the library's
    pool; the block returns to the pool when the array (and its views) die."""
    import weakref

    dtype = np.dtype(dtype)
    nbytes = max(int(n) * dtype.itemsize, 1)
    ptr = ctypes.c_void_p()
    check(lib().spmmm_host_alloc(nbytes, ctypes.byref(ptr)), "spmmm_host_alloc")
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    weakref.finalize(buf, lib().spmmm_host_free, ctypes.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dtype, count=int(n))


class Product:
    """Device-resident C returned by spmmm_multiply."""

    _shape = threading.local()

    def __init__(self, ctx: Context, handle: ctypes.c_void_p):
        self.ctx = ctx
        self._h = handle
        # one reusable out-array per thread (this runs once per product)
        vals = getattr(Product._shape, "vals", None)
        if vals is None:
            vals = Product._shape.vals = tuple(ctypes.c_uint64() for _ in range(4))
            Product._shape.ptrs = tuple(ctypes.pointer(x) for x in vals)
        check(lib().spmmm_product_shape(handle, *Product._shape.ptrs), "shape")
        self.rows, self.cols, self.nnz, self.multiplications = (x.value for x in vals)

    def reserved_bytes(self) -> int:
        n = ctypes.c_uint64()
        check(lib().spmmm_product_reserved_bytes(self._h, ctypes.byref(n)), "reserved bytes")
        return int(n.value)

    def download(self, pinned: bool = True):
        alloc = pinned_empty if pinned else np.empty
        rp = alloc(self.rows + 1, np.uint64)
        ci = alloc(self.nnz, np.uint64)
        v = alloc(self.nnz, np.float64)
        check(lib().spmmm_product_download(self._h, rp.ctypes.data,
                                           ci.ctypes.data if self.nnz else None,
                                           v.ctypes.data if self.nnz else None), "download")
        return rp, ci, v

    def device_arrays(self):
        rp, ci, v = (ctypes.c_void_p() for _ in range(3))
        check(lib().spmmm_product_device_arrays(self._h, ctypes.byref(rp), ctypes.byref(ci),
                                                ctypes.byref(v)), "device arrays")
        return rp.value, ci.value, v.value

    def download_offset(self, offset: int, rp_addr, ci_addr, v_addr):
        """Into caller memory at raw addresses, row pointers shifted by
        `offset` (spmmm_product_download_offset)."""
        check(lib().spmmm_product_download_offset(self._h, int(offset), rp_addr,
                                                  ci_addr if self.nnz else None,
                                                  v_addr if self.nnz else None), "download")

    def copy_device(self, rp_addr, ci_addr, v_addr):
        check(lib().spmmm_product_copy_device(self._h, rp_addr, ci_addr, v_addr), "copy")

    def row_stats(self):
        mn = np.empty(self.rows, np.uint64)
        mx = np.empty(self.rows, np.uint64)
        t = np.empty(self.rows, np.uint64)
        check(lib().spmmm_product_row_stats(self._h, mn.ctypes.data, mx.ctypes.data,
                                            t.ctypes.data), "row stats")
        return mn, mx, t

    def close(self):
        if self._h:
            lib().spmmm_product_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def multiply_views(ctx: Context, a: SpmmmCsr, b: SpmmmCsr, strategy_id: int,
                   flags: int = 0) -> Product:
    h = ctypes.c_void_p()
    check(lib().spmmm_multiply(ctx.handle, ctypes.byref(a), ctypes.byref(b), int(strategy_id),
                               int(flags), ctypes.byref(h)), "spmmm_multiply")
    return Product(ctx, h)


def _pool_array(ptr: int, n: int, dtype) -> np.ndarray:
    """numpy view of n elements of a pinned pool block (freed with the array)."""
    import weakref

    dtype = np.dtype(dtype)
    nbytes = max(int(n) * dtype.itemsize, 1)
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    weakref.finalize(buf, lib().spmmm_host_free, ctypes.c_void_p(ptr))
    return np.frombuffer(buf, dtype=dtype, count=int(n))


def multiply_host(ctx: Context, a: SpmmmCsr, b: SpmmmCsr, strategy_id: int, flags: int = 0,
                  blocks: int = 8):
    """spmmm_multiply_host: block-pipelined C = A·B of host operands.
    Returns (row_ptr, col_idx, values, multiplications) as numpy arrays in
    pinned pool memory."""
    out = SpmmmHostCsr()
    check(lib().spmmm_multiply_host(ctx.handle, ctypes.byref(a), ctypes.byref(b),
                                    int(strategy_id), int(flags), int(blocks),
                                    ctypes.byref(out)), "spmmm_multiply_host")
    rp = _pool_array(out.row_ptr, out.rows + 1, np.uint64)
    ci = _pool_array(out.col_idx, out.nnz, np.uint64)
    v = _pool_array(out.values, out.nnz, np.float64)
    global last_transfer
    last_transfer = {"h2d_bytes": int(out.h2d_bytes), "d2h_bytes": int(out.d2h_bytes)}
    return rp, ci, v, int(out.mults)


# PCIe bytes of the last multiply_host call (bench.py's e2e accounting)
last_transfer = None


def partition_rows(ctx: Context, a: SpmmmCsr, b: SpmmmCsr, parts: int):
    """Product-balanced row bounds (parts+1) and the product total, computed on
    the device (spmmm_partition_rows)."""
    bounds = np.zeros(int(parts) + 1, np.uint64)
    total = ctypes.c_uint64()
    check(lib().spmmm_partition_rows(ctx.handle, ctypes.byref(a), ctypes.byref(b), int(parts),
                                     bounds.ctypes.data, ctypes.byref(total)),
          "spmmm_partition_rows")
    return bounds.astype(np.int64), int(total.value)


def host_register(addr: int, nbytes: int) -> None:
    check(lib().spmmm_host_register(ctypes.c_void_p(int(addr)), int(nbytes)), "spmmm_host_register")


def host_unregister(addr: int) -> None:
    check(lib().spmmm_host_unregister(ctypes.c_void_p(int(addr))), "spmmm_host_unregister")


def transpose_view(ctx: Context, m: SpmmmCsr) -> Product:
    """CSR of M^T for the CSR view M (spmmm_transpose): the storage-order
    conversion of formats.py:302-357, on the device."""
    h = ctypes.c_void_p()
    check(lib().spmmm_transpose(ctx.handle, ctypes.byref(m), ctypes.byref(h)), "spmmm_transpose")
    return Product(ctx, h)


def product_view(p: Product) -> SpmmmCsr:
    """Device CSR view of a product's arrays (valid while `p` is open)."""
    rp, ci, v = p.device_arrays()
    return device_view(p.rows, p.cols, p.nnz, rp, ci, v)


_default_ctx = None
_default_lock = threading.Lock()


def default_context() -> Context:
    """Process-wide context on $SPMMM_DEVICE (default 0), created lazily."""
    global _default_ctx
    if _default_ctx is None:
        with _default_lock:
            if _default_ctx is None:
                _default_ctx = Context(int(os.environ.get("SPMMM_DEVICE", "0")))
    return _default_ctx
