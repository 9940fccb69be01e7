"""Device-resident operands for benchmarking and the multi-GPU driver.

PyTorch is only plumbing here: it owns device memory and streams
(torch.distributed moves tensors between ranks); the product itself runs in
libspmmm.so on device pointers taken from the tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .formats import csr_arrays


@dataclass
class DeviceCsr:
    rows: int
    cols: int
    row_ptr: torch.Tensor  # int64 view of uint64 data, rows+1 (row_ptr[0] may be != 0)
    col_idx: torch.Tensor
    values: torch.Tensor   # float64

    @property
    def nnz(self) -> int:
        return int(self.values.numel())

    @classmethod
    def from_host(cls, m, device) -> "DeviceCsr":
        rp, ci, v = csr_arrays(m)
        return cls(int(m.rows), int(m.cols),
                   torch.from_numpy(rp.view(np.int64)).to(device),
                   torch.from_numpy(ci.view(np.int64)).to(device),
                   torch.from_numpy(v).to(device))

    def view(self) -> _lib.SpmmmCsr:
        return _lib.device_view(self.rows, self.cols, self.nnz, self.row_ptr.data_ptr(),
                                self.col_idx.data_ptr(), self.values.data_ptr())

    def row_block(self, r0: int, r1: int) -> "DeviceCsr":
        """Rows [r0, r1) as a zero-copy view (row_ptr offset, shared arrays)."""
        return DeviceCsr(r1 - r0, self.cols, self.row_ptr[r0:r1 + 1], self.col_idx, self.values)

    def to_host(self):
        from .formats import CsrMatrix

        rp = self.row_ptr.cpu().numpy().view(np.uint64).copy()
        base = rp[0]
        rp -= base
        lo, hi = int(base), int(base + rp[-1])
        return CsrMatrix(self.rows, self.cols, rp,
                         self.col_idx[lo:hi].cpu().numpy().view(np.uint64).copy(),
                         self.values[lo:hi].cpu().numpy().copy())


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream's handle


def context_for_current_stream(device: torch.device) -> _lib.Context:
    """A libspmmm context bound to torch's current stream on `device`, so the
    library's kernels are ordered with torch's copies and collectives. torch's
    default stream has handle 0, which the C ABI reads as "make your own
    stream" (one that does not wait for the default stream), so it is passed
    as cudaStreamLegacy instead."""
    stream = torch.cuda.current_stream(device)
    handle = stream.cuda_stream or _CUDA_STREAM_LEGACY
    return _lib.Context(device.index if device.index is not None else 0, handle)


def multiply(ctx: _lib.Context, a: DeviceCsr, b: DeviceCsr, flags: int = 0,
             strategy_id: int = 6) -> _lib.Product:
    return _lib.multiply_views(ctx, a.view(), b.view(), strategy_id, flags)


def product_tensors(product: _lib.Product, device) -> DeviceCsr:
    """Copy C out of the library's buffers into fresh torch tensors."""
    rp = torch.empty(product.rows + 1, dtype=torch.int64, device=device)
    ci = torch.empty(product.nnz, dtype=torch.int64, device=device)
    v = torch.empty(product.nnz, dtype=torch.float64, device=device)
    product.copy_device(rp.data_ptr(), ci.data_ptr() if product.nnz else None,
                        v.data_ptr() if product.nnz else None)
    return DeviceCsr(product.rows, product.cols, rp, ci, v)
