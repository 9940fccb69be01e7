"""Per-call e2e times of the drop-in for one config (variance probe)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1303_1651_b200 import genmat  # noqa: E402
from paper_1303_1651_b200.formats import CsrMatrix  # noqa: E402
from paper_1303_1651_b200.kernels import multiply_rowmajor  # noqa: E402


def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype)
    out[...] = arr
    return out


a, b, _ = genmat.config_operands(sys.argv[1])
ap = CsrMatrix(a.rows, a.cols, pinned(a.row_ptr), pinned(a.col_idx), pinned(a.values))
bp = ap if b is a else CsrMatrix(b.rows, b.cols, pinned(b.row_ptr), pinned(b.col_idx),
                                 pinned(b.values))
w = [multiply_rowmajor(ap, bp) for _ in range(2)]
del w
ts = []
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    t = time.perf_counter()
    c = multiply_rowmajor(ap, bp)
    ts.append((time.perf_counter() - t) * 1e3)
print(sys.argv[1], " ".join(f"{x:.1f}" for x in ts))
