import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1303_1651_b200 import _lib, genmat
from paper_1303_1651_b200.formats import csr_arrays
a = genmat.gen_fd(2048)
def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype); out[...] = arr; return out
rp, ci, v = (pinned(x) for x in csr_arrays(a))
ctx = _lib.Context(0)
va = _lib.csr_view(a.rows, a.cols, rp, ci, v)
for i in range(4):
    t0 = time.perf_counter(); r = _lib.multiply_host(ctx, va, va, 6, 0, 12); t1 = time.perf_counter()
    print("call", i, round((t1-t0)*1e3, 2), file=sys.stderr)
    del r
