"""Break the drop-in's end-to-end time into upload+compute / download / wrap."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1303_1651_b200 import _lib, genmat
from paper_1303_1651_b200.formats import csr_arrays

label = sys.argv[1] if len(sys.argv) > 1 else "C2"
a, b, _ = genmat.config_operands(label)

def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype)
    out[...] = arr
    return out

for mode in ("pageable-in", "pinned-in"):
    if mode == "pinned-in":
        arrs = [pinned(x) for x in csr_arrays(a)]
    else:
        arrs = list(csr_arrays(a))
    va = _lib.csr_view(a.rows, a.cols, *arrs)
    vb = va if b is a else _lib.csr_view(b.rows, b.cols, *[pinned(x) if mode == "pinned-in" else x for x in csr_arrays(b)])
    ctx = _lib.default_context()
    for it in range(4):
        t0 = time.perf_counter()
        p = _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING)
        t1 = time.perf_counter()
        rp, ci, v = p.download(pinned=True)
        t2 = time.perf_counter()
        rp2, ci2, v2 = p.download(pinned=False)
        t3 = time.perf_counter()
        p.close()
        print(f"{label} {mode} it{it}: multiply {1e3*(t1-t0):.1f} ms (kernels {ctx.last_timings()}), "
              f"download pinned {1e3*(t2-t1):.1f} ms, pageable {1e3*(t3-t2):.1f} ms, nnz {len(v)}", flush=True)
