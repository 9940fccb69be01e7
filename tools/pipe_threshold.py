"""e2e of the drop-in at C2 sweep points, one-shot vs pipelined (2..8 blocks):
where the pipelined host path should start. python tools/pipe_threshold.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200.formats import csr_arrays  # noqa: E402


def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype)
    out[...] = arr
    return out


ctx = _lib.Context(0)
for g in (256, 362, 512, 724, 1024):
    a = genmat.gen_fd(g)
    rp, ci, v = (pinned(x) for x in csr_arrays(a))
    va = _lib.csr_view(a.rows, a.cols, rp, ci, v)
    res = {}

    def one_shot():
        with _lib.multiply_views(ctx, va, va, 6, 0) as p:
            p.download()

    def piped(nb):
        return lambda: _lib.multiply_host(ctx, va, va, 6, 0, nb)

    for name, fn in [("one-shot", one_shot)] + [(f"pipe{nb}", piped(nb)) for nb in (2, 3, 4, 6, 8)]:
        for _ in range(3):
            fn()
        t = []
        for _ in range(9):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        res[name] = round(1e3 * float(np.median(t)), 3)
    print(g, len(v), res, flush=True)
