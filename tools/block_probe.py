"""Device time of one row block product (A rows [r0, r1) of the C2 matrix
times all of B = A), count-free vs counted: python tools/block_probe.py [parts]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200 import device as dev  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 12
a = genmat.gen_fd(2048)
d = torch.device("cuda", 0)
ad = dev.DeviceCsr.from_host(a, d)
ctx = dev.context_for_current_stream(d)
r0, r1 = a.rows // parts * 3, a.rows // parts * 4
va, vb = ad.row_block(r0, r1).view(), ad.view()
for _ in range(5):
    _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING).close()
tot = {}
n = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    p = _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING)
    for k, v in ctx.last_timings().items():
        tot[k] = tot.get(k, 0.0) + v / n
    p.close()
e1.record()
torch.cuda.synchronize()
print(f"block 1/{parts}: {e0.elapsed_time(e1) / n:.4f} ms/product",
      {k: round(v, 4) for k, v in tot.items()})
