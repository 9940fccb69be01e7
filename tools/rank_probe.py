"""Per-rank work of the strong-scaling run, emulated on one GPU: for G ranks,
time the product of each rank's A row block (product-balanced) with the full
B, device-resident, CUDA events over K steps. Speed-up = T(1) / max_g T(g)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1303_1651_b200 import _lib, device as dev
from paper_1303_1651_b200.distributed import partition_rows, row_block_host
from paper_1303_1651_b200.genmat import config_operands
from paper_1303_1651_b200.kernels import row_products_prefix

label = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = 50
a, b, _ = config_operands(label)
d = torch.device("cuda", 0)
ctx = dev.context_for_current_stream(d)
bd = dev.DeviceCsr.from_host(b, d)
prefix = row_products_prefix(a, b)
base = None
for G in (1, 2, 4, 8):
    bounds = partition_rows(prefix, G)
    worst = 0.0
    for g in range(G):
        ad = dev.DeviceCsr.from_host(row_block_host(a, int(bounds[g]), int(bounds[g + 1])), d)
        for _ in range(3):
            dev.multiply(ctx, ad, bd).close()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            p = dev.multiply(ctx, ad, bd)
            _ = p.nnz
            p.close()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        worst = max(worst, ms)
        if g == 0:
            p = dev.multiply(ctx, ad, bd, _lib.FLAG_TIMING)
            t = ctx.last_timings()
            p.close()
    if base is None:
        base = worst
    print(f"{label} G={G}: worst rank {worst:.3f} ms/step, speed-up {base / worst:.2f}, "
          f"rank0 kernels {dict((k, round(v, 3)) for k, v in t.items())}", flush=True)
