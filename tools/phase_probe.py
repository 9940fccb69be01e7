"""Host/device phase timing of one config (diagnostic; run on the GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1303_1651_b200 import _lib, device as dev
from paper_1303_1651_b200.genmat import config_operands

label = sys.argv[1] if len(sys.argv) > 1 else "C5"
a, b, _ = config_operands(label)
same = a is b
ctx = dev.context_for_current_stream(torch.device("cuda", 0))
ad = dev.DeviceCsr.from_host(a, "cuda")
bd = ad if same else dev.DeviceCsr.from_host(b, "cuda")
for i in range(6):
    if i == 5:
        os.environ["SPMMM_TRACE"] = "1"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = dev.multiply(ctx, ad, bd, _lib.FLAG_TIMING)
    t1 = time.perf_counter()
    print(f"call {i}: host {1e3*(t1-t0):.2f} ms, kernels {ctx.last_timings()}", flush=True)
    p.close()
