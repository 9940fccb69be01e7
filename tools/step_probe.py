"""Host-overhead probe of one small product: per-step wall time of
multiply_views + close with and without FLAG_TIMING, the bare C call, and a
traced call. python tools/step_probe.py [grid]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200 import device as dev  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 100
a = genmat.gen_fd(g)
d = torch.device("cuda", 0)
ad = dev.DeviceCsr.from_host(a, d)
ctx = dev.context_for_current_stream(d)
va = ad.view()
L = _lib.lib()


def run(flags, n=2000):
    for _ in range(50):
        _lib.multiply_views(ctx, va, va, 6, flags).close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        _lib.multiply_views(ctx, va, va, 6, flags).close()
    e1.record()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6, e0.elapsed_time(e1) / n * 1e3


def bare(n=2000):
    h = ctypes.c_void_p()
    for _ in range(50):
        L.spmmm_multiply(ctx.handle, ctypes.byref(va), ctypes.byref(va), 6, 0, ctypes.byref(h))
        L.spmmm_product_destroy(h)
    t0 = time.perf_counter()
    for _ in range(n):
        L.spmmm_multiply(ctx.handle, ctypes.byref(va), ctypes.byref(va), 6, 0, ctypes.byref(h))
        L.spmmm_product_destroy(h)
    return (time.perf_counter() - t0) / n * 1e6


print(f"grid {g}: no timing  host {run(0)[0]:.1f} us/step")
print(f"grid {g}: timing     host/event {run(_lib.FLAG_TIMING)} us/step")
print(f"grid {g}: bare C ABI host {bare():.1f} us/step")
os.environ["SPMMM_TRACE"] = "1"
