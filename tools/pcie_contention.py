"""Does host-memory traffic slow a pinned D2H? D2H alone, then with torch CPU
copies (n threads) running beside it."""
import threading
import time

import torch

n = 512 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src = torch.empty(256 << 20, dtype=torch.uint8)
dst = torch.empty(512 << 20, dtype=torch.uint8)
s = torch.cuda.Stream()


def d2h_ms():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        h.copy_(d, non_blocking=True)
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


print("alone GB/s", n / min(d2h_ms() for _ in range(5)) / 1e6)
for threads in (1, 2, 4, 8):
    torch.set_num_threads(threads)
    stop = False

    def load():
        while not stop:
            dst[: src.numel()].copy_(src)
            dst[src.numel():].copy_(src)

    t = threading.Thread(target=load)
    t.start()
    time.sleep(0.05)
    bw = n / min(d2h_ms() for _ in range(5)) / 1e6
    stop = True
    t.join()
    print(f"with {threads} copy threads GB/s", bw)
