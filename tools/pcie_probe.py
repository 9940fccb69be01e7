"""PCIe probe: pinned H2D alone, D2H alone, and both at once on two streams."""
import json
import torch

n = 512 << 20  # bytes per direction
h_up = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def up():
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)


def down():
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)


def both():
    up()
    down()


t_up, t_dn, t_both = timed(up), timed(down), timed(both)
print(json.dumps({"h2d_GBs": n / t_up / 1e6, "d2h_GBs": n / t_dn / 1e6,
                  "both_ms": t_both, "up_ms": t_up, "down_ms": t_dn,
                  "bidir_GBs": 2 * n / t_both / 1e6}))
