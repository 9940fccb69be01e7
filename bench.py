"""spMMM benchmark: GFlop/s (2 flops per scalar product) and % of the HBM
roofline of one C = A·B (CSR x CSR, fp64) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one complete product — count pass, (long rows), fused kernel, C
complete in HBM including its allocation — with operands already resident
in HBM in the interface layout (uint64 indices, fp64 values), as in the
reference harness where operand generation sits outside the timed region
(bench.py:181-185; README.md:72-75). Workload: BASELINE.json configs[1]
(the 2D 5-point Laplacian sweep) at its largest point, grid 2048 (N=4.19M),
C = A·A — the largest single-GPU config of that sweep; `--config C1..C5`
selects the other configs.

N > 1 (torchrun, one rank per GPU, NCCL): strong scaling of the same
product — A split into product-balanced row blocks, B broadcast over NVLink
(setup, timed separately), each rank computes its block; the timed region is
the max over ranks (CUDA events, barrier + synchronize on both sides).

--impl reference: the reference's CPU algorithm (oracle/, the C port of
sparsemm.kernels.multiply_rowmajor, byte-identical to it) on all host
threads, on a bounded row-block sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "spMMM GFlop/s (2·products/s) and % of HBM roofline at 1/2/4/8 B200"
UNIT = "GFlop/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profile_traffic(config_label, kernel="k_fused"):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summary of this config (profiles/*.json), or None."""
    pdir = os.path.join(ROOT, "profiles")
    best = None
    if os.path.isdir(pdir):
        for name in sorted(os.listdir(pdir)):
            if not name.endswith(".json"):
                continue
            try:
                with open(os.path.join(pdir, name)) as f:
                    d = json.load(f)
            except Exception:
                continue
            ent = d.get("configs", {}).get(config_label, {}).get(kernel)
            if ent and ent.get("dram_bytes") is not None:
                best = (int(ent["dram_bytes"]), name)
    return best


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, p in zip(names, parts[4:8]):
                if p.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def operands(label, grid=None):
    from paper_1303_1651_b200 import genmat

    override = {"grid": grid} if grid else {}
    a, b, desc = genmat.config_operands(label, **override)
    return a, b, desc


def row_sample(a, b, target_products, prefix=None):
    """Leading row block of A with about `target_products` products."""
    from paper_1303_1651_b200.distributed import row_block_host

    if prefix is None:
        import oracle

        prefix = np.zeros(a.rows + 1, np.uint64)
        np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    r1 = int(np.searchsorted(prefix, np.uint64(target_products), side="left"))
    r1 = max(1, min(a.rows, r1))
    return row_block_host(a, 0, r1), int(prefix[r1]), r1


def cpu_oracle_rate(a, b, threads, budget_s):
    """Time the oracle port on a row-block sample sized to ~budget_s seconds.
    Returns (GFlop/s, sample description)."""
    import oracle

    prefix = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    total = int(prefix[-1])
    # calibrate on ~1/64 of the work
    probe, probe_prod, _ = row_sample(a, b, max(1, total // 64), prefix)
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(probe, b, threads=threads)
    rate = probe_prod / max(time.perf_counter() - t0, 1e-6)
    target = int(min(total, max(probe_prod, rate * budget_s)))
    blk, prods, rows = row_sample(a, b, target, prefix)
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(blk, b, threads=threads)
    dt = time.perf_counter() - t0
    return 2.0 * prods / dt / 1e9, (f"rows [0,{rows}) of A ({rows}/{a.rows} rows, {prods} of "
                                     f"{total} products), one timed call of {dt:.2f} s"), dt


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port), all host
    threads, bounded sample per step; rank 0 only."""
    if rank != 0:
        return 0
    import oracle

    label = args.config
    a, b, desc = operands(label, args.grid)
    threads = len(os.sched_getaffinity(0))
    prefix = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    total = int(prefix[-1])
    probe, probe_prod, _ = row_sample(a, b, max(1, total // 32), prefix)
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(probe, b, threads=threads)
    rate = probe_prod / max(time.perf_counter() - t0, 1e-6)
    per_step_budget = max(0.2, 150.0 / max(1, args.steps + args.warmup))
    blk, prods, rows = row_sample(a, b, int(min(total, rate * per_step_budget)), prefix)
    for _ in range(args.warmup):
        oracle.multiply_rowmajor(blk, b, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.multiply_rowmajor(blk, b, threads=threads)
        times.append(time.perf_counter() - t0)
    sec = float(np.sum(times))
    value = 2.0 * prods * args.steps / sec / 1e9
    sample = (f"rows [0,{rows}) of A ({rows}/{a.rows} rows, {prods}/{total} products) per step; "
              f"oracle/spmmm_oracle.c (C port of sparsemm.kernels.multiply_rowmajor, "
              f"byte-identical to it) on {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sec / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators; see DESIGN.md §4)",
        "config": {"workload": f"{label}: {desc}", "sample": "row block of A, full B"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--grid", type=int, default=None, help="override the stencil grid side")
    ap.add_argument("--e2e-steps", type=int, default=7)
    ap.add_argument("--cpu-budget", type=float, default=8.0,
                    help="seconds of single-thread CPU work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1303_1651_b200 import _lib
    from paper_1303_1651_b200 import device as dev
    from paper_1303_1651_b200.distributed import partition_rows
    from paper_1303_1651_b200.kernels import (PIPELINE_MIN_NNZ, multiply_rowmajor,
                                              row_products_prefix)
    from paper_1303_1651_b200.perfmodel import bytes_alg

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    os.environ.setdefault("SPMMM_DEVICE", str(local_rank))
    distributed = world > 1
    if distributed:
        dist.init_process_group("nccl", device_id=device)

    label = args.config
    a, b, desc = operands(label, args.grid)
    same = b is a
    ctx = dev.context_for_current_stream(device)

    # ---- operands resident in HBM (operand preparation, untimed) ----
    b_bcast_ms = None
    if distributed:
        prefix = row_products_prefix(a, b) if rank == 0 else None
        bounds_t = torch.zeros(world + 1, dtype=torch.int64, device=device)
        if rank == 0:
            bounds_t.copy_(torch.from_numpy(partition_rows(prefix, world)))
        dist.broadcast(bounds_t, 0)
        bounds = [int(x) for x in bounds_t.tolist()]
        # B replicated from rank 0 over NVLink (NCCL broadcast), timed separately
        if rank == 0:
            bd = dev.DeviceCsr.from_host(b, device)
        else:
            bd = dev.DeviceCsr(b.rows, b.cols,
                               torch.empty(b.rows + 1, dtype=torch.int64, device=device),
                               torch.empty(len(b.values), dtype=torch.int64, device=device),
                               torch.empty(len(b.values), dtype=torch.float64, device=device))
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in (bd.row_ptr, bd.col_idx, bd.values):
            dist.broadcast(t, 0)
        e1.record()
        torch.cuda.synchronize()
        b_bcast_ms = e0.elapsed_time(e1)
        from paper_1303_1651_b200.distributed import row_block_host

        ad = dev.DeviceCsr.from_host(row_block_host(a, bounds[rank], bounds[rank + 1]), device)
    else:
        ad = dev.DeviceCsr.from_host(a, device)
        bd = ad if same else dev.DeviceCsr.from_host(b, device)

    va, vb = ad.view(), bd.view()  # (device views built once, not per step)

    def step(flags=_lib.FLAG_TIMING):
        p = _lib.multiply_views(ctx, va, vb, 6, flags)
        info = (p.multiplications, p.nnz, ctx.last_timings(), ctx.last_launch_count())
        p.close()
        return info

    for _ in range(args.warmup):
        step()
    mults_local, nnz_local, _, _ = step()

    # ---- timed region: exactly K steps ----
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = {}
    launches = 0
    with ClockSampler(local_rank) as clk:
        start.record()
        for _ in range(args.steps):
            _, _, t, n = step()
            launches += n
            for k, v in t.items():
                kernel_ms[k] = kernel_ms.get(k, 0.0) + v
        end.record()
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    elapsed_ms = start.elapsed_time(end)
    stats = torch.tensor([elapsed_ms, float(mults_local), float(nnz_local)], dtype=torch.float64,
                         device=device)
    if distributed:
        mx = stats.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        sums = stats.clone()
        dist.all_reduce(sums[1:], op=dist.ReduceOp.SUM)
        elapsed_ms = float(mx[0])
        total_mults, total_nnz = int(sums[1]), int(sums[2])
        kf = torch.tensor([kernel_ms.get("k_fused", 0.0)], dtype=torch.float64, device=device)
        dist.all_reduce(kf, op=dist.ReduceOp.MAX)
        kernel_ms["k_fused"] = float(kf[0])
    else:
        total_mults, total_nnz = mults_local, nnz_local

    ms_per_step = elapsed_ms / args.steps
    flops = 2.0 * total_mults
    value = flops / (ms_per_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel ----
    # k_fused for C1-C4 (it computes every row); in split mode (C5) the
    # expand-sort-compress block kernel, whose units are the products of the
    # rows past kEscWarpLimit (512) — the rows it computes (mid rows whole,
    # huge rows as column-range parts). Bytes per unit: the workload's
    # bytes_alg / products.
    nnz_a = len(a.values)
    balg = bytes_alg(a.rows, nnz_a, total_mults, total_nnz)
    peak, peak_src = hbm_peak()
    per_kernel = {k: round(v / args.steps, 4) for k, v in kernel_ms.items()}
    dom = max(kernel_ms, key=kernel_ms.get) if kernel_ms else "k_fused"
    if dom not in ("k_fused", "k_esc_block"):
        dom = "k_fused"
    kf_ms = kernel_ms.get(dom, 0.0) / args.steps
    units, launch_bytes = total_mults, balg
    if dom == "k_esc_block" and not distributed:
        prefix = row_products_prefix(a, b)
        prod = np.diff(prefix.astype(np.int64))
        units = int(prod[prod > 512].sum())
        launch_bytes = int(round(balg * units / max(total_mults, 1)))
    achieved = launch_bytes / (kf_ms * 1e-3) / 1e9 if kf_ms > 0 else None
    traffic = profile_traffic(label, dom)
    roof = {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
            "peak": peak, "unit": "GB/s",
            "frac": round(achieved / (peak * world), 4) if achieved else None,
            "traffic": traffic[0] if traffic else None,
            "kernel": dom, "bytes_alg_per_launch": launch_bytes,
            "units_per_launch": units, "bytes_per_unit": round(balg / max(total_mults, 1), 2),
            "kernel_ms_per_launch": round(kf_ms, 4),
            "step_frac": round(balg / (ms_per_step * 1e-3) / 1e9 / (peak * world), 4),
            "peak_source": peak_src,
            "traffic_source": traffic[1] if traffic else "no ncu --set full summary committed"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators; see DESIGN.md §4)",
        "config": {"workload": f"{label}: {desc}", "rows": a.rows, "nnz_a": nnz_a,
                   "products": total_mults, "nnz_c": total_nnz,
                   "parallelism": f"row-blocks x{world}" if distributed else "single GPU",
                   "l2": "inputs larger than L2 (no flush)" if 16 * nnz_a > 126e6 else
                         "inputs smaller than L2 (L2-warm)"},
        "kernel_ms": per_kernel,
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if b_bcast_ms is not None:
        line["b_broadcast_ms"] = round(b_bcast_ms, 3)

    # ---- e2e through the public drop-in API (host numpy in -> host numpy out) ----
    if not args.no_e2e and rank == 0 and not distributed:
        import torch as _t

        def pinned(arr):
            buf = _t.empty(max(arr.nbytes, 1), dtype=_t.uint8, pin_memory=True)
            out = buf.numpy()[:arr.nbytes].view(arr.dtype)
            out[...] = arr
            return out

        from paper_1303_1651_b200.formats import CsrMatrix

        ap_ = CsrMatrix(a.rows, a.cols, pinned(a.row_ptr), pinned(a.col_idx), pinned(a.values))
        bp_ = ap_ if same else CsrMatrix(b.rows, b.cols, pinned(b.row_ptr), pinned(b.col_idx),
                                         pinned(b.values))
        # warm: two live results, so the pinned pool holds the blocks a step
        # allocates while the previous step's result is still referenced
        warm = [multiply_rowmajor(ap_, bp_) for _ in range(2)]
        del warm
        multiply_rowmajor(ap_, bp_)  # one more with a single live result, as in the loop
        times = []
        for _ in range(max(1, args.e2e_steps)):
            t0 = time.perf_counter()
            c = multiply_rowmajor(ap_, bp_)
            times.append(time.perf_counter() - t0)
        e2e_s = float(np.median(times))  # host-side noise (page cache, scheduler): median
        h2d = 8 * (a.rows + 1) + 16 * nnz_a
        if not same:
            h2d += 8 * (b.rows + 1) + 16 * len(b.values)
        d2h = 8 * (c.rows + 1) + 16 * len(c.values)
        if _lib.last_transfer is not None and nnz_a >= PIPELINE_MIN_NNZ:
            # the pipelined path moves C's column indices as u32
            h2d = _lib.last_transfer["h2d_bytes"]
            d2h = _lib.last_transfer["d2h_bytes"]
        line["e2e"] = {"value": round(flops / e2e_s / 1e9, 3), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": round(e2e_s * 1e3, 3), "steps": len(times),
                       "stat": "median of the timed calls",
                       "ms_min_mean_max": [round(min(times) * 1e3, 3),
                                           round(float(np.mean(times)) * 1e3, 3),
                                           round(max(times) * 1e3, 3)],
                       "ms_each": [round(t * 1e3, 2) for t in times],
                       "api": "paper_1303_1651_b200.multiply_rowmajor (pinned numpy in, numpy out backed by the pinned pool; block-pipelined spmmm_multiply_host for >= 2^20 A entries)"}

    # ---- CPU baseline: the oracle port, 1 thread, bounded sample ----
    if not args.no_cpu_baseline and rank == 0 and not distributed:
        rate, sample, _ = cpu_oracle_rate(a, b, 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": round(rate, 4), "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
