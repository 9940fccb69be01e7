"""spMMM benchmark: GFlop/s (2 flops per scalar product) and % of the HBM
roofline of one C = A·B (CSR x CSR, fp64) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--grid G]
                    [--impl ours|reference]

A step is one complete product — count pass, (long rows), fused kernel, C
complete in HBM including its allocation — with operands already resident
in HBM in the interface layout (uint64 indices, fp64 values), as in the
reference harness where operand generation sits outside the timed region
(bench.py:181-185; README.md:72-75). Workload: BASELINE.json configs[1]
(the 2D 5-point Laplacian sweep) at its largest point, grid 2048 (N=4.19M),
C = A·A — the largest single-GPU config of that sweep; `--config C1..C5`
selects the other configs, `--grid` another point of the sweep.

e2e: the same product through the public drop-in (`multiply_rowmajor`,
host numpy in, host numpy out) with the host->device copies of the inputs
and the device->host copy of C inside the timed region: from pinned host
memory (`e2e`) and from ordinary pageable numpy arrays (`e2e_pageable`).

N > 1 (`--gpus N`: re-launched under torch.distributed.run unless already
running under it; one rank per GPU, NCCL): strong scaling of the same product
by product-balanced row blocks (paper_1303_1651_b200.distributed). Plan
(untimed): operands in node-wide shared memory, each rank uploads 1/N and
NCCL all-gathers the rest over NVLink (`b_allgather_ms`), the device
partition. Timed (`value`): every rank's block product, max over ranks (CUDA
events, barrier + synchronize on both sides). `e2e`: the whole
multiply_distributed call from shared host operands to the shared host
result, max over ranks; `gather_ms`: its download phase.

--impl reference: the reference's CPU algorithm (oracle/: the C port of
sparsemm.kernels.multiply_rowmajor, byte-identical to it) on all host
threads, on a bounded row-block sample of the same workload, operands built
by oracle/gen_oracle.c — the product library is never loaded; rank 0 only.
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
DATA = "synthetic (seeded generators; see DESIGN.md §4)"

WORKLOADS = {
    "C1": ("2D 5-pt Laplacian 100x100, C = A*A", None),
    "C2": ("2D 5-pt Laplacian {g}x{g} (BASELINE configs[1]: the 32..2048 sweep), C = A*A", 2048),
    "C3": ("random N=2,000,000, 5 distinct cols/row, seeds 0/1, C = A*B", None),
    "C4": ("3D 27-pt stencil 100^3, C = A*A", None),
    "C5": ("Zipf(2) row lengths clipped to [1,4096], N=2,000,000, seeds 0/1, C = A*B", None),
}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def workload_config(label, grid, a, b, products):
    """The `config` dict — identical in both arms for the same workload."""
    desc, default_grid = WORKLOADS[label]
    g = grid or default_grid
    cfg = {"workload": f"{label}: {desc.format(g=g)}", "rows": int(a.rows),
           "nnz_a": int(len(a.values)), "nnz_b": int(len(b.values)), "products": int(products)}
    if g:
        cfg["grid"] = int(g)
    return cfg


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profile_traffic(config_label, kernel="k_fused"):
    """DRAM bytes per launch of `kernel` from the newest committed ncu
    --set full summary of this config (profiles/*_traffic.json), or None."""
    pdir = os.path.join(ROOT, "profiles")
    best = None
    if os.path.isdir(pdir):
        for name in sorted(os.listdir(pdir)):
            if not name.endswith("_traffic.json"):
                continue
            try:
                with open(os.path.join(pdir, name)) as f:
                    d = json.load(f)
            except Exception:
                continue
            ent = d.get("configs", {}).get(config_label, {}).get(kernel)
            if ent and ent.get("dram_bytes") is not None:
                best = (int(ent["dram_bytes"]), name, ent.get("duration_ms"))
    return best


def native_libs_mapped():
    """Shared objects of this repo mapped into the process (evidence of
    which native code ran)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                path = ln.split()[-1] if ln.strip() else ""
                if path.startswith(ROOT) and ".so" in path:
                    libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

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


def merge_clocks(summaries):
    sm = [s["sm_mhz"] for s in summaries if s.get("sm_mhz") is not None]
    mx = [s["sm_max_mhz"] for s in summaries if s.get("sm_max_mhz") is not None]
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted({r for s in summaries for r in s.get("reasons", [])}),
            "samples": int(sum(s.get("samples", 0) for s in summaries)),
            "ranks": len(summaries)}


# ---------------------------------------------------------------------------
# CPU legs (the oracle: reference algorithm, C port)


def _prefix(a, b):
    import oracle

    prefix = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    return prefix


def _row_sample(a, target_products, prefix):
    """Leading row block of A with about `target_products` products (the
    row-block view the oracle computes; rows are independent)."""
    from types import SimpleNamespace

    r1 = int(np.searchsorted(prefix, np.uint64(target_products), side="left"))
    r1 = max(1, min(a.rows, r1))
    rp = np.asarray(a.row_ptr)
    lo, hi = int(rp[0]), int(rp[r1])
    blk = SimpleNamespace(rows=r1, cols=a.cols, row_ptr=(rp[:r1 + 1] - rp[0]).astype(np.uint64),
                          col_idx=np.asarray(a.col_idx)[lo:hi], values=np.asarray(a.values)[lo:hi])
    return blk, int(prefix[r1]), r1


def cpu_oracle_rate(a, b, threads, budget_s, prefix=None):
    """The oracle port on a row-block sample sized to ~budget_s seconds.
    Returns (GFlop/s, sample description, seconds)."""
    import oracle

    prefix = _prefix(a, b) if prefix is None else prefix
    total = int(prefix[-1])
    probe, probe_prod, _ = _row_sample(a, max(1, total // 64), prefix)  # calibrate on ~1/64
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(probe, b, threads=threads)
    rate = probe_prod / max(time.perf_counter() - t0, 1e-6)
    target = int(min(total, max(probe_prod, rate * budget_s)))
    blk, prods, rows = _row_sample(a, target, prefix)
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(blk, b, threads=threads)
    dt = time.perf_counter() - t0
    return 2.0 * prods / dt / 1e9, (f"rows [0,{rows}) of A ({rows}/{a.rows} rows, {prods} of "
                                     f"{total} products), one timed call of {dt:.2f} s"), dt


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port), all host
    threads, bounded sample per step; rank 0 only. Operands from
    oracle/gen_oracle.c: the product library is not loaded."""
    if rank != 0:
        return 0
    import oracle

    label = args.config
    a, b, _ = oracle.config_operands(label, args.grid)
    threads = len(os.sched_getaffinity(0))
    prefix = _prefix(a, b)
    total = int(prefix[-1])
    probe, probe_prod, _ = _row_sample(a, max(1, total // 32), prefix)
    t0 = time.perf_counter()
    oracle.multiply_rowmajor(probe, b, threads=threads)
    rate = probe_prod / max(time.perf_counter() - t0, 1e-6)
    per_step_budget = max(0.2, 150.0 / max(1, args.steps + args.warmup))
    blk, prods, rows = _row_sample(a, int(min(total, rate * per_step_budget)), prefix)
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
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(label, args.grid, a, b, total),
        "parallelism": f"{threads} host threads (row blocks)",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_libs_mapped": native_libs_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# roofline of the dominant kernel


def roofline_entry(label, kernel_ms_per_launch, dom, balg, units, total_mults, nnz_c_total,
                   rows, nnz_a, nnz_b, rows_b, ms_per_step, world):
    from paper_1303_1651_b200.perfmodel import compulsory_bytes

    peak, peak_src = hbm_peak()
    kf_ms = kernel_ms_per_launch
    launch_bytes = int(round(balg * units / max(total_mults, 1)))
    achieved = launch_bytes / (kf_ms * 1e-3) / 1e9 if kf_ms > 0 else None
    traffic = profile_traffic(label, dom) if world == 1 else None
    flops = 2.0 * total_mults
    comp = compulsory_bytes(rows, nnz_a, nnz_b, rows_b, nnz_c_total)
    roof_alg = flops / (balg / (peak * world * 1e9)) / 1e9
    roof_comp = flops / (comp / (peak * world * 1e9)) / 1e9
    value = flops / (ms_per_step * 1e-3) / 1e9
    return {
        "bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
        "peak": peak * world, "unit": "GB/s",
        "frac": round(achieved / (peak * world), 4) if achieved else None,
        "traffic": traffic[0] if traffic else None,
        "kernel": dom, "bytes_alg_per_launch": launch_bytes, "units_per_launch": int(units),
        "bytes_per_unit": round(balg / max(total_mults, 1), 2),
        "kernel_ms_per_launch": round(kf_ms, 4),
        "step_frac": round(value / roof_alg, 4),
        "roofline_gflops": round(roof_alg, 1),
        # SURVEY.md §8(d) secondary column: every array touched once, no
        # accumulator term (the floor DRAM traffic is compared to)
        "compulsory_bytes": int(comp), "roofline_compulsory_gflops": round(roof_comp, 1),
        "step_frac_compulsory": round(value / roof_comp, 4),
        # ncu DRAM bytes of the committed capture over the live kernel time
        "dram_gbs": round(traffic[0] / (kf_ms * 1e-3) / 1e9, 1) if traffic and kf_ms else None,
        "dram_frac": round(traffic[0] / (kf_ms * 1e-3) / 1e9 / peak, 4) if traffic and kf_ms
        else None,
        "peak_source": peak_src + (f" x {world} GPUs" if world > 1 else ""),
        "traffic_source": traffic[1] if traffic else
        ("no ncu --set full summary committed" if world == 1 else "per-GPU ncu is single-GPU only"),
    }


def c_abi_step(_lib, ctx, va, vb):
    """One product through the C ABI as a native caller makes it —
    spmmm_multiply then spmmm_product_destroy on prebuilt arguments — so the
    timed step carries no Python wrapper objects (the Product class adds ~4 us
    a call, visible only at C1's size). Raises on any failure."""
    import ctypes

    L = _lib.lib()
    mul, destroy = L.spmmm_multiply, L.spmmm_product_destroy
    h = ctypes.c_void_p()
    args = (ctx.handle, ctypes.byref(va), ctypes.byref(vb), 6, 0, ctypes.byref(h))

    def step():
        rc = mul(*args)
        if rc:
            _lib.check(rc, "spmmm_multiply")
        destroy(h)
    return step


def dominant_kernel(kernel_ms):
    dom = max(kernel_ms, key=kernel_ms.get) if kernel_ms else "k_fused"
    return dom if dom in ("k_fused", "k_esc_block") else "k_fused"


def esc_units(a, b, prod_per_row):
    """k_esc_block's units: the products of the rows it computes — rows past
    the warp-row limit (mid rows whole, huge rows as column-range parts) that
    are not dominated by one long B row (those are k_esc_dom's). The limits
    are the library's own (spmmm_row_classes)."""
    import ctypes

    from paper_1303_1651_b200 import _lib

    lim = (ctypes.c_uint32 * 5)()
    _lib.check(_lib.lib().spmmm_row_classes(lim), "spmmm_row_classes")
    warp_limit, _, rcap, minrun, half = (int(x) for x in lim)
    arp = a.row_ptr.astype(np.int64)
    lens_b = np.diff(b.row_ptr.astype(np.int64))[a.col_idx.astype(np.int64)]
    longest = np.zeros(a.rows, np.int64)
    nz = np.flatnonzero(np.diff(arp) > 0)
    if nz.size:
        longest[nz] = np.maximum.reduceat(lens_b, arp[nz])
    dominated = (longest >= minrun) & (prod_per_row - longest <= rcap)
    if half:
        dominated &= 2 * longest >= prod_per_row
    return int(prod_per_row[(prod_per_row > warp_limit) & ~dominated].sum())


# ---------------------------------------------------------------------------
# our arm, one GPU


def run_single(args):
    import torch

    from paper_1303_1651_b200 import _lib
    from paper_1303_1651_b200 import device as dev
    from paper_1303_1651_b200 import genmat
    from paper_1303_1651_b200.formats import CsrMatrix
    from paper_1303_1651_b200.kernels import (PIPELINE_MIN_NNZ, multiply_rowmajor,
                                              row_products_prefix)
    from paper_1303_1651_b200.perfmodel import bytes_alg

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    label = args.config
    override = {"grid": args.grid} if args.grid else {}
    a, b, _ = genmat.config_operands(label, **override)
    same = b is a
    ctx = dev.context_for_current_stream(device)
    ad = dev.DeviceCsr.from_host(a, device)
    bd = ad if same else dev.DeviceCsr.from_host(b, device)
    va, vb = ad.view(), bd.view()  # (device views built once, not per step)

    def step(flags=_lib.FLAG_TIMING):
        p = _lib.multiply_views(ctx, va, vb, 6, flags)
        info = (p.multiplications, p.nnz, ctx.last_timings(), ctx.last_launch_count())
        p.close()
        return info

    bare_step = c_abi_step(_lib, ctx, va, vb)

    for _ in range(args.warmup):
        step()
        bare_step()
    mults, nnz_c, _, _ = step()
    with _lib.multiply_views(ctx, va, vb, 6, 0) as p:
        reserved = p.reserved_bytes()
    torch.cuda.synchronize()
    free0, total_mem = torch.cuda.mem_get_info(device)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms, launches = {}, 0
    with ClockSampler(0) as clk:
        # timed region: exactly K products as a caller runs them
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            bare_step()
        end.record()
        torch.cuda.synchronize()
        elapsed_ms = start.elapsed_time(end)
        # per-kernel durations: K more products with the library's CUDA events
        # on its launch stream (SPMMM_FLAG_TIMING: ~15 us of host-side event
        # work per product, so these steps are not the headline)
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record()
        for _ in range(args.steps):
            _, _, t, n = step()
            launches += n
            for k, v in t.items():
                kernel_ms[k] = kernel_ms.get(k, 0.0) + v
        i1.record()
        torch.cuda.synchronize()
        instrumented_ms = i0.elapsed_time(i1) / args.steps
    ms_per_step = elapsed_ms / args.steps
    flops = 2.0 * mults
    value = flops / (ms_per_step * 1e-3) / 1e9

    nnz_a = len(a.values)
    balg = bytes_alg(a.rows, nnz_a, mults, nnz_c)
    dom = dominant_kernel(kernel_ms)
    units = mults
    if dom == "k_esc_block":
        units = esc_units(a, b, np.diff(row_products_prefix(a, b).astype(np.int64)))
    roof = roofline_entry(label, kernel_ms.get(dom, 0.0) / args.steps, dom, balg, units, mults,
                          nnz_c, a.rows, nnz_a, len(b.values), b.rows, ms_per_step, 1)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": workload_config(label, args.grid, a, b, mults),
        "parallelism": "single GPU",
        "l2": "inputs larger than L2 (no flush)" if 16 * nnz_a > 126e6 else
              "inputs smaller than L2 (L2-warm)",
        "nnz_c": int(nnz_c),
        "kernel_ms": {k: round(v / args.steps, 4) for k, v in kernel_ms.items()},
        "kernel_ms_how": ("CUDA events around each kernel on the library's stream, in K more "
                          f"products right after the timed ones ({instrumented_ms:.4f} ms/step "
                          "with the events)"),
        "roofline": roof,
        "gpu_launches": launches,
        "gpu_launches_how": "launches per product (counted by the library) x K",
        "clocks": clk.summary(),
        "hbm_bytes": {"operands": int(16 * nnz_a + 8 * (a.rows + 1) +
                                      (0 if same else 16 * len(b.values) + 8 * (b.rows + 1))),
                      "result": int(16 * nnz_c + 8 * (a.rows + 1)),
                      "result_reserved": int(reserved),
                      "device_used_between_steps": int(total_mem - free0)},
    }

    # ---- e2e through the public drop-in API (host numpy in -> host numpy out) ----
    if not args.no_e2e:
        def pinned(arr):
            buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
            out = buf.numpy()[:arr.nbytes].view(arr.dtype)
            out[...] = arr
            return out

        def e2e_times(x, y):
            # warm: two live results, so the pinned pool holds the blocks a
            # step allocates while the previous step's result is still referenced
            warm = [multiply_rowmajor(x, y) for _ in range(2)]
            del warm
            multiply_rowmajor(x, y)  # one more with a single live result, as in the loop
            times, c = [], None
            for _ in range(max(1, args.e2e_steps)):
                t0 = time.perf_counter()
                c = multiply_rowmajor(x, y)
                times.append(time.perf_counter() - t0)
            return times, c

        def e2e_entry(times, c, api):
            e2e_s = float(np.median(times))  # host-side noise (page cache, scheduler): median
            h2d = 8 * (a.rows + 1) + 16 * nnz_a
            if not same:
                h2d += 8 * (b.rows + 1) + 16 * len(b.values)
            d2h = 8 * (c.rows + 1) + 16 * len(c.values)
            if _lib.last_transfer is not None and nnz_a >= PIPELINE_MIN_NNZ:
                # the pipelined path moves C's indices narrowed (u32 / u16 deltas)
                h2d = _lib.last_transfer["h2d_bytes"]
                d2h = _lib.last_transfer["d2h_bytes"]
            return {"value": round(flops / e2e_s / 1e9, 3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_s * 1e3, 3), "steps": len(times),
                    "stat": "median of the timed calls",
                    "ms_min_mean_max": [round(min(times) * 1e3, 3),
                                        round(float(np.mean(times)) * 1e3, 3),
                                        round(max(times) * 1e3, 3)],
                    "ms_each": [round(t * 1e3, 2) for t in times], "api": api}

        ap_ = CsrMatrix(a.rows, a.cols, pinned(a.row_ptr), pinned(a.col_idx), pinned(a.values))
        bp_ = ap_ if same else CsrMatrix(b.rows, b.cols, pinned(b.row_ptr), pinned(b.col_idx),
                                         pinned(b.values))
        times, c = e2e_times(ap_, bp_)
        line["e2e"] = e2e_entry(times, c, "paper_1303_1651_b200.multiply_rowmajor (pinned numpy "
                                "in, numpy out backed by the pinned pool; block-pipelined "
                                f"spmmm_multiply_host for >= {PIPELINE_MIN_NNZ} A entries)")
        del c, ap_, bp_
        times, c = e2e_times(a, b)  # the generator's ordinary (pageable) numpy arrays
        line["e2e_pageable"] = e2e_entry(times, c, "paper_1303_1651_b200.multiply_rowmajor "
                                         "(pageable numpy in, numpy out)")
        del c

    # ---- CPU baseline: the oracle port, 1 thread, bounded sample ----
    if not args.no_cpu_baseline:
        rate, sample, _ = cpu_oracle_rate(a, b, 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": round(rate, 4), "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": sample}
    line["native_libs_mapped"] = native_libs_mapped()
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


# ---------------------------------------------------------------------------
# our arm, N GPUs (one rank per GPU)


def run_distributed(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1303_1651_b200 import _lib
    from paper_1303_1651_b200 import distributed as D
    from paper_1303_1651_b200.perfmodel import bytes_alg

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    ngpu = torch.cuda.device_count()
    backend = args.backend
    if backend == "nccl":
        # the driver counts ranks in NCCL's INFO log (the image may preset a
        # quieter level); NCCL logs to stdout by default, where rank 0's one
        # JSON line goes: send the log to stderr
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if world > ngpu:
            raise SystemExit(f"--gpus {world} needs {world} GPUs, this node has {ngpu} "
                             "(use --backend gloo to run oversubscribed ranks as a functional test)")
    device = torch.device("cuda", local_rank % ngpu)
    torch.cuda.set_device(device)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group("gloo")
    ctrl = D.control_group()
    label = args.config

    # operands: built once on rank 0, shared node-wide (operand preparation)
    a = b = None
    if rank == 0:
        from paper_1303_1651_b200 import genmat

        override = {"grid": args.grid} if args.grid else {}
        a, b, _ = genmat.config_operands(label, **override)
    same_box = [b is a]
    dist.broadcast_object_list(same_box, src=0, group=ctrl)
    a = D.share_csr(a)
    b = a if same_box[0] else D.share_csr(b)
    same = b is a

    # plan (untimed): operands resident on every GPU, partition
    dist.barrier(group=ctrl)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    ev0.record()
    ad = D.replicate_csr(a, None, device)
    bd = ad if same else D.replicate_csr(b, None, device)
    ev1.record()
    torch.cuda.synchronize()
    replicate_ms = max(ev0.elapsed_time(ev1), 1e3 * (time.perf_counter() - h0))
    bounds = [int(x) for x in D.gpu_partition(ad, bd, world)]
    r0, r1 = bounds[rank], bounds[rank + 1]
    ctx = D._context(device)
    va, vb = D._view(ad, r0, r1), D._view(bd)

    def step():
        p = _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING)
        info = (p.multiplications, p.nnz, ctx.last_timings(), ctx.last_launch_count())
        p.close()
        return info

    bare_step = c_abi_step(_lib, ctx, va, vb)

    for _ in range(args.warmup):
        step()
        bare_step()
    mults_local, nnz_local, _, _ = step()

    # ---- timed region: exactly K steps of every rank's block ----
    dist.barrier(group=ctrl)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms, launches = {}, 0
    with ClockSampler(device.index) as clk:
        start.record()
        for _ in range(args.steps):
            bare_step()
        end.record()
        torch.cuda.synchronize()
        dist.barrier(group=ctrl)
        elapsed_ms = start.elapsed_time(end)
        # per-kernel durations: K more steps with the library's CUDA events
        for _ in range(args.steps):
            _, _, t, n = step()
            launches += n
            for k, v in t.items():
                kernel_ms[k] = kernel_ms.get(k, 0.0) + v
        torch.cuda.synchronize()
    dist.barrier(group=ctrl)

    # ---- e2e: the whole distributed call, shared host operands -> shared host result ----
    e2e = None
    if not args.no_e2e:
        tm = {}
        for _ in range(2):  # warm: arena growth and page-locking happen here
            D.multiply_distributed(a, b, timings=tm)
        per_call, gathers = [], []
        for _ in range(max(1, args.e2e_steps)):
            dist.barrier(group=ctrl)
            t0 = time.perf_counter()
            c = D.multiply_distributed(a, b, timings=tm)
            per_call.append(time.perf_counter() - t0)
            gathers.append(tm["gather_ms"])
            del c
        e2e = (per_call, gathers, dict(tm))

    # ---- max over ranks ----
    mine = {"elapsed_ms": elapsed_ms, "mults": int(mults_local), "nnz": int(nnz_local),
            "kernel_ms": kernel_ms, "launches": launches, "clocks": clk.summary(),
            "replicate_ms": replicate_ms, "bounds": [r0, r1], "e2e": e2e}
    allr = [None] * world
    dist.all_gather_object(allr, mine, group=ctrl)
    if rank == 0:
        elapsed = max(r["elapsed_ms"] for r in allr)
        total_mults = sum(r["mults"] for r in allr)
        total_nnz = sum(r["nnz"] for r in allr)
        ms_per_step = elapsed / args.steps
        flops = 2.0 * total_mults
        value = flops / (ms_per_step * 1e-3) / 1e9
        kmax = {}
        for r in allr:
            for k, v in r["kernel_ms"].items():
                kmax[k] = max(kmax.get(k, 0.0), v / args.steps)
        dom = dominant_kernel(kmax)
        nnz_a = len(a.values)
        balg = bytes_alg(a.rows, nnz_a, total_mults, total_nnz)
        units = total_mults
        if dom == "k_esc_block":
            from paper_1303_1651_b200.kernels import row_products_prefix

            units = esc_units(a, b, np.diff(row_products_prefix(a, b).astype(np.int64)))
        roof = roofline_entry(label, kmax.get(dom, 0.0), dom, balg, units, total_mults, total_nnz,
                              a.rows, nnz_a, len(b.values), b.rows, ms_per_step, world)
        roof["note"] = ("achieved = all ranks' algorithmic bytes / the slowest rank's kernel "
                        "time; peak = N x the one-GPU HBM peak")
        per_rank_prod = [r["mults"] for r in allr]
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": workload_config(label, args.grid, a, b, total_mults),
            "parallelism": f"product-balanced row blocks x{world} ({backend})",
            "l2": "inputs larger than L2 (no flush)" if 16 * nnz_a > 126e6 else
                  "inputs smaller than L2 (L2-warm)",
            "nnz_c": int(total_nnz),
            "kernel_ms": {k: round(v, 4) for k, v in kmax.items()},
            "kernel_ms_stat": "per launch, max over ranks",
            "rank_ms_per_step": [round(r["elapsed_ms"] / args.steps, 4) for r in allr],
            "rank_products": per_rank_prod,
            "balance": round(max(per_rank_prod) / max(1.0, total_mults / world), 4),
            "b_allgather_ms": round(max(r["replicate_ms"] for r in allr), 3),
            "b_allgather_what": ("each rank uploads 1/N of A" + ("" if same else " and of B") +
                                 f" from shared host memory, then all-gather ({backend})"),
            "roofline": roof,
            "gpu_launches": int(sum(r["launches"] for r in allr)),
            "gpu_launches_stat": "sum over ranks",
            "clocks": merge_clocks([r["clocks"] for r in allr]),
        }
        if backend != "nccl" or world > ngpu:
            line["oversubscribed"] = f"{world} ranks on {ngpu} GPU(s): functional run, not a measurement"
        if e2e is not None:
            calls = len(allr[0]["e2e"][0])
            worst = [max(r["e2e"][0][i] for r in allr) for i in range(calls)]
            gth = [max(r["e2e"][1][i] for r in allr) for i in range(calls)]
            e2e_s = float(np.median(worst))
            h2d = 8 * (a.rows + 1) + 16 * nnz_a
            if not same:
                h2d += 8 * (b.rows + 1) + 16 * len(b.values)
            d2h = 8 * (a.rows + 1) + 16 * total_nnz
            line["e2e"] = {"value": round(flops / e2e_s / 1e9, 3), "unit": UNIT,
                           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                           "ms_per_step": round(e2e_s * 1e3, 3), "steps": calls,
                           "stat": "median over calls of the max over ranks (host clock)",
                           "ms_each": [round(t * 1e3, 2) for t in worst],
                           "api": "paper_1303_1651_b200.distributed.multiply_distributed "
                                  "(shared page-locked host operands in, shared host result out)"}
            line["gather_ms"] = round(float(np.median(gth)), 3)
            line["gather_what"] = ("nnz all-gather, result reservation, every rank's D2H of its "
                                   "block into its slice of the shared host result")
        line["native_libs_mapped"] = native_libs_mapped()
        print(json.dumps(line), flush=True)
    dist.barrier(group=ctrl)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--grid", type=int, default=None, help="another point of the stencil sweep")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="N > 1: NCCL (product); gloo runs oversubscribed ranks as a functional test")
    ap.add_argument("--distributed", action="store_true",
                    help="take the N-GPU path even at N = 1 (a one-rank NCCL run of its code)")
    ap.add_argument("--e2e-steps", type=int, default=7)
    ap.add_argument("--cpu-budget", type=float, default=8.0,
                    help="seconds of single-thread CPU work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.grid and args.config not in ("C2",):
        raise SystemExit("--grid applies to the C2 sweep")

    from paper_1303_1651_b200.launch import spawn, under_torchrun

    if not under_torchrun() and args.gpus > 1:
        # one process per GPU: re-run this command under torch.distributed.run
        return spawn(args.gpus, os.path.abspath(__file__), sys.argv[1:]).returncode
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 or args.distributed:
        return run_distributed(args, rank, world, local_rank)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
