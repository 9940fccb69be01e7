"""Benchmark-harness integration: B200 cells in the
reference harness's experiment grid and CSV contract.

The reference harness (`sparsemm.bench`, bench.py:39-40, 97-142, 209-237,
353-381) measures (family, size, kernel, strategy) cells with a calibrated
protocol — the inner repetition count doubles until one batch takes more than
`min_total_seconds`, then `trials` batches are timed and the best
per-invocation time is reported, as MFlop/s from the worst-case flop count —
and writes `case,family,n,kernel,strategy,seed,inner_iters,best_seconds,mflops`
rows. This module runs the same grid for the GPU kernels under their own
kernel names, so their rows can be concatenated with the reference's CPU rows:

    b200            multiply_rowmajor through the drop-in: host CSR in, host CSR
                    out (the reference `rowmajor` cell's contract, on the GPU)
    b200-colmajor   multiply_colmajor on CSC operands converted outside the
                    timed region (the `colmajor` cell)
    b200-mixed      multiply_mixed with B column-major: the one conversion runs
                    inside the timed region (the `mixed` cell)
    b200-device     operands resident in HBM, result left on the device; timed
                    with CUDA events on the context's stream (kernel-only rate)

Operands come from the native bit-identical generators (genmat.py:79-151:
`fd` picks the grid side nearest sqrt(n) and squares one matrix; `random` and
`fill` multiply two matrices seeded `seed` and `seed + 1`). Like the
reference, SPARSEMM_CLOCK_OVERRIDE installs a virtual clock that advances by
that many seconds per invocation (deterministic protocol tests).

    python -m paper_1303_1651_b200.harness run --case fd --kernel b200 b200-device \\
        --sizes 64:4194304:x4 --csv gpu.csv
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

CLOCK_OVERRIDE_ENV = "SPARSEMM_CLOCK_OVERRIDE"
CSV_HEADER = "case,family,n,kernel,strategy,seed,inner_iters,best_seconds,mflops"
FAMILIES = ("fd", "random", "fill")
KERNEL_NAMES = ("b200", "b200-colmajor", "b200-mixed", "b200-device")
STRATEGIES = ("bfdouble", "bfbool", "bfchar", "minmax", "minmaxchar", "sort", "combined")
DENSE_CHECK_LIMIT = 512  # largest dimension the dense fold check runs at


@dataclass(frozen=True)
class TimingResult:
    inner_iters: int
    best_seconds: float
    mflops: float


@dataclass(frozen=True)
class BenchRecord:
    case: str
    family: str
    n: int
    kernel: str
    strategy: str
    seed: int
    inner_iters: int
    best_seconds: float
    mflops: float


@dataclass(frozen=True)
class SkipRecord:
    case: str
    n: int
    kernel: str
    strategy: str
    reason: str


@dataclass
class GridResult:
    records: list
    skipped: list


class _VirtualClock:
    def __init__(self, tick: float):
        if tick <= 0:
            raise ValueError("tick must be positive")
        self.tick, self.now = tick, 0.0


def _event_clock():
    """A clock over CUDA events on the current stream: reading it records an
    event; differences of readings are device time (seconds)."""
    import torch

    base = torch.cuda.Event(enable_timing=True)
    base.record()

    def read():
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        ev.synchronize()
        return base.elapsed_time(ev) / 1e3

    return read


def time_kernel(work, flops: int, *, clock=None, min_total_seconds: float = 2.0,
                trials: int = 5) -> TimingResult:
    """The reference protocol (bench.py:97-142): double the inner count until
    a batch exceeds `min_total_seconds`, then the best of `trials` batches per
    invocation. `clock=None` uses perf_counter (or the virtual clock of
    SPARSEMM_CLOCK_OVERRIDE); `clock="events"` uses CUDA events."""
    if trials < 1:
        raise ValueError("need at least one trial")
    if clock is None:
        tick = os.environ.get(CLOCK_OVERRIDE_ENV)
        if tick is not None:
            vc = _VirtualClock(float(tick))
            inner_work = work

            def work():
                inner_work()
                vc.now += vc.tick

            clock = lambda: vc.now  # noqa: E731
        else:
            clock = time.perf_counter
    elif clock == "events":
        clock = _event_clock()
    inner = 1
    while True:
        t0 = clock()
        for _ in range(inner):
            work()
        if clock() - t0 > min_total_seconds:
            break
        if inner > 1 << 40:
            raise RuntimeError("clock does not advance; cannot calibrate")
        inner *= 2
    best = math.inf
    for _ in range(trials):
        t0 = clock()
        for _ in range(inner):
            work()
        best = min(best, (clock() - t0) / inner)
    return TimingResult(inner, best, flops / best / 1e6)


def case_label(family: str, n: int, k: int, fill: float) -> str:
    """bench.py:144-150 (no commas: one CSV field)."""
    if family == "fd":
        return f"fd[n={n}]"
    if family == "random":
        return f"random[n={n};k={k}]"
    return f"fill[n={n};fill={fill:g}]"


def fill_row_count(n: int, fill: float) -> int:
    """genmat.py:133-137: round half up, at least one entry."""
    if not 0.0 < fill <= 1.0:
        raise ValueError("need 0 < fill <= 1")
    return max(1, int(fill * n + 0.5))


def operands(family: str, n: int, seed: int, k: int = 5, fill: float = 0.001):
    """(a, b, k_used) of one grid cell (genmat.py:145-151, bench.py:205-211)."""
    from .genmat import gen_fd, gen_random_k

    if family not in FAMILIES:
        raise ValueError(f"unknown family {family!r}")
    if n < 1:
        raise ValueError("n must be at least 1")
    if family == "fd":
        a = gen_fd(max(1, round(math.sqrt(n))))
        return a, a, k
    kk = min(k, n) if family == "random" else fill_row_count(n, fill)
    seed2 = (seed + 1) & ((1 << 64) - 1)
    return gen_random_k(n, kk, seed), gen_random_k(n, kk, seed2), kk


def _dense_fold(a, b):
    """C = A·B densely as rank-1 updates in ascending k: every entry is the
    left fold over k of separately rounded products (kernels.py:441-457)."""
    ad, bd = a.to_dense(), b.to_dense()
    out = np.zeros((ad.shape[0], bd.shape[1]))
    for k in range(ad.shape[1]):
        out += np.multiply.outer(ad[:, k], bd[k, :])
    return out


def _verify(result, a, b, ref_rowmajor, label):
    """bench.py:161-182 with the GPU row-major result as the scatter kernel's
    stand-in: structure equal, values within 1e-12; dense fold check when
    small."""
    from .formats import csc_to_csr

    c = csc_to_csr(result) if hasattr(result, "col_ptr") else result
    ok = (np.array_equal(c.row_ptr, ref_rowmajor.row_ptr)
          and np.array_equal(c.col_idx, ref_rowmajor.col_idx)
          and np.allclose(c.values, ref_rowmajor.values, rtol=1e-12, atol=0.0))
    if not ok:
        raise RuntimeError(f"verification failed: {label} disagrees with the row-major kernel")
    if max(a.rows, a.cols, b.cols) <= DENSE_CHECK_LIMIT:
        exp, got = _dense_fold(a, b), c.to_dense()
        if not (np.array_equal(got != 0.0, exp != 0.0)
                and np.allclose(got, exp, rtol=1e-12, atol=0.0)):
            raise RuntimeError(f"verification failed: {label} disagrees with the dense fold")


def run_grid(families, kernels, strategies, sizes, seed, *, k: int = 5, fill: float = 0.001,
             verify: bool = False, min_total_seconds: float = 2.0, trials: int = 5) -> GridResult:
    """bench.py:185-249 for the B200 kernel names. Conversions a cell's input
    format needs happen outside the timed region, except for `b200-mixed`,
    whose contract includes its one conversion."""
    from . import device as dev
    from .formats import csr_to_csc
    from .kernels import StrategyKind, multiply_colmajor, multiply_mixed, multiply_rowmajor
    from .perfmodel import count_mults

    records, skipped = [], []
    for family in families:
        for n in sizes:
            a, b, kk = operands(family, n, seed, k, fill)
            label = case_label(family, a.rows, kk, fill)
            flops = count_mults(a, b).flops
            cache = {}

            def csc(m, key):
                if key not in cache:
                    cache[key] = csr_to_csc(m)
                return cache[key]

            ref = multiply_rowmajor(a, b) if verify else None
            for kernel in kernels:
                for strategy in strategies:
                    sname = strategy.value if hasattr(strategy, "value") else str(strategy)
                    if kernel not in KERNEL_NAMES:
                        skipped.append(SkipRecord(label, a.rows, kernel, sname, "unknown kernel"))
                        continue
                    if strategy is None or sname == "none":
                        skipped.append(SkipRecord(label, a.rows, kernel, "none",
                                                  "kernel requires a storing strategy"))
                        continue
                    s = StrategyKind(sname)
                    clock = None
                    closers = []
                    if kernel == "b200":
                        work = lambda a=a, b=b, s=s: multiply_rowmajor(a, b, s)  # noqa: E731
                    elif kernel == "b200-colmajor":
                        ac, bc = csc(a, "a"), csc(b, "b")
                        work = lambda a=ac, b=bc, s=s: multiply_colmajor(a, b, s)  # noqa: E731
                    elif kernel == "b200-mixed":
                        bc = csc(b, "b")
                        work = lambda a=a, b=bc, s=s: multiply_mixed(a, b, s)  # noqa: E731
                    else:  # b200-device
                        import torch

                        d = torch.device("cuda", torch.cuda.current_device())
                        ctx = dev.context_for_current_stream(d)
                        ad = dev.DeviceCsr.from_host(a, d)
                        bd = ad if b is a else dev.DeviceCsr.from_host(b, d)

                        def work(ctx=ctx, ad=ad, bd=bd):
                            dev.multiply(ctx, ad, bd).close()

                        clock = "events"
                        closers.append(ctx.close)
                    result = work()
                    if verify and result is not None:
                        _verify(result, a, b, ref, f"{label}/{kernel}/{sname}")
                    t = time_kernel(work, flops, clock=clock,
                                    min_total_seconds=min_total_seconds, trials=trials)
                    for close in closers:
                        close()
                    records.append(BenchRecord(label, family, a.rows, kernel, sname, seed,
                                               t.inner_iters, t.best_seconds, t.mflops))
    return GridResult(records, skipped)


def emit_csv(records) -> str:
    """bench.py:252-260: the reference's CSV, one row per record."""
    out = [CSV_HEADER]
    for r in records:
        out.append(f"{r.case},{r.family},{r.n},{r.kernel},{r.strategy},{r.seed},"
                   f"{r.inner_iters},{r.best_seconds:.5e},{r.mflops:.6g}")
    return "\n".join(out) + "\n"


def parse_csv(text: str) -> list:
    """bench.py:263-275 (reads both the reference's rows and ours)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("missing or malformed CSV header")
    recs = []
    for ln in lines[1:]:
        case, fam, n, kern, strat, seed, inner, best, mf = ln.split(",")
        recs.append(BenchRecord(case, fam, int(n), kern, strat, int(seed), int(inner),
                                float(best), float(mf)))
    return recs


def parse_sizes(text: str) -> list:
    """bench.py:278-299: '64,128' or log-spaced 'start:stop:xF'."""
    if ":" not in text:
        return [int(p) for p in text.split(",") if p.strip()]
    start_s, stop_s, step_s = text.split(":")
    start, stop = int(start_s), int(stop_s)
    if not step_s.startswith("x"):
        raise ValueError(f"range step must look like 'x2', got {step_s!r}")
    factor = float(step_s[1:])
    if factor <= 1.0 or start < 1 or stop < start:
        raise ValueError(f"bad size range {text!r}")
    sizes, value = [], float(start)
    while round(value) <= stop:
        if not sizes or int(round(value)) != sizes[-1]:
            sizes.append(int(round(value)))
        value *= factor
    return sizes


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="paper_1303_1651_b200.harness",
                                description="B200 cells of the sparsemm benchmark grid (CSV).")
    sub = p.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="measure a grid of cases and emit CSV")
    run.add_argument("--case", nargs="+", choices=FAMILIES, default=["fd"])
    run.add_argument("--kernel", nargs="+", choices=KERNEL_NAMES, default=["b200"])
    run.add_argument("--strategy", nargs="+", choices=STRATEGIES, default=["combined"])
    run.add_argument("--sizes", default="64:1024:x2")
    run.add_argument("--seed", type=int, default=0)
    run.add_argument("--k", type=int, default=5)
    run.add_argument("--fill", type=float, default=0.001)
    run.add_argument("--csv")
    run.add_argument("--verify", action="store_true")
    run.add_argument("--strict", action="store_true")
    run.add_argument("--min-seconds", type=float, default=2.0)
    run.add_argument("--trials", type=int, default=5)
    args = p.parse_args(argv)
    from .kernels import StrategyKind

    res = run_grid(args.case, args.kernel, [StrategyKind(s) for s in args.strategy],
                   parse_sizes(args.sizes), args.seed, k=args.k, fill=args.fill,
                   verify=args.verify, min_total_seconds=args.min_seconds, trials=args.trials)
    text = emit_csv(res.records)
    if args.csv:
        with open(args.csv, "w", encoding="ascii") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    for s in res.skipped:
        print(f"skipped {s.case} kernel={s.kernel} strategy={s.strategy}: {s.reason}",
              file=sys.stderr)
    return 2 if args.strict and res.skipped else 0


if __name__ == "__main__":
    sys.exit(main())
