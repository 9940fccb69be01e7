"""Randomised parity stress: many seeded shapes and distributions through the
drop-in (stats on and off, one-shot and pipelined paths, count-free and
counted, pageable operands through the staging) against the oracle, bit for
bit. Usage: python tools/stress_parity.py SECONDS [SEED]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import oracle  # noqa: E402
from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200.formats import CsrMatrix  # noqa: E402
from paper_1303_1651_b200.kernels import (KernelStats, StrategyKind,  # noqa: E402
                                          multiply_rowmajor)


def rand_csr(rng, rows, cols, lens, values):
    lens = np.minimum(lens, cols)
    rp = np.zeros(rows + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    parts = []
    for r in range(rows):
        n = int(lens[r])
        if n == 0:
            parts.append(np.zeros(0, np.int64))
            continue
        if n > cols // 4:
            c = rng.choice(cols, n, replace=False)
        else:
            c = np.unique(rng.integers(0, cols, 2 * n))
            while c.size < n:
                c = np.unique(np.concatenate([c, rng.integers(0, cols, n)]))
            c = rng.permutation(c)[:n]
        parts.append(np.sort(c))
    ci = np.concatenate(parts).astype(np.uint64) if parts else np.zeros(0, np.uint64)
    if values == "quantized":
        v = rng.choice([-2.0, -1.0, 0.5, 1.0, 2.0], ci.size)
    elif values == "zeros":
        v = rng.choice([0.0, -0.0, 1.0, -1.0], ci.size)
    else:
        v = rng.uniform(-1, 1, ci.size)
    return CsrMatrix(rows, cols, rp, ci, v)


def case(rng):
    kind = rng.choice(["uniform", "zipf", "wide", "dense", "narrow", "short", "shortcsr"])
    values = rng.choice(["uniform", "quantized", "zeros"])
    m = int(rng.integers(1, 20000))
    k = m if rng.random() < 0.3 else int(rng.integers(1, 20000))
    n = int(rng.integers(1, 30000))
    if kind == "uniform":
        la = rng.integers(0, 40, m)
        lb = rng.integers(0, 40, k)
    elif kind == "zipf":
        la = np.minimum(rng.zipf(2.0, m), 3000)
        lb = np.minimum(rng.zipf(2.0, k), 600)
    elif kind == "wide":
        n = int(rng.integers(1 << 23, 1 << 31))
        la = rng.integers(0, 30, m)
        lb = rng.integers(0, 40, k)
    elif kind == "dense":
        n = int(rng.integers(1, 200))
        la = rng.integers(0, 60, m)
        lb = rng.integers(0, 60, k)
    elif kind == "short":  # the count-free path, ELL flavour (rows <= 6 and <= 5 entries)
        la = rng.integers(0, 7, m)
        lb = rng.integers(0, 6, k)
    elif kind == "shortcsr":  # the count-free path, CSR flavour (na * nb <= 32)
        la = rng.integers(0, 5, m)
        lb = rng.integers(0, 9, k)
    else:
        n = int(rng.integers(1, 3000))
        la = np.minimum(rng.zipf(1.7, m), 2000)
        lb = np.minimum(rng.zipf(1.7, k), 300)
    a = rand_csr(rng, m, k, la, values)
    b = rand_csr(rng, k, n, lb, values)
    return f"{kind}/{values}/{m}x{k}x{n}", a, b


def check(name, a, b):
    ref = oracle.multiply_rowmajor(a, b, row_choices=True, threads=8)
    stats = KernelStats()
    c1 = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
    c2 = multiply_rowmajor(a, b)
    for c, tag in ((c1, "stats"), (c2, "plain")):
        for x, y, what in ((c.row_ptr, ref.row_ptr, "row_ptr"), (c.col_idx, ref.col_idx, "col_idx"),
                           (c.values, ref.values, "values")):
            if np.asarray(x).tobytes() != np.asarray(y).tobytes():
                raise AssertionError(f"{name} [{tag}]: {what} differs")
    # the pipelined host path directly, random block count (A·A when square)
    ctx = _lib.default_context()
    va = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    for bb, vb in ((b, _lib.csr_view(b.rows, b.cols, b.row_ptr, b.col_idx, b.values)),):
        blocks = int(np.random.default_rng(a.rows).integers(1, 17))
        rp, ci, v, m = _lib.multiply_host(ctx, va, vb, 6, 0, blocks)
        for x, y, what in ((rp, ref.row_ptr, "row_ptr"), (ci, ref.col_idx, "col_idx"),
                           (v, ref.values, "values")):
            if np.asarray(x).tobytes() != np.asarray(y).tobytes():
                raise AssertionError(f"{name} [pipelined, {blocks} blocks]: {what} differs")
    if a.rows == a.cols == b.rows:
        # C = A·A through the pipelined path (blocks wait for the rows they read)
        ref2 = oracle.multiply_rowmajor(a, a, threads=8)
        rp, ci, v, m = _lib.multiply_host(ctx, va, va, 6, 0, 1 + a.rows % 16)
        for x, y, what in ((rp, ref2.row_ptr, "row_ptr"), (ci, ref2.col_idx, "col_idx"),
                           (v, ref2.values, "values")):
            if np.asarray(x).tobytes() != np.asarray(y).tobytes():
                raise AssertionError(f"{name} [pipelined A·A]: {what} differs")
    ch = np.full(a.rows, -1, np.int8)
    for r, s in stats.row_choices:
        ch[r] = 0 if s == StrategyKind.MIN_MAX else 1
    if not np.array_equal(ch, ref.row_choices):
        raise AssertionError(f"{name}: row choices differ")
    if stats.multiplications != ref.multiplications:
        raise AssertionError(f"{name}: multiplications differ")


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
    t0 = time.time()
    n = 0
    while time.time() - t0 < budget:
        name, a, b = case(rng)
        check(name, a, b)
        n += 1
    # the pipelined path at a size past its threshold, skewed and stencil
    for name, a, b in [("zipf800k", genmat.gen_zipf(800_000, 21), genmat.gen_zipf(800_000, 22)),
                       ("fd1100", genmat.gen_fd(1100), None)]:
        check(name, a, a if b is None else b)
        n += 1
    print(f"stress ok: {n} cases in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
