"""The count-free path (k_prep -> k_fused, one host round trip) against the
pinned oracle: both flavours (ELL records of a whole B; CSR rows of B for a
row block of A), stats included, and every way it must decline — a long A
row, a long B row, malformed row pointers, an A column past B.rows — where
the counted path must produce the same bytes or the reference's error."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import assert_csr_bitwise_equal, have_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200.formats import CsrMatrix  # noqa: E402
from paper_1303_1651_b200.kernels import (KernelStats, StrategyKind,  # noqa: E402
                                          _record_row_choices)


def _ref(a, b):
    r = oracle.multiply_rowmajor(a, b, row_choices=True, threads=8)
    return CsrMatrix(r.rows, r.cols, r.row_ptr, r.col_idx, r.values), r


def _choices(stats, rows):
    out = np.full(rows, -1, np.int8)
    for r, ch in stats.row_choices:
        out[r] = 0 if ch == StrategyKind.MIN_MAX else 1
    return out


def _run(ctx, a, b, stats=True):
    va = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    vb = va if b is a else _lib.csr_view(b.rows, b.cols, b.row_ptr, b.col_idx, b.values)
    flags = _lib.FLAG_TIMING | (_lib.FLAG_ROW_STATS if stats else 0)
    with _lib.multiply_views(ctx, va, vb, 6, flags) as p:
        rp, ci, v = p.download()
        st = KernelStats()
        if stats:
            _record_row_choices(st, p, StrategyKind, a.row_ptr)
        names = set(ctx.last_timings())
        return CsrMatrix(a.rows, b.cols, rp, ci, v), p.multiplications, st, names


def _random_rows(rng, rows, cols, kmax, signed=True):
    lens = rng.integers(0, kmax + 1, rows)
    rp = np.zeros(rows + 1, np.uint64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(cols, int(n), replace=False)) for n in lens]
                        ).astype(np.uint64) if lens.sum() else np.zeros(0, np.uint64)
    v = rng.integers(-3, 4, int(lens.sum())).astype(np.float64) if signed else \
        rng.random(int(lens.sum()))
    return CsrMatrix(rows, cols, rp, ci, v)


@pytest.mark.parametrize("grid", [1, 2, 7, 64, 100, 300])
def test_ell_flavour_stencil_squares(grid):
    ctx = _lib.Context(0)
    a = genmat.gen_fd(grid)
    ref, r = _ref(a, a)
    for _ in range(2):  # the second call reuses the cached C blocks
        c, mults, st, names = _run(ctx, a, a)
        # count-free: no k_count (small products run the prep pass inside k_fused)
        assert "k_count" not in names and ("k_prep" in names or a.rows <= 1 << 14), names
        assert_csr_bitwise_equal(c, ref, f"fd{grid}")
        assert mults == r.multiplications
        assert np.array_equal(_choices(st, a.rows), r.row_choices)
    ctx.close()


@pytest.mark.parametrize("seed", range(6))
def test_ell_flavour_random_with_cancellations(seed):
    """Values in {-3..3}: exact cancellations and transient zeros inside rows."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    a = _random_rows(rng, n, n, 6)
    b = _random_rows(rng, n, int(rng.integers(1, 5000)), 5)
    ref, r = _ref(a, b)
    ctx = _lib.Context(0)
    c, mults, st, names = _run(ctx, a, b)
    assert "k_count" not in names, names
    assert_csr_bitwise_equal(c, ref, f"random{seed}")
    assert mults == r.multiplications
    assert np.array_equal(_choices(st, a.rows), r.row_choices)
    ctx.close()


def test_csr_flavour_row_blocks():
    """A row block of A against all of B (the distributed and pipelined
    shape): B is read as CSR, rows with na * nb <= 32."""
    import torch

    from paper_1303_1651_b200 import device as dev
    from paper_1303_1651_b200.distributed import concat_row_blocks

    rng = np.random.default_rng(11)
    a = _random_rows(rng, 40_000, 30_000, 4)
    b = _random_rows(rng, 30_000, 50_000, 8)
    full, _ = _ref(a, b)
    d = torch.device("cuda", 0)
    ad, bd = dev.DeviceCsr.from_host(a, d), dev.DeviceCsr.from_host(b, d)
    ctx = dev.context_for_current_stream(d)
    bounds = [0, 5000, 17_000, 17_001, 40_000]
    blocks = []
    for g in range(4):
        with dev.multiply(ctx, ad.row_block(bounds[g], bounds[g + 1]), bd,
                          flags=_lib.FLAG_TIMING) as p:
            blocks.append(p.download())
            assert "k_prep" in ctx.last_timings()
    assert_csr_bitwise_equal(concat_row_blocks(blocks, b.cols), full, "csr flavour")
    ctx.close()


@pytest.mark.parametrize("what", ["long_a", "long_b", "wide_product"])
def test_declines_to_counted_path_with_same_bytes(what):
    rng = np.random.default_rng(5)
    n = 2000
    a = _random_rows(rng, n, n, 5)
    b = _random_rows(rng, n, 3000, 5)
    if what == "long_a":
        a = _random_rows(rng, n, n, 12)
    elif what == "long_b":
        b = _random_rows(rng, n, 3000, 9)
    else:  # CSR flavour (A a small block of B's rows) with na * nb > 32
        a = _random_rows(rng, 100, n, 6)
        b = _random_rows(rng, n, 3000, 7)
    ref, r = _ref(a, b)
    ctx = _lib.Context(0)
    launches = []
    for call in range(2):
        c, mults, st, names = _run(ctx, a, b)
        assert "k_count" in names, names
        launches.append(ctx.last_launch_count())
        assert_csr_bitwise_equal(c, ref, what)
        assert mults == r.multiplications
        assert np.array_equal(_choices(st, a.rows), r.row_choices)
    # first call: the count-free path tried and declined (its launches come on
    # top of the counted path's); second call: not tried again
    assert launches[0] > launches[1], launches
    ctx.close()


def test_bad_column_gets_the_reference_error():
    a = genmat.gen_fd(20)
    ci = a.col_idx.copy()
    ci[17] = np.uint64(a.cols + 3)
    bad = CsrMatrix(a.rows, a.cols, a.row_ptr.copy(), ci, a.values.copy())
    ctx = _lib.Context(0)
    vb = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    va = _lib.csr_view(bad.rows, bad.cols, bad.row_ptr, bad.col_idx, bad.values)
    with pytest.raises(ValueError, match="a.col_idx entry >= b.rows"):
        _lib.multiply_views(ctx, va, vb, 6, 0)
    # the context is still usable, and good operands still take the fast path
    c, _, _, names = _run(ctx, a, a)
    assert "k_count" not in names
    ref, _ = _ref(a, a)
    assert_csr_bitwise_equal(c, ref, "after error")
    ctx.close()


def test_malformed_row_ptr_gets_the_reference_error():
    a = genmat.gen_fd(10)
    rp = a.row_ptr.copy()
    rp[5], rp[6] = rp[6], rp[5]  # decreasing
    bad = CsrMatrix(a.rows, a.cols, rp, a.col_idx.copy(), a.values.copy())
    ctx = _lib.Context(0)
    va = _lib.csr_view(bad.rows, bad.cols, bad.row_ptr, bad.col_idx, bad.values)
    vb = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    with pytest.raises(ValueError, match="malformed a.row_ptr"):
        _lib.multiply_views(ctx, va, vb, 6, 0)
    ctx.close()


def test_single_host_round_trip_launches():
    """k_prep and k_fused (whose last warp reports to the host): two launches
    and one host round trip per product; small products one launch (the prep
    pass inside k_fused, behind a grid barrier)."""
    ctx = _lib.Context(0)
    for g, launches in ((100, 1), (300, 2)):
        a = genmat.gen_fd(g)
        va = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
        for _ in range(3):
            with _lib.multiply_views(ctx, va, va, 6, 0):
                assert ctx.last_launch_count() == launches, g
    ctx.close()


def test_medium_reservation_overflow_is_redone_exactly():
    """The medium variant reserves min(products, SPMMM_C_RESERVE x nnz(A))
    entries (at least 2^20); with a factor of 1 the 40^3 27-point stencil's square (nnz(C) ~ 4.5
    nnz(A)) outgrows it, writes nothing past it and is redone sized by the
    product count: same bytes, and the redo's reservation is the exact one."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path[:0] = ['.', 'oracle']\n"
        "import oracle\n"
        "from paper_1303_1651_b200 import _lib, genmat\n"
        "a = genmat.gen_fd3(40)\n"
        "ctx = _lib.Context(0)\n"
        "v = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)\n"
        "with _lib.multiply_views(ctx, v, v, 6, 0) as p:\n"
        "    rp, ci, vv = p.download(); res = p.reserved_bytes(); m = p.multiplications\n"
        "r = oracle.multiply_rowmajor(a, a, threads=8)\n"
        "assert rp.tobytes() == r.row_ptr.tobytes() and ci.tobytes() == r.col_idx.tobytes()\n"
        "assert vv.tobytes() == r.values.tobytes() and m == r.multiplications\n"
        "print(res, len(vv), m)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for factor in ("1", "8"):
        env = dict(os.environ, SPMMM_C_RESERVE=factor)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        out[factor] = [int(x) for x in r.stdout.split()]
    res1, nnz, mults = out["1"]
    res8, _, _ = out["8"]
    assert res1 >= 16 * mults  # redone at the product count
    assert res8 < 16 * mults and res8 >= 16 * nnz  # the bounded reservation held
