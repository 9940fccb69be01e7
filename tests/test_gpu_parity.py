"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and the pinned CPU oracle.

Bar (north_star): C.row_ptr / C.col_idx bit-exact, values within 1e-12
relative to the reference — the helper additionally flags any value that is
not bit-identical, since the kernels reproduce the reference's summation
order exactly.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import pytest

import oracle
from conftest import (assert_csr_bitwise_equal, fingerprints, golden_case, golden_names,
                      have_gpu)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

from paper_1303_1651_b200 import _lib, genmat  # noqa: E402
from paper_1303_1651_b200.formats import CsrMatrix, validate_csr  # noqa: E402
from paper_1303_1651_b200.kernels import (KernelStats, StrategyKind, estimate_nnz,  # noqa: E402
                                          multiply_rowmajor, row_products_prefix)

ALL_STRATEGIES = list(StrategyKind)


def _oracle_csr(a, b):
    r = oracle.multiply_rowmajor(a, b, threads=8)
    return CsrMatrix(r.rows, r.cols, r.row_ptr, r.col_idx, r.values)


def _choices_array(stats, rows):
    out = np.full(rows, -1, np.int8)
    for r, ch in stats.row_choices:
        out[r] = 0 if ch == StrategyKind.MIN_MAX else 1
    return out


@pytest.mark.parametrize("name", golden_names())
def test_golden_case(name):
    a, b, c_ref, mults, choices = golden_case(name)
    stats = KernelStats()
    c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
    assert_csr_bitwise_equal(c, c_ref, name)
    assert stats.multiplications == mults
    assert np.array_equal(_choices_array(stats, a.rows), choices), name
    assert estimate_nnz(a, b) == mults
    validate_csr(c)


def test_strategies_are_bitwise_unanimous():
    for name in ("random_0", "signed_k40", "long_rows", "medium_rows", "fd_9"):
        a, b, c_ref, _, _ = golden_case(name)
        for s in ALL_STRATEGIES:
            assert_csr_bitwise_equal(multiply_rowmajor(a, b, s), c_ref, f"{name}/{s.value}")


def test_errors_match_reference():
    a, b, _, _, _ = golden_case("rect_7x13_13x5")
    with pytest.raises(ValueError, match="dimension mismatch"):
        multiply_rowmajor(b, b)
    with pytest.raises(ValueError):
        multiply_rowmajor(a, b, "quicksort")


def test_malformed_input_raises_instead_of_faulting():
    a = CsrMatrix(2, 3, np.array([0, 2, 1], np.uint64), np.array([0, 1], np.uint64),
                  np.array([1.0, 2.0]))
    b = CsrMatrix(3, 3, np.array([0, 1, 2, 3], np.uint64), np.array([0, 1, 2], np.uint64),
                  np.ones(3))
    with pytest.raises(ValueError, match="row_ptr"):
        multiply_rowmajor(a, b)
    a2 = CsrMatrix(1, 3, np.array([0, 1], np.uint64), np.array([7], np.uint64), np.ones(1))
    with pytest.raises(ValueError):
        multiply_rowmajor(a2, b)


def _rand_csr(rng, rows, cols, per_row_max, values="uniform", min_len=0):
    lens = rng.integers(min_len, per_row_max + 1, size=rows)
    lens = np.minimum(lens, cols)
    rp = np.zeros(rows + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    ci = np.empty(int(rp[-1]), np.uint64)
    for r in range(rows):
        picked = np.unique(rng.integers(0, cols, size=lens[r]))
        while picked.size < lens[r]:
            picked = np.unique(np.concatenate([picked, rng.integers(0, cols, size=lens[r])]))
        ci[rp[r]:rp[r + 1]] = np.sort(rng.permutation(picked)[:lens[r]])
    n = ci.size
    if values == "uniform":
        v = rng.uniform(-1.0, 1.0, n)
    elif values == "quantized":  # many exact cancellations
        v = rng.choice([-2.0, -1.0, 1.0, 2.0], n)
    else:
        v = rng.uniform(0.1, 1.0, n)
    return CsrMatrix(rows, cols, rp, ci, v)


@pytest.mark.parametrize("seed,shape", [
    (1, (300, 200, 150, 8, 8)),          # short rows
    (2, (400, 300, 500, 20, 20)),        # medium rows (table 256/512)
    (3, (200, 150, 400, 40, 30)),        # medium rows, table 1024
    (4, (60, 2000, 3000, 1500, 6)),      # long rows (k_long)
    (5, (500, 64, 64, 64, 64)),          # collision heavy, dense-ish
    (6, (1000, 3000, 5000, 45, 4)),      # A rows longer than 32, short B rows
    (7, (40, 2000, 300, 300, 30)),       # on-chip long rows, few columns (dup rounds)
    (8, (24, 3000, 60000, 2500, 14)),    # rows past the on-chip limit (global tables)
    (9, (30, 2000, 400, 1500, 40)),      # global tables, heavy duplicates per chunk
    (10, (2000, 3000, 4000, 32, 1)),     # ELL copy of B, wide A rows (generic short path)
    (11, (2000, 3000, 4000, 6, 5)),      # ELL fast path, empty and partial B rows
])
@pytest.mark.parametrize("values", ["uniform", "quantized"])
def test_random_vs_oracle(seed, shape, values):
    rows, inner, cols, amax, bmax = shape
    rng = np.random.default_rng(seed)
    a = _rand_csr(rng, rows, inner, amax, values)
    b = _rand_csr(rng, inner, cols, bmax, values)
    stats = KernelStats()
    c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
    ref = oracle.multiply_rowmajor(a, b, row_choices=True)
    assert_csr_bitwise_equal(c, CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx,
                                          ref.values), f"seed{seed}/{values}")
    assert stats.multiplications == ref.multiplications
    assert np.array_equal(_choices_array(stats, rows), ref.row_choices)


def test_wide_column_keys():
    """Columns beyond 2^22 / 2^27 switch the sort keys to 64 bits."""
    rng = np.random.default_rng(11)
    for cols in (1 << 23, (1 << 28) + 5, 0xFFFF_FFF0):
        a = _rand_csr(rng, 200, 300, 12)
        b = _rand_csr(rng, 300, cols, 40)
        c = multiply_rowmajor(a, b)
        assert_csr_bitwise_equal(c, _oracle_csr(a, b), f"cols={cols}")


def _clustered_operands(rng, rows, inner, entries, blen, cols, far):
    """A rows of `entries` entries over B rows whose columns crowd into
    [0, 2*inner) except a few far columns: long rows whose output columns are
    clustered inside a wide range (big column buckets in extraction)."""
    a_rp = np.arange(rows + 1, dtype=np.uint64) * np.uint64(entries)
    a_ci = np.concatenate([np.sort(rng.choice(inner, entries, replace=False))
                           for _ in range(rows)]).astype(np.uint64)
    a = CsrMatrix(rows, inner, a_rp, a_ci, rng.uniform(-1, 1, a_ci.size))
    b_ci = []
    for k in range(inner):
        c = rng.choice(2 * inner, blen, replace=False)
        if k % far == 0:
            c[0] = cols - 1 - k
        b_ci.append(np.sort(c))
    b_rp = np.arange(inner + 1, dtype=np.uint64) * np.uint64(blen)
    b = CsrMatrix(inner, cols, b_rp, np.concatenate(b_ci).astype(np.uint64),
                  rng.uniform(-1, 1, inner * blen))
    return a, b


@pytest.mark.parametrize("rows,inner,entries,blen", [
    (12, 3000, 1500, 4),     # on-chip long rows (k_long_smem), clustered buckets
    (6, 6000, 4000, 5),      # rows past the on-chip limit (cluster of column parts)
    (3, 20000, 4000, 10),    # one part outgrows its table: handed on to k_long
    (40, 2000, 200, 3),      # warp rows (k_rows)
])
def test_long_rows_clustered_columns(rows, inner, entries, blen):
    rng = np.random.default_rng(rows * 7 + blen)
    a, b = _clustered_operands(rng, rows, inner, entries, blen, 5_000_000, 997)
    stats = KernelStats()
    c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
    ref = oracle.multiply_rowmajor(a, b, row_choices=True)
    assert_csr_bitwise_equal(c, CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx,
                                          ref.values), "clustered")
    assert np.array_equal(_choices_array(stats, rows), ref.row_choices)


def test_row_block_views_concatenate_to_full_product():
    """Row blocks of A as zero-copy device views (row_ptr[0] != 0) multiply to
    the matching row blocks of C (kernels.py:323-329: rows are independent)."""
    import torch

    from paper_1303_1651_b200 import device as dev
    from paper_1303_1651_b200.distributed import concat_row_blocks, partition_rows

    a, b = genmat.gen_zipf(20_000, 3), genmat.gen_zipf(20_000, 4)
    full = _oracle_csr(a, b)
    d = torch.device("cuda", 0)
    ad, bd = dev.DeviceCsr.from_host(a, d), dev.DeviceCsr.from_host(b, d)
    ctx = dev.context_for_current_stream(d)
    bounds = partition_rows(row_products_prefix(a, b), 5)
    blocks = []
    for g in range(5):
        with dev.multiply(ctx, ad.row_block(int(bounds[g]), int(bounds[g + 1])), bd) as p:
            blocks.append(p.download())
    assert_csr_bitwise_equal(concat_row_blocks(blocks, b.cols), full, "row blocks")
    ctx.close()


def test_device_api_and_timings():
    import torch

    from paper_1303_1651_b200 import device as dev

    a = genmat.gen_fd(64)
    d = torch.device("cuda", 0)
    ad = dev.DeviceCsr.from_host(a, d)
    ctx = _lib.Context(0)
    with _lib.multiply_views(ctx, ad.view(), ad.view(), 6, _lib.FLAG_TIMING) as p:
        rp, ci, v = p.download()
        assert p.multiplications == 100104
        t = ctx.last_timings()
        assert "k_fused" in t  # (4096 rows: the count-free prep pass runs inside k_fused)
        assert all(x > 0 for x in t.values())
        assert ctx.last_launch_count() >= 1
        out = dev.product_tensors(p, d)
        assert np.array_equal(out.col_idx.cpu().numpy().view(np.uint64), ci)
    assert_csr_bitwise_equal(CsrMatrix(a.rows, a.cols, rp, ci, v), _oracle_csr(a, a), "fd64")
    ctx.close()


def test_repeated_calls_reuse_context_state():
    """Status-word epochs and pooled buffers across many calls and shapes."""
    cases = [golden_case(n) for n in ("fd_16", "long_rows", "random_5", "medium_rows",
                                      "zero_rows", "signed_k40")]
    for rep in range(3):
        for a, b, c_ref, _, _ in cases:
            assert_csr_bitwise_equal(multiply_rowmajor(a, b), c_ref, f"rep{rep}")


def _config_ops(label):
    if label.startswith("C1"):
        a = genmat.gen_fd(100)
        return a, a
    if label.startswith("C2"):
        a = genmat.gen_fd(int(label[len("C2_fd"):]))
        return a, a
    if label.startswith("C3"):
        return genmat.gen_random_k(2_000_000, 5, 0), genmat.gen_random_k(2_000_000, 5, 1)
    if label.startswith("C4"):
        a = genmat.gen_fd3(100)
        return a, a
    return genmat.gen_zipf(2_000_000, 0), genmat.gen_zipf(2_000_000, 1)


FULL = ["C1_fd100", "C2_fd32", "C2_fd64", "C2_fd128", "C2_fd256", "C2_fd512", "C2_fd1024",
        "C2_fd2048", "C3_random2M", "C4_fd3_100", "C5_zipf2M"]


@pytest.mark.parametrize("label", FULL)
def test_full_size_config_matches_reference(label):
    """Full BASELINE configs against the reference's own product digests."""
    fp = fingerprints().get(label)
    if fp is None:
        pytest.skip(f"{label} missing from fingerprints.json")
    a, b = _config_ops(label)
    stats = KernelStats()
    c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
    assert stats.multiplications == fp["multiplications"]
    d = genmat.digests(c)
    if d["fingerprint"] != fp["c"]["fingerprint"]:
        # localise the failure against the (reference-pinned) oracle
        assert_csr_bitwise_equal(c, _oracle_csr(a, b), label)
    assert d["row_ptr_sha256"] == fp["c"]["row_ptr_sha256"]
    assert d["col_idx_sha256"] == fp["c"]["col_idx_sha256"]
    assert d["values_sha256"] == fp["c"]["values_sha256"]


def _skewed_csr(rng, rows, cols, lmax, values, window=None, far_every=0):
    """Zipf(2) row lengths clipped to [1, lmax] (C5's shape at test size).
    `window`: columns crowd into [0, window) (duplicate-heavy products);
    `far_every`: every n-th row also gets the last column (wide column range
    around a narrow cluster: oversized sort buckets)."""
    lens = np.minimum(rng.zipf(2.0, rows), lmax)
    span = cols if window is None else min(window, cols)
    lens = np.minimum(lens, span - 1)
    rp = np.zeros(rows + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    parts = []
    for r in range(rows):
        c = rng.choice(span - 1, lens[r], replace=False) if lens[r] > 64 else \
            np.unique(rng.integers(0, span - 1, lens[r] * 2))[:lens[r]]
        while c.size < lens[r]:
            c = np.unique(np.concatenate([c, rng.integers(0, span - 1, lens[r])]))[:lens[r]]
        if far_every and r % far_every == 0 and c.size:
            c[-1] = cols - 1
        parts.append(np.sort(c))
    ci = np.concatenate(parts).astype(np.uint64)
    lens = np.array([p.size for p in parts])
    rp[1:] = np.cumsum(lens)
    if values == "quantized":  # exact cancellations and transient zeros
        v = rng.choice([-2.0, -1.0, 1.0, 2.0], ci.size)
    else:
        v = rng.uniform(-1.0, 1.0, ci.size)
    return CsrMatrix(rows, cols, rp, ci, v)


@pytest.mark.parametrize("case", ["random", "dups", "clustered"])
@pytest.mark.parametrize("values", ["uniform", "quantized"])
def test_split_mode_esc_kernels(case, values):
    """Skewed operands (non-short rows a minority): split mode, with the
    expand-sort-compress kernels for rows up to kEscBlockCap products (warp
    rows, block rows with ~32-key buckets, oversized buckets) and the cluster
    variant past it. Bitwise against the oracle, stats included; the ESC
    kernels must actually have run."""
    rng = np.random.default_rng({"random": 1, "dups": 2, "clustered": 3}[case])
    n = 30_000
    if case == "random":
        a = _skewed_csr(rng, n, n, 3000, values)
        b = _skewed_csr(rng, n, 2_000_000, 200, values)
    elif case == "dups":
        a = _skewed_csr(rng, n, n, 3000, values)
        b = _skewed_csr(rng, n, 5000, 200, values, window=3000)
    else:
        a = _skewed_csr(rng, n, n, 3000, values)
        b = _skewed_csr(rng, n, 5_000_000, 100, values, window=4000, far_every=3)
    ref = oracle.multiply_rowmajor(a, b, row_choices=True, threads=8)
    ctx = _lib.Context(0)
    arp, aci, av = a.row_ptr, a.col_idx, a.values
    brp, bci, bv = b.row_ptr, b.col_idx, b.values
    va = _lib.csr_view(a.rows, a.cols, arp, aci, av)
    vb = _lib.csr_view(b.rows, b.cols, brp, bci, bv)
    with _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING | _lib.FLAG_ROW_STATS) as p:
        rp, ci, v = p.download()
        names = set(ctx.last_timings())
        stats = KernelStats()
        from paper_1303_1651_b200.kernels import _record_row_choices
        _record_row_choices(stats, p, StrategyKind, arp)
        mults = p.multiplications
    ctx.close()
    assert {"k_esc_warp", "k_esc_block", "k_esc_plan"} <= names, names
    assert mults == ref.multiplications
    assert_csr_bitwise_equal(CsrMatrix(a.rows, b.cols, rp, ci, v),
                             CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx, ref.values),
                             f"esc/{case}/{values}")
    assert np.array_equal(_choices_array(stats, a.rows), ref.row_choices)


def _dominated_operands(rng, values, window):
    """A: many short rows, a few wider ones; B: one row in 25 is long
    (64..3000 entries; non-short rows of C stay a minority: split mode). So many rows of C are one long B row plus a few other
    products (k_esc_dom), with every tie-break shape: the dominant entry
    first, last and in the middle of its A row, columns shared between the
    dominant row and the others (`window` crowds them), exact cancellations."""
    n = 20_000
    cols = 60_000

    def mk(rows, lens, span):
        rp = np.zeros(rows + 1, np.uint64)
        rp[1:] = np.cumsum(lens)
        parts = [np.sort(rng.choice(span, int(k), replace=False)) for k in lens]
        ci = np.concatenate(parts).astype(np.uint64)
        if values == "quantized":
            v = rng.choice([-2.0, -1.0, 1.0, 2.0], ci.size)
        elif values == "zeros":
            v = rng.choice([0.0, -0.0, 1.0, -1.0], ci.size)
        else:
            v = rng.uniform(-1.0, 1.0, ci.size)
        return rp, ci, v

    lb = np.where(rng.random(n) < 0.04, rng.integers(64, 3000, n), rng.integers(0, 6, n))
    brp, bci, bv = mk(n, lb, window)
    la = np.where(rng.random(n) < 0.03, rng.integers(20, 200, n), rng.integers(0, 5, n))
    arp, aci, av = mk(n, la, n)
    return CsrMatrix(n, n, arp, aci, av), CsrMatrix(n, cols, brp, bci, bv)


@pytest.mark.parametrize("window", [60_000, 4_000])
@pytest.mark.parametrize("values", ["uniform", "quantized", "zeros"])
@pytest.mark.parametrize("with_stats", [False, True])
def test_split_mode_dominant_rows(values, window, with_stats):
    """Rows that are one long B row plus a few other products are merged by
    k_esc_dom (the dominant run streamed from B, the others sorted and merged
    in on the way): bitwise against the oracle, with the reference's row
    choices, and the kernel must actually have run."""
    rng = np.random.default_rng(17)
    a, b = _dominated_operands(rng, values, window)
    ref = oracle.multiply_rowmajor(a, b, row_choices=True, threads=8)
    ctx = _lib.Context(0)
    va, vb = (_lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values),
              _lib.csr_view(b.rows, b.cols, b.row_ptr, b.col_idx, b.values))
    flags = _lib.FLAG_TIMING | (_lib.FLAG_ROW_STATS if with_stats else 0)
    with _lib.multiply_views(ctx, va, vb, 6, flags) as p:
        rp, ci, v = p.download()
        names = set(ctx.last_timings())
        mults = p.multiplications
        if with_stats:
            stats = KernelStats()
            from paper_1303_1651_b200.kernels import _record_row_choices
            _record_row_choices(stats, p, StrategyKind, a.row_ptr)
    ctx.close()
    assert "k_esc_dom" in names, names
    assert mults == ref.multiplications
    assert_csr_bitwise_equal(CsrMatrix(a.rows, b.cols, rp, ci, v),
                             CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx, ref.values),
                             f"dom/{values}/{window}")
    if with_stats:
        assert np.array_equal(_choices_array(stats, a.rows), ref.row_choices)


def test_dominant_row_with_unsorted_b_row_is_redone():
    """k_esc_dom merges its dominant B row as it is stored. Ascending columns
    are the storage contract (formats.py:40-46), but the reference's kernel
    sorts whatever it is given and so do the other kernels: a B row whose
    columns do not ascend is reported by k_esc_dom and the product redone
    without it — the reference's bytes either way."""
    rng = np.random.default_rng(23)
    a, b = _dominated_operands(rng, "quantized", 60_000)
    bci = b.col_idx.copy()
    lens = np.diff(b.row_ptr.astype(np.int64))
    for r in np.flatnonzero(lens >= 64)[:50]:  # swap two entries' columns inside long rows
        s = int(b.row_ptr[r])
        bci[s + 3], bci[s + 40] = bci[s + 40], bci[s + 3]
    b2 = CsrMatrix(b.rows, b.cols, b.row_ptr.copy(), bci, b.values.copy())
    ref = oracle.multiply_rowmajor(a, b2, threads=8)
    ctx = _lib.Context(0)
    va, vb = (_lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values),
              _lib.csr_view(b2.rows, b2.cols, b2.row_ptr, b2.col_idx, b2.values))
    with _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING) as p:
        rp, ci, v = p.download()
        names = set(ctx.last_timings())
    ctx.close()
    assert "k_esc_dom" not in names, names  # (the timings are the redo's)
    assert_csr_bitwise_equal(CsrMatrix(a.rows, b2.cols, rp, ci, v),
                             CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx, ref.values),
                             "dom/unsorted")


def _host_views(a, b):
    return (_lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values),
            _lib.csr_view(b.rows, b.cols, b.row_ptr, b.col_idx, b.values))


@pytest.mark.parametrize("blocks", [1, 3, 8, 16])
def test_pipelined_host_product_matches_oracle(blocks):
    """spmmm_multiply_host (row blocks: values up, compute, C down, overlapped)
    gives the bytes of the one-shot path: A·A (blocks wait for the B rows they
    read), A·B, skewed rows (split mode per block), empty rows, empty A."""
    rng = np.random.default_rng(blocks)
    fd = genmat.gen_fd(200)
    z = genmat.gen_zipf(30_000, 5)
    rect_a = _rand_csr(rng, 700, 300, 12, "quantized")
    rect_b = _rand_csr(rng, 300, 900, 10, "quantized")
    zero_a = CsrMatrix(50, 300, np.zeros(51, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    no_rows = CsrMatrix(0, 300, np.zeros(1, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    # empty rows around the block boundaries
    gap_rp = np.array(rect_a.row_ptr, dtype=np.uint64).copy()
    lens = np.diff(gap_rp.astype(np.int64))
    lens[100:400] = 0
    gap_ci = np.concatenate([np.asarray(rect_a.col_idx)[int(gap_rp[r]):int(gap_rp[r + 1])]
                             for r in range(rect_a.rows) if lens[r]]).astype(np.uint64)
    gap_v = np.concatenate([np.asarray(rect_a.values)[int(gap_rp[r]):int(gap_rp[r + 1])]
                            for r in range(rect_a.rows) if lens[r]])
    gap_rp2 = np.zeros(rect_a.rows + 1, np.uint64)
    gap_rp2[1:] = np.cumsum(lens)
    gap_a = CsrMatrix(rect_a.rows, rect_a.cols, gap_rp2, gap_ci, gap_v)
    ctx = _lib.Context(0)
    for name, a, b in [("fd200^2", fd, fd), ("zipf", z, genmat.gen_zipf(30_000, 6)),
                       ("rect", rect_a, rect_b), ("zero", zero_a, rect_b),
                       ("no rows", no_rows, rect_b), ("gaps", gap_a, rect_b),
                       ("zipf^2", z, z)]:
        va, vb = _host_views(a, b)
        if b is a:
            vb = va
        rp, ci, v, mults = _lib.multiply_host(ctx, va, vb, 6, 0, blocks)
        ref = oracle.multiply_rowmajor(a, b, threads=8)
        assert mults == ref.multiplications, name
        assert_csr_bitwise_equal(CsrMatrix(a.rows, b.cols, rp, ci, v),
                                 CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx,
                                           ref.values), f"pipelined/{name}/{blocks}")
    ctx.close()


def test_pipelined_host_product_errors():
    ctx = _lib.Context(0)
    b = CsrMatrix(3, 3, np.array([0, 1, 2, 3], np.uint64), np.array([0, 1, 2], np.uint64),
                  np.ones(3))
    bad_rp = CsrMatrix(2, 3, np.array([0, 2, 1], np.uint64), np.array([0, 1], np.uint64),
                       np.array([1.0, 2.0]))
    bad_col = CsrMatrix(1, 3, np.array([0, 1], np.uint64), np.array([7], np.uint64), np.ones(1))
    past = CsrMatrix(1, 3, np.array([0, 5], np.uint64), np.array([0, 1], np.uint64), np.ones(2))
    for a, what in [(bad_rp, "row_ptr"), (bad_col, "col_idx"), (past, "row_ptr")]:
        va, vb = _host_views(a, b)
        with pytest.raises(ValueError, match=what):
            _lib.multiply_host(ctx, va, vb, 6, 0, 2)
    va, vb = _host_views(b, bad_rp)
    with pytest.raises(ValueError, match="dimension mismatch"):
        _lib.multiply_host(ctx, va, vb, 6, 0, 2)
    # the context stays usable after errors
    va, vb = _host_views(b, b)
    rp, ci, v, m = _lib.multiply_host(ctx, va, vb, 6, 0, 2)
    assert m == 3 and list(ci) == [0, 1, 2]
    ctx.close()


@pytest.mark.parametrize("label", ["C2_fd2048", "C3_random2M", "C4_fd3_100", "C5_zipf2M"])
def test_full_size_drop_in_without_stats_matches_reference(label):
    """The drop-in without stats takes the pipelined host path at these sizes."""
    from paper_1303_1651_b200 import kernels as km

    fp = fingerprints().get(label)
    if fp is None:
        pytest.skip(f"{label} missing from fingerprints.json")
    a, b = _config_ops(label)
    assert len(a.values) >= km.PIPELINE_MIN_NNZ
    c = multiply_rowmajor(a, b)
    d = genmat.digests(c)
    assert d["row_ptr_sha256"] == fp["c"]["row_ptr_sha256"]
    assert d["col_idx_sha256"] == fp["c"]["col_idx_sha256"]
    assert d["values_sha256"] == fp["c"]["values_sha256"]


def test_drop_in_pipelined_path_equals_stats_path():
    """Without stats, large operands take spmmm_multiply_host (u32 column
    indices down, widened on the host); with stats, the one-shot path. Same
    bytes, and both match the oracle (A·A stencil and skewed A·B)."""
    from paper_1303_1651_b200 import _lib as L
    from paper_1303_1651_b200 import kernels as km

    cases = [("fd1024^2", genmat.gen_fd(1024), None),
             ("zipf800k", genmat.gen_zipf(800_000, 7), genmat.gen_zipf(800_000, 8))]
    for name, a, b in cases:
        b = a if b is None else b
        assert len(a.values) >= km.PIPELINE_MIN_NNZ, name
        L.last_transfer = None
        c_fast = multiply_rowmajor(a, b)
        if len(a.values) >= km.PIPELINE_MIN_NNZ:
            assert L.last_transfer is not None, name
            assert L.last_transfer["d2h_bytes"] < 8 * (a.rows + 1) + 16 * len(c_fast.values)
        stats = KernelStats()
        c_stats = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
        assert_csr_bitwise_equal(c_fast, c_stats, name)
        assert_csr_bitwise_equal(c_fast, _oracle_csr(a, b), name)


def test_pipelined_host_product_reservation_overflow(monkeypatch):
    """The pipelined path reserves max(8 nnz(A), 2^20) result entries; a
    result past the reservation is redone in one shot — same bytes. Forced
    here with a tiny reservation (SPMMM_PIPE_CAP, read per call)."""
    monkeypatch.setenv("SPMMM_PIPE_CAP", "1000")
    ctx = _lib.Context(0)
    for name, a, b in [("fd200^2", genmat.gen_fd(200), None),
                       ("zipf", genmat.gen_zipf(30_000, 5), genmat.gen_zipf(30_000, 6))]:
        b = a if b is None else b
        va, vb = _host_views(a, b)
        if b is a:
            vb = va
        rp, ci, v, mults = _lib.multiply_host(ctx, va, vb, 6, 0, 8)
        ref = oracle.multiply_rowmajor(a, b, threads=8)
        assert mults == ref.multiplications, name
        assert_csr_bitwise_equal(CsrMatrix(a.rows, b.cols, rp, ci, v),
                                 CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx,
                                           ref.values), f"overflow/{name}")
    ctx.close()


@pytest.mark.parametrize("values", ["uniform", "quantized"])
def test_split_mode_hash_kernels_past_esc_key_range(values):
    """Columns past 2^23 do not fit ESC's 32-bit sort keys: split mode then
    runs the hash-table kernels (k_rows, k_long_smem and its cluster variant,
    k_long). Bitwise against the oracle, stats included."""
    rng = np.random.default_rng(11)
    n = 30_000
    a = _skewed_csr(rng, n, n, 3000, values)
    b = _skewed_csr(rng, n, 9_000_000, 200, values)
    ref = oracle.multiply_rowmajor(a, b, row_choices=True, threads=8)
    ctx = _lib.Context(0)
    va = _lib.csr_view(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
    vb = _lib.csr_view(b.rows, b.cols, b.row_ptr, b.col_idx, b.values)
    with _lib.multiply_views(ctx, va, vb, 6, _lib.FLAG_TIMING | _lib.FLAG_ROW_STATS) as p:
        rp, ci, v = p.download()
        names = set(ctx.last_timings())
        stats = KernelStats()
        from paper_1303_1651_b200.kernels import _record_row_choices
        _record_row_choices(stats, p, StrategyKind, a.row_ptr)
    ctx.close()
    assert "k_rows" in names and "k_esc_warp" not in names, names
    assert_csr_bitwise_equal(CsrMatrix(a.rows, b.cols, rp, ci, v),
                             CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx, ref.values),
                             f"hash/{values}")
    assert np.array_equal(_choices_array(stats, a.rows), ref.row_choices)


def _banded_then_random(n=200_000, seed=3):
    """Top half: tridiagonal rows (C rows span a few columns: u16 deltas);
    bottom half: 4 random columns over n > 2^16 (u32 fallback)."""
    rng = np.random.default_rng(seed)
    rows = []
    for r in range(n // 2):
        rows.append(np.array([c for c in (r - 1, r, r + 1) if 0 <= c < n]))
    for _ in range(n - n // 2):
        rows.append(np.sort(rng.choice(n, 4, replace=False)))
    lens = np.array([len(x) for x in rows])
    rp = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate(rows).astype(np.uint64)
    v = rng.integers(-3, 4, ci.size).astype(np.float64)
    return CsrMatrix(n, n, rp, ci, v)


@pytest.mark.parametrize("no_delta", [False, True])
def test_pipelined_mixed_u16_and_u32_blocks(no_delta):
    """One product whose first row blocks go down as u16 column deltas and
    whose last blocks fall back to u32 (the cb_next / blk_cb bookkeeping
    across mixed blocks), bitwise against the oracle; and the same with the
    deltas off (SPMMM_NO_DELTA16, read once per process: a subprocess)."""
    import os
    import subprocess
    import sys

    if no_delta:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        code = ("import sys; sys.path[:0] = ['.', 'oracle', 'tests']\n"
                "import test_gpu_parity as t\n"
                "t.test_pipelined_mixed_u16_and_u32_blocks(False)\n")
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                           env=dict(os.environ, SPMMM_NO_DELTA16="1"), timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return
    a = _banded_then_random()
    ref = oracle.multiply_rowmajor(a, a, threads=8)
    ctx = _lib.Context(0)
    va, _ = _host_views(a, a)
    for blocks in (4, 8, 13):
        rp, ci, v, mults = _lib.multiply_host(ctx, va, va, 6, 0, blocks)
        assert mults == ref.multiplications
        assert_csr_bitwise_equal(CsrMatrix(a.rows, a.cols, rp, ci, v),
                                 CsrMatrix(ref.rows, ref.cols, ref.row_ptr, ref.col_idx,
                                           ref.values), f"mixed/{blocks}")
        # fewer bytes than u32 indices for all of C: some blocks went as u16
        d2h = _lib.last_transfer["d2h_bytes"]
        if os.environ.get("SPMMM_NO_DELTA16") is None:
            assert d2h < 4 * (a.rows + 1) + 12 * len(v), (blocks, d2h)
    ctx.close()


@pytest.mark.parametrize("family,grids", [("fd", [1, 2, 3, 7, 64, 100, 1000]),
                                          ("fd3", [1, 2, 3, 5, 17, 100])])
def test_device_stencil_generators_match_host(family, grids):
    """spmmm_gen_fd_device / spmmm_gen_fd3_device write the bytes of the host
    generators (gen_fd restates the reference's genmat.py:79-103) into HBM."""
    for g in grids:
        host = genmat.gen_fd(g) if family == "fd" else genmat.gen_fd3(g)
        dev = genmat.gen_stencil_device(family, g).to_host()
        assert dev.row_ptr.tobytes() == np.asarray(host.row_ptr).tobytes(), (family, g)
        assert dev.col_idx.tobytes() == np.asarray(host.col_idx).tobytes(), (family, g)
        assert dev.values.tobytes() == np.asarray(host.values).tobytes(), (family, g)
