"""Harness integration: the B200 grid cells follow the
reference harness's protocol and CSV contract (bench.py:97-142, 144-150,
252-299). Where the reference package is importable (the build container),
its own functions are the oracle for the protocol pieces."""

from __future__ import annotations

import os
import sys

import pytest

from conftest import have_gpu
from paper_1303_1651_b200 import harness

REF_SRC = "/root/reference/pkg/src"


def _ref_bench():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, REF_SRC)
    try:
        import sparsemm.bench as rb
    finally:
        sys.path.remove(REF_SRC)
    return rb


@pytest.mark.parametrize("text", ["64:1024:x2", "64,128,256", "10:1000:x3.5", "1:1:x2",
                                  "100:4194304:x4"])
def test_parse_sizes_matches_reference(text):
    rb = _ref_bench()
    assert harness.parse_sizes(text) == rb.parse_sizes(text)


@pytest.mark.parametrize("bad", ["64:32:x2", "64:128:+2", "0:10:x2", "4:8:x1"])
def test_parse_sizes_rejects(bad):
    with pytest.raises(ValueError):
        harness.parse_sizes(bad)


def test_virtual_clock_protocol_matches_reference(monkeypatch):
    rb = _ref_bench()
    monkeypatch.setenv(harness.CLOCK_OVERRIDE_ENV, "0.3")
    ours = harness.time_kernel(lambda: None, 1000, min_total_seconds=2.0, trials=3)
    ref = rb.time_kernel(lambda: None, 1000, min_total_seconds=2.0, trials=3)
    assert (ours.inner_iters, ours.best_seconds, ours.mflops) == \
        (ref.inner_iters, ref.best_seconds, ref.mflops)
    assert ours.inner_iters == 8


def test_labels_and_csv_match_reference():
    rb = _ref_bench()
    from sparsemm.genmat import GenSpec

    for fam, n, k, fill in (("fd", 4096, 5, 0.001), ("random", 100, 7, 0.001),
                            ("fill", 5000, 5, 0.0025)):
        assert harness.case_label(fam, n, k, fill) == rb._case_label(
            fam, GenSpec(family=fam, n=n, k=k, fill=fill), n)
    recs = [harness.BenchRecord("fd[n=4096]", "fd", 4096, "b200", "combined", 0, 64,
                                1.234567e-4, 12.3456789),
            harness.BenchRecord("random[n=100;k=7]", "random", 100, "b200-device", "sort",
                                3, 1, 2.5e-6, 0.5)]
    ref_recs = [rb.BenchRecord(**r.__dict__) for r in recs]
    assert harness.emit_csv(recs) == rb.emit_csv(ref_recs)
    assert harness.parse_csv(rb.emit_csv(ref_recs)) == [
        harness.BenchRecord(**r.__dict__) for r in rb.parse_csv(rb.emit_csv(ref_recs))]


def test_csv_round_trip_and_header():
    recs = [harness.BenchRecord("fill[n=10;fill=0.5]", "fill", 10, "b200-mixed", "minmax", 1,
                                2, 3.0e-3, 7.0)]
    text = harness.emit_csv(recs)
    assert text.splitlines()[0] == harness.CSV_HEADER
    back = harness.parse_csv(text)
    assert back[0].case == recs[0].case and back[0].inner_iters == 2
    with pytest.raises(ValueError):
        harness.parse_csv("bad,header\n")


def test_operands_follow_reference_generators():
    rb = _ref_bench()
    from sparsemm.genmat import GenSpec, generate

    for fam, n in (("fd", 50), ("random", 40), ("fill", 300)):
        a, b, _ = harness.operands(fam, n, 7, k=5, fill=0.01)
        ra = generate(GenSpec(family=fam, n=n, k=min(5, n), fill=0.01, seed=7))
        assert a.row_ptr.tobytes() == ra.row_ptr.tobytes()
        assert a.col_idx.tobytes() == ra.col_idx.tobytes()
        assert a.values.tobytes() == ra.values.tobytes()


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
def test_gpu_grid_cells_verify_and_emit():
    from paper_1303_1651_b200.kernels import StrategyKind

    res = harness.run_grid(["fd", "random", "fill"], list(harness.KERNEL_NAMES),
                           [StrategyKind.COMBINED, StrategyKind.SORT], [64, 300], 0,
                           fill=0.02, verify=True, min_total_seconds=0.01, trials=2)
    assert not res.skipped
    assert len(res.records) == 3 * 2 * len(harness.KERNEL_NAMES) * 2
    assert all(r.mflops > 0 and r.inner_iters >= 1 for r in res.records)
    back = harness.parse_csv(harness.emit_csv(res.records))
    assert [r.kernel for r in back] == [r.kernel for r in res.records]
    res = harness.run_grid(["fd"], ["b200", "nope"], [None, StrategyKind.COMBINED], [16], 0,
                           min_total_seconds=0.01, trials=1)
    assert {s.reason for s in res.skipped} == {"unknown kernel",
                                               "kernel requires a storing strategy"}
