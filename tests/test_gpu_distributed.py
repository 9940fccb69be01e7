"""The multi-GPU path with the CUDA library as the per-rank product.

Only one GPU is available to these tests, so the ranks share cuda:0 and talk
over gloo (host-side collectives: no kernel waits on another rank's kernel).
Everything else is the product path of `bench.py --gpus N`: shared-memory
operands, chunked upload + all-gather, the device partition
(spmmm_partition_rows), each rank's block through libspmmm, the nnz
all-gather and every rank downloading its slice of the shared, page-locked
result (spmmm_product_download_offset). Checked against the reference's
own outputs: golden cases byte for byte, C3 and C5 by the sha256 digests of
the reference's full-size products."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import ROOT, fingerprints, golden_case, golden_names
from paper_1303_1651_b200.launch import spawn

pytestmark = pytest.mark.gpu
WORKER = os.path.join(ROOT, "tests", "dist_worker.py")


def _run(nproc, *args, timeout=600):
    r = spawn(nproc, WORKER, list(args) + ["--device", "cuda:0"], timeout=timeout, capture=True)
    assert r.returncode == 0, f"ranks failed:\n{r.stdout[-3000:]}\n{r.stderr[-6000:]}"


def test_device_partition_matches_host_partition():
    import oracle
    from paper_1303_1651_b200 import _lib
    from paper_1303_1651_b200.distributed import partition_rows
    from paper_1303_1651_b200.formats import csr_arrays

    ctx = _lib.Context(0)
    rng = np.random.default_rng(5)
    names = golden_names()
    for name in [names[i] for i in rng.choice(len(names), 40, replace=False)] + ["long_rows"]:
        a, b, _, mults, _ = golden_case(name)
        prefix = np.zeros(a.rows + 1, np.uint64)
        np.cumsum(oracle.row_products(a, b), out=prefix[1:])
        va = _lib.csr_view(a.rows, a.cols, *csr_arrays(a))
        vb = _lib.csr_view(b.rows, b.cols, *csr_arrays(b))
        for parts in (1, 2, 3, 5, 8, 64):
            bounds, total = _lib.partition_rows(ctx, va, vb, parts)
            assert total == mults, name
            assert bounds.tolist() == partition_rows(prefix, parts).tolist(), (name, parts)
    ctx.close()


def test_device_partition_large_skewed():
    """Past one scan chunk (4096 rows) and past 4096 chunks (chunk doubling)."""
    import oracle
    from paper_1303_1651_b200 import _lib, genmat
    from paper_1303_1651_b200.distributed import partition_rows
    from paper_1303_1651_b200.formats import csr_arrays

    ctx = _lib.Context(0)
    for a, b in ((genmat.gen_zipf(300_000, 0), genmat.gen_zipf(300_000, 1)),
                 (genmat.gen_fd(4096), None)):
        b = a if b is None else b
        prefix = np.zeros(a.rows + 1, np.uint64)
        np.cumsum(oracle.row_products(a, b), out=prefix[1:])
        va = _lib.csr_view(a.rows, a.cols, *csr_arrays(a))
        vb = _lib.csr_view(b.rows, b.cols, *csr_arrays(b))
        for parts in (2, 7, 8, 64):
            bounds, total = _lib.partition_rows(ctx, va, vb, parts)
            assert total == int(prefix[-1])
            assert bounds.tolist() == partition_rows(prefix, parts).tolist(), parts
    ctx.close()


@pytest.mark.parametrize("case,world", [("signed_k40", 2), ("long_rows", 3), ("fd_16", 2),
                                        ("empty_rows_mix", 3), ("transient_zero", 2),
                                        ("rect_7x13_13x5", 2)])
def test_ranks_on_gpu_equal_reference(case, world, tmp_path):
    out = str(tmp_path / "c.npz")
    _run(world, "--case", case, "--out", out, "--stats", "--calls", "3")
    r = np.load(out)
    _, _, c_ref, mults, choices = golden_case(case)
    assert r["rp"].tobytes() == c_ref.row_ptr.tobytes()
    assert r["ci"].tobytes() == c_ref.col_idx.tobytes()
    assert r["v"].tobytes() == c_ref.values.tobytes()
    assert int(r["mults"][0]) == mults
    assert np.array_equal(r["choices"], choices)


@pytest.mark.parametrize("expect", ["mismatch", "malformed"])
def test_gpu_errors_raise_on_every_rank(expect, tmp_path):
    out = str(tmp_path / "err")
    _run(2, "--case", "fd_16", "--out", out, "--expect", expect)
    msgs = [open(f"{out}.rank{r}").read() for r in range(2)]
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("label,config", [("C3_random2M", "C3"), ("C5_zipf2M", "C5")])
def test_full_size_two_ranks_match_reference_digests(label, config, tmp_path):
    fp = fingerprints().get(label)
    if fp is None:
        pytest.skip(f"{label} missing from fingerprints.json")
    out = str(tmp_path / "d.json")
    _run(2, "--config", config, "--out", out, timeout=900)
    d = json.load(open(out))
    assert d["nnz"] == fp["c"]["nnz"]
    assert d["digests"]["row_ptr"] == fp["c"]["row_ptr_sha256"]
    assert d["digests"]["col_idx"] == fp["c"]["col_idx_sha256"]
    assert d["digests"]["values"] == fp["c"]["values_sha256"]
    b = d["bounds"]
    assert b[0] == 0 and 0 < b[1] < b[2]


@pytest.mark.parametrize("case", ["signed_k40", "long_rows", "empty_rows_mix"])
def test_nccl_path_one_rank(case, tmp_path):
    """The NCCL code path (chunked upload + all_gather_into_tensor, the gloo
    control group beside it, the shared result) with the one rank a single
    GPU allows: NCCL refuses two ranks on one device."""
    out = str(tmp_path / "c.npz")
    r = spawn(1, WORKER, ["--case", case, "--out", out, "--stats", "--calls", "2", "--device",
                          "cuda:0", "--backend", "nccl"], timeout=600, capture=True)
    assert r.returncode == 0, f"{r.stdout[-3000:]}\n{r.stderr[-6000:]}"
    z = np.load(out)
    _, _, c_ref, mults, choices = golden_case(case)
    assert z["rp"].tobytes() == c_ref.row_ptr.tobytes()
    assert z["ci"].tobytes() == c_ref.col_idx.tobytes()
    assert z["v"].tobytes() == c_ref.values.tobytes()
    assert int(z["mults"][0]) == mults and np.array_equal(z["choices"], choices)


def test_bench_distributed_path_nccl_one_rank():
    """bench.py's N-GPU path under torch.distributed.run with NCCL, one rank."""
    import json
    import subprocess
    import sys

    from paper_1303_1651_b200.launch import torchrun_argv

    r = subprocess.run(torchrun_argv(1, os.path.join(ROOT, "bench.py"),
                                     ["--distributed", "--config", "C3", "--steps", "3",
                                      "--warmup", "3", "--e2e-steps", "2"]),
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    # stdout is rank 0's one JSON line (NCCL's log goes to stderr)
    assert len(r.stdout.strip().splitlines()) == 1, r.stdout[:2000]
    line = json.loads(r.stdout)
    assert line["n_gpus"] == 1 and line["value"] > 0 and "nccl" in line["parallelism"]
    assert line["e2e"]["value"] > 0 and line["b_allgather_ms"] > 0
    assert sum(line["rank_products"]) == line["config"]["products"]
    assert "NCCL INFO" in r.stderr  # NCCL_DEBUG=INFO stays on
