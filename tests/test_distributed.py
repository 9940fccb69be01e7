"""The multi-GPU orchestration (distributed.multiply_distributed) with
world_size 2 and 3 on CPU over gloo, launched exactly as `bench.py --gpus N`
launches it (paper_1303_1651_b200.launch: torch.distributed.run, rendezvous
on 127.0.0.1): operands shared through node-wide shared memory, each rank
uploading 1/G and all-gathering the rest, product-balanced partition, per-rank
products, nnz all-gather, each rank writing its slice of one shared result.
The per-rank product is injected (the CPU oracle stands in for the GPU
library, which needs a device); the result must equal the reference's bytes.
Error paths: every rank raises the same ValueError (no rank hangs)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import ROOT, golden_case
from paper_1303_1651_b200.launch import spawn

WORKER = os.path.join(ROOT, "tests", "dist_worker.py")


def _run(nproc, *args, timeout=240):
    r = spawn(nproc, WORKER, args, timeout=timeout, capture=True)
    assert r.returncode == 0, f"ranks failed:\n{r.stdout[-3000:]}\n{r.stderr[-6000:]}"
    return r


@pytest.mark.parametrize("case,world", [("signed_k40", 2), ("long_rows", 2), ("fd_16", 3),
                                        ("empty_rows_mix", 2), ("rect_7x13_13x5", 3),
                                        ("hand_2x2", 3)])
def test_ranks_product_equals_reference(case, world, tmp_path):
    out = str(tmp_path / "c.npz")
    _run(world, "--case", case, "--out", out, "--stats", "--calls", "2")
    r = np.load(out)
    _, _, c_ref, mults, choices = golden_case(case)
    assert tuple(r["shape"]) == (c_ref.rows, c_ref.cols)
    assert r["rp"].tobytes() == c_ref.row_ptr.tobytes()
    assert r["ci"].tobytes() == c_ref.col_idx.tobytes()
    assert r["v"].tobytes() == c_ref.values.tobytes()
    assert int(r["mults"][0]) == mults
    assert np.array_equal(r["choices"], choices)
    assert len(r["bounds"]) == world + 1 and r["bounds"][0] == 0 and r["bounds"][-1] == c_ref.rows


@pytest.mark.parametrize("expect", ["mismatch", "malformed"])
def test_errors_raise_on_every_rank(expect, tmp_path):
    out = str(tmp_path / "err")
    _run(2, "--case", "fd_16", "--out", out, "--expect", expect)
    msgs = [open(f"{out}.rank{r}").read() for r in range(2)]
    assert msgs[0] == msgs[1]
    if expect == "mismatch":
        assert msgs[0].startswith("dimension mismatch")
