"""The multi-GPU orchestration (distributed.multiply_distributed) with
world_size 2 on CPU over gloo: partition on the root, B broadcast, A row
blocks scattered, per-rank products, nnz all_gather, blocks gathered and
offset on the root. The per-rank product is injected (the CPU oracle stands
in for the GPU library, which needs a device); the result must equal the
single-process product byte for byte."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local(a_blk, b):
    import torch

    import oracle
    from paper_1303_1651_b200.device import DeviceCsr
    from paper_1303_1651_b200.formats import CsrMatrix

    a = CsrMatrix(a_blk.rows, a_blk.cols, a_blk.row_ptr.numpy().view(np.uint64).copy(),
                  a_blk.col_idx.numpy().view(np.uint64).copy(), a_blk.values.numpy().copy())
    bb = CsrMatrix(b.rows, b.cols, b.row_ptr.numpy().view(np.uint64).copy(),
                   b.col_idx.numpy().view(np.uint64).copy(), b.values.numpy().copy())
    r = oracle.multiply_rowmajor(a, bb)
    return DeviceCsr(r.rows, r.cols, torch.from_numpy(r.row_ptr.view(np.int64).copy()),
                     torch.from_numpy(r.col_idx.view(np.int64).copy()),
                     torch.from_numpy(r.values.copy()))


def _oracle_prefix(a, b):
    import oracle

    p = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=p[1:])
    return p


def _worker(rank, world, port, case, result_path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    from conftest import golden_case
    from paper_1303_1651_b200.distributed import multiply_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = b = None
        if rank == 0:
            a, b, _, _, _ = golden_case(case)
        c = multiply_distributed(a, b, local_multiply=_oracle_local, prefix_fn=_oracle_prefix)
        if rank == 0:
            np.savez(result_path, rp=c.row_ptr, ci=c.col_idx, v=c.values,
                     shape=np.array([c.rows, c.cols]))
        else:
            assert c is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["signed_k40", "long_rows", "fd_16", "empty_rows_mix",
                                  "rect_7x13_13x5"])
def test_two_rank_product_equals_single_process(case, tmp_path):
    from conftest import golden_case

    out = str(tmp_path / "c.npz")
    mp.start_processes(_worker, args=(2, _free_port(), case, out), nprocs=2, join=True,
                       start_method="spawn")
    r = np.load(out)
    _, _, c_ref, _, _ = golden_case(case)
    assert tuple(r["shape"]) == (c_ref.rows, c_ref.cols)
    assert r["rp"].tobytes() == c_ref.row_ptr.tobytes()
    assert r["ci"].tobytes() == c_ref.col_idx.tobytes()
    assert r["v"].tobytes() == c_ref.values.tobytes()
