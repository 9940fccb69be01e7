"""Multi-GPU C = A·B by row blocks.

Rows of C are independent (each depends on its A row and all of B:
kernels.py:323-329), so the path shards without any data-path collective:

1. partition  — the root runs the GPU count pass on A, and `partition_rows`
   cuts A into G contiguous row blocks of ~equal *product* count (not row
   count: C5's rows range from 1 to ~40K products);
2. replicate B — `broadcast` of B's three arrays from the root (NCCL over
   NVLink on the GPU box);
3. scatter A — each rank receives its row block (point-to-point);
4. compute   — each rank runs libspmmm on its block: a standalone CSR block;
5. gather    — `all_gather` of the per-block nnz (8 B per rank), then each
   block's arrays go to the root, which offsets the row pointers.

One process per GPU; torch.distributed (nccl, or gloo for the CPU tests) is
the plumbing. `local_multiply` / `prefix_fn` are injectable so the same
orchestration is exercised on CPU with world_size 2 (tests/test_distributed.py).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .device import DeviceCsr
from .formats import CsrMatrix, csr_arrays


def partition_rows(prefix, parts: int) -> np.ndarray:
    """Row bounds (parts+1) splitting rows so that block g holds the rows whose
    product prefix lies in [g*T/G, (g+1)*T/G): bounds[g] = lower_bound(prefix,
    g*T/G). `prefix` is the exclusive prefix of per-row products (rows+1
    entries, prefix[0] = 0). Rows are never split."""
    prefix = np.asarray(prefix, dtype=np.uint64)
    if parts < 1:
        raise ValueError("need at least one part")
    rows = prefix.size - 1
    total = int(prefix[-1]) if rows >= 0 else 0
    targets = np.array([(total * g) // parts for g in range(parts + 1)], dtype=np.uint64)
    bounds = np.searchsorted(prefix, targets, side="left").astype(np.int64)
    bounds[0] = 0
    bounds[-1] = rows
    return np.maximum.accumulate(np.minimum(bounds, rows))


def row_block_host(m, r0: int, r1: int) -> CsrMatrix:
    rp, ci, v = csr_arrays(m)
    lo, hi = int(rp[r0]), int(rp[r1])
    return CsrMatrix(r1 - r0, m.cols, (rp[r0:r1 + 1] - rp[r0]).astype(np.uint64),
                     ci[lo:hi].copy(), v[lo:hi].copy())


def concat_row_blocks(blocks, cols: int) -> CsrMatrix:
    """Stack CSR row blocks (host arrays, each row_ptr starting at 0)."""
    rows = sum(int(rp.size) - 1 for rp, _, _ in blocks)
    nnz = sum(int(ci.size) for _, ci, _ in blocks)
    out_rp = np.zeros(rows + 1, np.uint64)
    out_ci = np.empty(nnz, np.uint64)
    out_v = np.empty(nnz, np.float64)
    r = 0
    e = 0
    for rp, ci, v in blocks:
        n = int(rp.size) - 1
        out_rp[r + 1:r + n + 1] = rp[1:] + np.uint64(e)
        out_ci[e:e + ci.size] = ci
        out_v[e:e + v.size] = v
        r += n
        e += ci.size
    return CsrMatrix(rows, cols, out_rp, out_ci, out_v)


def _gpu_local_multiply(a_blk: DeviceCsr, b: DeviceCsr):
    from . import device as dev_mod

    ctx = dev_mod.context_for_current_stream(b.values.device)
    with dev_mod.multiply(ctx, a_blk, b) as prod:
        out = dev_mod.product_tensors(prod, b.values.device)
    ctx.close()
    return out


def _gpu_prefix(a, b):
    from .kernels import row_products_prefix

    return row_products_prefix(a, b)


def _send(t, dst, group):
    if t.numel():
        dist.send(t, dst, group=group)


def _recv(t, src, group):
    if t.numel():
        dist.recv(t, src, group=group)


def multiply_distributed(a, b, *, group=None, device=None, root: int = 0,
                         local_multiply=None, prefix_fn=None, timings: dict | None = None):
    """C = A·B over all ranks of `group`. The root passes host CSR `a` and `b`
    (other ranks pass None) and gets the host CsrMatrix back; other ranks get
    None. `device`: where this rank's tensors live (cuda:LOCAL_RANK for nccl,
    cpu for gloo)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if device is None:
        device = torch.device("cpu") if dist.get_backend(group) == "gloo" else \
            torch.device("cuda", torch.cuda.current_device())
    local_multiply = local_multiply or _gpu_local_multiply
    prefix_fn = prefix_fn or _gpu_prefix
    i64 = dict(dtype=torch.int64, device=device)

    # shapes + partition
    meta = torch.zeros(6 + world + 1, **i64)
    if rank == root:
        if a.cols != b.rows:
            raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
        bounds = partition_rows(prefix_fn(a, b), world)
        meta[:6] = torch.tensor([a.rows, a.cols, len(a.values), b.rows, b.cols, len(b.values)])
        meta[6:] = torch.from_numpy(bounds)
    dist.broadcast(meta, root, group=group)
    a_rows, a_cols, a_nnz, b_rows, b_cols, b_nnz = (int(x) for x in meta[:6].tolist())
    bounds = [int(x) for x in meta[6:].tolist()]

    # replicate B
    if rank == root:
        bd = DeviceCsr.from_host(b, device)
    else:
        bd = DeviceCsr(b_rows, b_cols, torch.empty(b_rows + 1, **i64), torch.empty(b_nnz, **i64),
                       torch.empty(b_nnz, dtype=torch.float64, device=device))
    for t in (bd.row_ptr, bd.col_idx, bd.values):
        if t.numel():
            dist.broadcast(t, root, group=group)

    # scatter A row blocks (row pointers rebased to 0)
    r0, r1 = bounds[rank], bounds[rank + 1]
    if rank == root:
        arp, aci, av = csr_arrays(a)
        mine = None
        for g in range(world):
            g0, g1 = bounds[g], bounds[g + 1]
            blk = DeviceCsr.from_host(row_block_host(a, g0, g1), device)
            if g == rank:
                mine = blk
            else:
                for t in (blk.row_ptr, blk.col_idx, blk.values):
                    _send(t, g, group)
        a_blk = mine
    else:
        rp = torch.empty(r1 - r0 + 1, **i64)
        _recv(rp, root, group)
        n = int(rp[-1].item()) if rp.numel() else 0
        ci = torch.empty(n, **i64)
        v = torch.empty(n, dtype=torch.float64, device=device)
        _recv(ci, root, group)
        _recv(v, root, group)
        a_blk = DeviceCsr(r1 - r0, a_cols, rp, ci, v)

    # local product
    c_blk = local_multiply(a_blk, bd)

    # gather nnz, then the blocks
    nnz_t = torch.tensor([c_blk.nnz], **i64)
    all_nnz = [torch.zeros(1, **i64) for _ in range(world)]
    dist.all_gather(all_nnz, nnz_t, group=group)
    if rank != root:
        for t in (c_blk.row_ptr, c_blk.col_idx, c_blk.values):
            _send(t, root, group)
        return None
    blocks = []
    for g in range(world):
        if g == rank:
            blk = c_blk
        else:
            n = int(all_nnz[g].item())
            blk = DeviceCsr(bounds[g + 1] - bounds[g], b_cols,
                            torch.empty(bounds[g + 1] - bounds[g] + 1, **i64),
                            torch.empty(n, **i64),
                            torch.empty(n, dtype=torch.float64, device=device))
            for t in (blk.row_ptr, blk.col_idx, blk.values):
                _recv(t, g, group)
        blocks.append((blk.row_ptr.cpu().numpy().view(np.uint64),
                       blk.col_idx.cpu().numpy().view(np.uint64),
                       blk.values.cpu().numpy()))
    return concat_row_blocks(blocks, b_cols)
