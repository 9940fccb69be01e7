"""One rank of a multi-rank product, run under torch.distributed.run by
tests/test_distributed.py (CPU, gloo, oracle injected as the per-rank
product) and tests/test_gpu_distributed.py (every rank on cuda:0 over gloo,
the CUDA library as the per-rank product). Test infrastructure.

    python -m torch.distributed.run --nproc-per-node 2 ... tests/dist_worker.py
        --case NAME | --config C3   --out result.npz  [--device cuda] [--stats]
        [--expect mismatch|malformed] [--calls K]
"""

from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1303_1651_b200.distributed import (multiply_distributed, partition_rows,  # noqa: E402
                                              share_csr)
from paper_1303_1651_b200.formats import CsrMatrix  # noqa: E402
from paper_1303_1651_b200.kernels import KernelStats  # noqa: E402


def _host(m, r0=None, r1=None):
    rp = m.row_ptr.cpu().numpy().view(np.uint64)
    ci = m.col_idx.cpu().numpy().view(np.uint64)
    v = m.values.cpu().numpy()
    if r0 is None:
        return CsrMatrix(m.rows, m.cols, rp.copy(), ci.copy(), v.copy())
    lo, hi = int(rp[r0]), int(rp[r1])
    return CsrMatrix(r1 - r0, m.cols, (rp[r0:r1 + 1] - rp[r0]).astype(np.uint64),
                     ci[lo:hi].copy(), v[lo:hi].copy())


class OracleBlock:
    def __init__(self, r, row0):
        self.r = r
        self.nnz = r.nnz
        self.multiplications = r.multiplications
        self.choices = None
        if r.row_choices is not None:
            self.choices = [(row0 + i, int(c) == 0) for i, c in enumerate(r.row_choices.tolist())
                            if c >= 0]

    def download(self, offset, rp_addr, ci_addr, v_addr):
        rp = np.ascontiguousarray(self.r.row_ptr + np.uint64(offset))
        ctypes.memmove(rp_addr, rp.ctypes.data, rp.nbytes)
        if self.nnz:
            ci = np.ascontiguousarray(self.r.col_idx)
            v = np.ascontiguousarray(self.r.values)
            ctypes.memmove(ci_addr, ci.ctypes.data, ci.nbytes)
            ctypes.memmove(v_addr, v.ctypes.data, v.nbytes)

    def close(self):
        pass


def oracle_local(ad, bd, r0, r1, sid, want_stats):
    import oracle

    return OracleBlock(oracle.multiply_rowmajor(_host(ad, r0, r1), _host(bd),
                                                row_choices=want_stats), r0)


def oracle_partition(ad, bd, parts):
    import oracle

    a, b = _host(ad), _host(bd)
    if a.col_idx.size and int(a.col_idx.max()) >= b.rows:
        raise ValueError("a.col_idx entry >= b.rows")  # as the GPU count pass reports it
    prefix = np.zeros(a.rows + 1, np.uint64)
    np.cumsum(oracle.row_products(a, b), out=prefix[1:])
    return partition_rows(prefix, parts)


def _operands(args):
    """Rank 0's operands (None elsewhere), then shared with every rank."""
    a = b = None
    if dist.get_rank() == 0:
        if args.case:
            from conftest import golden_case

            a, b, _, _, _ = golden_case(args.case)
        else:
            from paper_1303_1651_b200 import genmat

            a, b, _ = genmat.config_operands(args.config)
            if b is a:
                b = None
        if args.expect == "mismatch":
            b = CsrMatrix(b.rows + 1, b.cols, np.concatenate([b.row_ptr, b.row_ptr[-1:]]),
                          b.col_idx.copy(), b.values.copy())
        if args.expect == "malformed":
            ci = a.col_idx.copy()
            ci[len(ci) // 2] = np.uint64(a.cols + 7)  # past b.rows
            a = CsrMatrix(a.rows, a.cols, a.row_ptr.copy(), ci, a.values.copy())
    flags = [b is None and args.config is not None]
    dist.broadcast_object_list(flags, src=0)
    sa = share_csr(a)
    sb = sa if flags[0] else share_csr(b)
    return sa, sb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case")
    ap.add_argument("--config")
    ap.add_argument("--out", required=True)
    ap.add_argument("--device", default="cpu")
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--expect", choices=["mismatch", "malformed"])
    ap.add_argument("--calls", type=int, default=1)
    ap.add_argument("--backend", default="gloo", choices=["gloo", "nccl"])
    args = ap.parse_args()
    if args.backend == "nccl":
        torch.cuda.set_device(torch.device(args.device))
        dist.init_process_group("nccl", device_id=torch.device(args.device))
    else:
        dist.init_process_group("gloo")
    rank = dist.get_rank()
    try:
        device = torch.device(args.device)
        kw = {}
        if device.type == "cpu":
            kw = dict(local_multiply=oracle_local, partition_fn=oracle_partition)
        else:
            torch.cuda.set_device(device)
        a, b = _operands(args)
        if args.expect:
            try:
                multiply_distributed(a, b, device=device, **kw)
            except ValueError as e:
                msg = str(e)
                with open(f"{args.out}.rank{rank}", "w") as f:
                    f.write(msg)
                return 0
            raise SystemExit(f"rank {rank}: no error raised")
        c = None
        for _ in range(args.calls):  # repeated calls reuse (and grow) the result arena
            stats = KernelStats() if args.stats else None
            timings = {}
            c = multiply_distributed(a, b, stats=stats, device=device, timings=timings, **kw)
        if rank == 0:
            out = dict(rp=np.asarray(c.row_ptr), ci=np.asarray(c.col_idx),
                       v=np.asarray(c.values), shape=np.array([c.rows, c.cols]),
                       bounds=np.array(timings["bounds"]))
            if stats is not None:
                ch = np.full(c.rows, -1, np.int8)
                for r, x in stats.row_choices:
                    ch[r] = 0 if x.value == "minmax" else 1
                out.update(mults=np.array([stats.multiplications]), choices=ch)
            if args.config:
                # digests like tests/golden/fingerprints.json
                dig = {k: hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
                       for k, arr in (("row_ptr", out["rp"]), ("col_idx", out["ci"]),
                                      ("values", out["v"]))}
                with open(args.out, "w") as f:
                    json.dump({"digests": dig, "nnz": int(out["ci"].size),
                               "bounds": out["bounds"].tolist()}, f)
            else:
                np.savez(args.out, **out)
        else:
            assert c is None
    finally:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
