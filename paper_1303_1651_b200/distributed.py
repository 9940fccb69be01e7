"""Multi-GPU C = A·B by product-balanced row blocks.

Rows of C are independent — each depends on its A row and all of B
(kernels.py:323-329) — so the product shards with no data-path collective
beyond replicating the operands. One process per GPU; `torch.distributed`
is the plumbing (NCCL for the bulk operand exchange over NVLink, a gloo
group for the few words of control).

Every rank calls `multiply_distributed(a, b)` with the same host operands
(typically views of one node-wide shared-memory copy, see `share_csr`).
One call is:

1. upload     — rank r copies chunk r (1/G of each array) of A, and of B when
                B is not A, over its own PCIe link;
2. all-gather — NCCL all-gathers the chunks over NVLink, so every GPU holds
                all of A and B (no single link carries the whole operand);
3. partition  — every GPU runs the count pass and cuts A into G row blocks of
                equal *product* count on the device (spmmm_partition_rows:
                lower_bound over the product prefix — C5's rows range from 1
                to ~40K products). Same data, same integer arithmetic: every
                rank derives the same bounds without a collective;
4. compute    — rank g multiplies its row block (a zero-copy view of the
                resident A) by B with libspmmm;
5. offsets    — all-gather of (status, nnz, multiplications), 24 B per rank;
                every rank raises the same error if any rank failed;
6. gather     — the root reserves the result in a node-wide shared-memory
                arena (page-locked in every rank) and broadcasts where; each
                rank downloads its block over its own PCIe link straight into
                its slice (row pointers shifted by the nnz before it on the
                device), so no link or GPU relays another rank's C.

The root returns the CsrMatrix (arrays in the arena, released when the
arrays die); the other ranks return None. `local_multiply` and
`partition_fn` are injectable so the orchestration runs on CPU with gloo
(tests/test_distributed.py); with a CUDA device the product is libspmmm's.
"""

from __future__ import annotations

import ctypes
import mmap
import os
import threading
import time
import uuid
import warnings
import weakref
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .formats import CsrMatrix, csr_arrays

_SHM_DIR = "/dev/shm"
_ALIGN = 256


def partition_rows(prefix, parts: int) -> np.ndarray:
    """Row bounds (parts+1) splitting rows so that block g holds the rows whose
    product prefix lies in [g*T/G, (g+1)*T/G): bounds[g] = lower_bound(prefix,
    g*T/G). `prefix` is the exclusive prefix of per-row products (rows+1
    entries, prefix[0] = 0). Rows are never split. The device version is
    spmmm_partition_rows (same targets, same lower_bound)."""
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
    r = e = 0
    for rp, ci, v in blocks:
        n = int(rp.size) - 1
        out_rp[r + 1:r + n + 1] = rp[1:] + np.uint64(e)
        out_ci[e:e + ci.size] = ci
        out_v[e:e + v.size] = v
        r += n
        e += ci.size
    return CsrMatrix(rows, cols, out_rp, out_ci, out_v)


# ---------------------------------------------------------------------------
# node-wide shared memory


class SharedSegment:
    """A /dev/shm file mapped by every rank of the node. The creator unlinks
    it once every rank has mapped it (the mappings stay valid), so nothing
    outlives the processes."""

    def __init__(self, name: str, size: int, create: bool):
        self.name = name
        self.size = max(int(size), mmap.PAGESIZE)
        path = os.path.join(_SHM_DIR, name)
        fd = os.open(path, os.O_RDWR | (os.O_CREAT | os.O_EXCL if create else 0), 0o600)
        try:
            if create:
                os.ftruncate(fd, self.size)
            self.mm = mmap.mmap(fd, self.size)
        finally:
            os.close(fd)
        self.addr = ctypes.addressof(ctypes.c_char.from_buffer(self.mm))
        self.registered = False

    def unlink(self):
        try:
            os.unlink(os.path.join(_SHM_DIR, self.name))
        except FileNotFoundError:
            pass

    def register(self):
        """Page-lock the mapping in this process (DMA-speed copies)."""
        if not self.registered and torch.cuda.is_available():
            from . import _lib

            _lib.host_register(self.addr, self.size)
            self.registered = True

    def unregister(self):
        if self.registered:
            from . import _lib

            try:
                _lib.host_unregister(self.addr)
            except RuntimeError:
                pass
            self.registered = False

    def array(self, offset: int, n: int, dtype, keepalive=None) -> np.ndarray:
        """numpy view of n elements at byte `offset`. With `keepalive`, the
        view is built on a ctypes buffer whose death calls keepalive()."""
        dtype = np.dtype(dtype)
        if keepalive is None:
            return np.frombuffer(self.mm, dtype=dtype, count=int(n), offset=int(offset))
        nbytes = max(int(n) * dtype.itemsize, 1)
        buf = (ctypes.c_char * nbytes).from_address(self.addr + int(offset))
        buf._segment = self  # the mapping outlives every view
        weakref.finalize(buf, keepalive)
        return np.frombuffer(buf, dtype=dtype, count=int(n))


def _new_name() -> str:
    return f"spmmm-{os.getpid()}-{uuid.uuid4().hex[:12]}"


def share_csr(m, group=None, root: int = 0, register: bool = True) -> CsrMatrix:
    """Collective: the root's CSR matrix copied once into node-wide shared
    memory; every rank gets a CsrMatrix over the same pages (page-locked in
    each rank when a GPU is present, so uploads from it run at DMA speed).
    Operand preparation, outside any timed region."""
    ctrl = control_group(group)
    rank = dist.get_rank(group)
    meta = [None]
    if rank == root:
        rp, ci, v = csr_arrays(m)
        sizes = [rp.nbytes, ci.nbytes, v.nbytes]
        offs = [0]
        for s in sizes[:-1]:
            offs.append(_align(offs[-1] + s))
        total = offs[-1] + sizes[-1]
        seg = SharedSegment(_new_name(), total, create=True)
        for arr, off in zip((rp, ci, v), offs):
            seg.array(off, arr.size, arr.dtype)[...] = arr
        meta = [(seg.name, seg.size, int(m.rows), int(m.cols), int(rp.size), int(ci.size), offs)]
    dist.broadcast_object_list(meta, src=_global_rank(ctrl, root), group=ctrl)
    name, size, rows, cols, n_rp, nnz, offs = meta[0]
    if rank != root:
        seg = SharedSegment(name, size, create=False)
    dist.barrier(group=ctrl)
    if rank == root:
        seg.unlink()
    if register:
        seg.register()
    rp = seg.array(offs[0], n_rp, np.uint64)
    ci = seg.array(offs[1], nnz, np.uint64)
    v = seg.array(offs[2], nnz, np.float64)
    out = CsrMatrix(rows, cols, rp, ci, v)
    out._shared_segment = seg  # keeps the mapping (and its registration) alive
    return out


def _align(x: int) -> int:
    return (int(x) + _ALIGN - 1) // _ALIGN * _ALIGN


# ---------------------------------------------------------------------------
# the result arena: one shared segment per generation, ranges handed out by
# the root (first fit), freed when the root's result arrays die


class _Arena:
    def __init__(self):
        self.gen = -1
        self.seg = None
        self.free = []       # root: sorted (offset, size) ranges of the current segment
        self.retired = {}    # root: gen -> [segment, live count]
        self.live = 0
        self.lock = threading.Lock()

    # root side
    def alloc(self, sizes):
        """Offsets for `sizes` in the current segment, or None if it is too
        small (the caller grows it)."""
        with self.lock:
            if self.seg is None:
                return None
            need = sum(_align(s) for s in sizes)
            for i, (off, size) in enumerate(self.free):
                if size >= need:
                    rest = (off + need, size - need)
                    self.free[i:i + 1] = [rest] if rest[1] else []
                    offs, o = [], off
                    for s in sizes:
                        offs.append(o)
                        o += _align(s)
                    self.live += 1
                    return offs, need
            return None

    def release(self, gen, off, need):
        with self.lock:
            if gen == self.gen:
                self.free.append((off, need))
                self.free.sort()
                merged = []
                for o, s in self.free:
                    if merged and merged[-1][0] + merged[-1][1] == o:
                        merged[-1] = (merged[-1][0], merged[-1][1] + s)
                    else:
                        merged.append((o, s))
                self.free = merged
                self.live -= 1
            elif gen in self.retired:
                ent = self.retired[gen]
                ent[1] -= 1
                if ent[1] == 0:
                    ent[0].unregister()
                    del self.retired[gen]

    def install(self, gen, seg, is_root):
        with self.lock:
            if self.seg is not None:
                if is_root and self.live:
                    self.retired[self.gen] = [self.seg, self.live]
                else:
                    self.seg.unregister()
            self.gen, self.seg = gen, seg
            self.free = [(0, seg.size)] if is_root else []
            self.live = 0


_arenas: dict = {}
_ctrl_groups: dict = {}


def control_group(group=None):
    """A gloo group over the same ranks for the control words (CPU tensors,
    no device sync); the group itself when it already is gloo."""
    key = group if group is not None else dist.group.WORLD
    g = _ctrl_groups.get(key)
    if g is None:
        if dist.get_backend(group) == "gloo":
            g = key
        else:
            ranks = dist.get_process_group_ranks(key) if group is not None else None
            g = dist.new_group(ranks=ranks, backend="gloo")
        _ctrl_groups[key] = g
    return g


def _global_rank(group, rank):
    return dist.get_global_rank(group, rank) if group not in (None, dist.group.WORLD) else rank


# ---------------------------------------------------------------------------
# operand replication: chunked upload + all-gather


def _to_tensor(arr: np.ndarray) -> torch.Tensor:
    a = arr.view(np.int64) if arr.dtype == np.uint64 else arr
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # read-only arrays: we only read them
        return torch.from_numpy(a)


def _replicate(arr: np.ndarray, rank: int, world: int, device, group,
               nccl: bool) -> torch.Tensor:
    """All of `arr` on this rank's device; this rank uploads only its chunk.
    Returns a tensor of arr.size elements (a prefix of the padded buffer)."""
    n = int(arr.size)
    dtype = torch.float64 if arr.dtype == np.float64 else torch.int64
    chunk = max(1, -(-n // world))
    lo, hi = min(n, rank * chunk), min(n, (rank + 1) * chunk)
    src = _to_tensor(arr)
    if nccl:
        buf = torch.empty(world * chunk, dtype=dtype, device=device)
        mine = torch.empty(chunk, dtype=dtype, device=device)  # (the padding is never read)
        if hi > lo:
            mine[:hi - lo].copy_(src[lo:hi], non_blocking=True)
        dist.all_gather_into_tensor(buf, mine, group=group)
        return buf[:n]
    if device.type == "cuda":
        # gloo (ranks sharing a GPU: a functional run): no NVLink to all-gather
        # over; every rank reads the whole node-wide shared operand itself
        return src.to(device, non_blocking=True)
    # gloo on CPU (tests): gather the chunks on the host
    mine = torch.zeros(chunk, dtype=dtype)
    if hi > lo:
        mine[:hi - lo].copy_(src[lo:hi])
    parts = [torch.empty(chunk, dtype=dtype) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat(parts)[:n].to(device)


@dataclass
class ResidentCsr:
    """A CSR matrix resident on this rank's device (tensors; uint64 data
    viewed as int64)."""

    rows: int
    cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    values: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.values.numel())


def replicate_csr(m, group=None, device=None) -> ResidentCsr:
    """Collective: every rank ends with all of `m` on its device, each rank
    having uploaded 1/G of it (NCCL all-gather over NVLink; gloo on CPU)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = _device(group, device)
    nccl = dist.get_backend(group) == "nccl"
    rp, ci, v = csr_arrays(m)
    return ResidentCsr(int(m.rows), int(m.cols),
                       _replicate(rp, rank, world, device, group, nccl),
                       _replicate(ci, rank, world, device, group, nccl),
                       _replicate(v, rank, world, device, group, nccl))


def _device(group, device):
    """This rank's device: the given one, else the current CUDA device (there
    is no CPU product: only the tests inject one, with device="cpu")."""
    if device is not None:
        return torch.device(device)
    if dist.get_backend(group) == "nccl" or torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


# ---------------------------------------------------------------------------
# the GPU defaults of the injectable steps


class _GpuBlock:
    """The rank's block of C, device-resident in libspmmm."""

    def __init__(self, product, choices):
        self.product = product
        self.nnz = product.nnz
        self.multiplications = product.multiplications
        self.choices = choices  # [(row, is_minmax)] with global rows, or None

    def download(self, offset, rp_addr, ci_addr, v_addr):
        self.product.download_offset(offset, rp_addr, ci_addr, v_addr)

    def close(self):
        self.product.close()


_contexts: dict = {}


def _context(device):
    from . import _lib

    idx = device.index if device.index is not None else torch.cuda.current_device()
    ctx = _contexts.get(idx)
    if ctx is None:
        from .device import context_for_current_stream

        ctx = context_for_current_stream(torch.device("cuda", idx))
        _contexts[idx] = ctx
    return ctx


def _view(m: ResidentCsr, r0=None, r1=None):
    from . import _lib

    if m.values.device.type != "cuda":
        raise RuntimeError("libspmmm needs device-resident operands (there is no CPU product)")
    rp = m.row_ptr if r0 is None else m.row_ptr[r0:r1 + 1]
    rows = m.rows if r0 is None else r1 - r0
    return _lib.device_view(rows, m.cols, m.nnz, rp.data_ptr(), m.col_idx.data_ptr(),
                            m.values.data_ptr())


def gpu_partition(a: ResidentCsr, b: ResidentCsr, parts: int):
    from . import _lib

    bounds, _ = _lib.partition_rows(_context(a.values.device), _view(a), _view(b), parts)
    return bounds


def gpu_block_multiply(a: ResidentCsr, b: ResidentCsr, r0: int, r1: int, strategy_id: int,
                       want_stats: bool):
    from . import _lib

    from .kernels import choices_from_row_stats

    flags = _lib.FLAG_ROW_STATS if want_stats else 0
    p = _lib.multiply_views(_context(a.values.device), _view(a, r0, r1), _view(b), strategy_id,
                            flags)
    choices = None
    if want_stats:
        a_rp = a.row_ptr[r0:r1 + 1].cpu().numpy().view(np.uint64)
        choices = choices_from_row_stats(p.row_stats() if b.cols else None, b.cols, a_rp, r0)
    return _GpuBlock(p, choices)


# ---------------------------------------------------------------------------


def _exchange_status(ctrl, words):
    """all-gather of int64 words per rank over the control group."""
    t = torch.tensor(words, dtype=torch.int64)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(ctrl))]
    dist.all_gather(out, t, group=ctrl)
    return [o.tolist() for o in out]


def _raise_collective(ctrl, err):
    """Every rank raises the first failing rank's error (no rank is left
    waiting in a collective)."""
    msgs = [None] * dist.get_world_size(ctrl)
    dist.all_gather_object(msgs, None if err is None else (type(err).__name__, str(err)),
                           group=ctrl)
    for m in msgs:
        if m is not None:
            kind, text = m
            raise (ValueError if kind == "ValueError" else RuntimeError)(text)


def multiply_distributed(a, b, strategy="combined", stats=None, *, group=None, device=None,
                         root: int = 0, local_multiply=None, partition_fn=None,
                         timings: dict | None = None):
    """C = A·B over all ranks of `group` (kernels.py:302-332 semantics, bytes
    identical to the single-GPU product). Every rank passes the same host
    operands; the root gets the host CsrMatrix, the other ranks None.
    `stats` (root): multiplications and row_choices as multiply_rowmajor."""
    from .kernels import _choice_enum, _strategy_id

    t0 = time.perf_counter()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctrl = control_group(group)
    device = _device(group, device)
    nccl = dist.get_backend(group) == "nccl"
    if a.cols != b.rows:  # every rank holds the shapes: all raise, none waits
        raise ValueError(f"dimension mismatch: {a.cols} (cols of a) != {b.rows} (rows of b)")
    sid = _strategy_id(strategy)
    local_multiply = local_multiply or gpu_block_multiply
    partition_fn = partition_fn or gpu_partition
    same = b is a or (a.row_ptr is b.row_ptr and a.col_idx is b.col_idx and a.values is b.values)

    # 1-2. operands on every device, each rank uploading 1/G over its link
    ad = replicate_csr(a, group, device)
    bd = ad if same else replicate_csr(b, group, device)
    t1 = time.perf_counter()

    # 3-4. partition (same on every rank) and this rank's block
    err, blk, bounds = None, None, None
    try:
        bounds = [int(x) for x in partition_fn(ad, bd, world)]
        r0, r1 = bounds[rank], bounds[rank + 1]
        blk = local_multiply(ad, bd, r0, r1, sid, stats is not None)
    except (ValueError, RuntimeError) as e:
        err = e
    t2 = time.perf_counter()

    # 5. status, nnz and multiplications of every block
    words = _exchange_status(ctrl, [0 if err is None else 1,
                                    blk.nnz if blk is not None else 0,
                                    blk.multiplications if blk is not None else 0])
    if any(w[0] for w in words):
        if blk is not None:
            blk.close()
        _raise_collective(ctrl, err)
    nnzs = [w[1] for w in words]
    offsets = np.concatenate([[0], np.cumsum(nnzs)]).astype(np.int64)
    total_nnz = int(offsets[-1])
    mults = sum(w[2] for w in words)

    # 6. the result in the shared arena; each rank downloads its slice. Every
    # step that can fail on one rank is followed by a status exchange, so all
    # ranks raise together instead of leaving the others in a collective.
    arena = _arenas.setdefault(ctrl, _Arena())
    sizes = [8 * (a.rows + 1), 8 * total_nnz, 8 * total_nnz]
    plan, new_seg = None, None
    if rank == root:
        try:
            got = arena.alloc(sizes)
            if got is not None:
                plan = ("fit", got)
            else:
                cur = arena.seg.size if arena.seg is not None else 0
                want = max(2 * sum(_align(s) for s in sizes) + (1 << 20), cur + cur // 2)
                new_seg = SharedSegment(_new_name(), want, create=True)
                plan = ("grow", new_seg.name, new_seg.size, arena.gen + 1)
        except OSError as e:
            plan = ("error", f"result arena: {e}")
    plan = _bcast(ctrl, root, plan)
    if plan[0] == "error":
        blk.close()
        raise RuntimeError(plan[1])
    if plan[0] == "grow":
        _, name, size, gen = plan
        err = None
        try:
            seg = new_seg if rank == root else SharedSegment(name, size, create=False)
            if device.type == "cuda":
                seg.register()
        except (OSError, RuntimeError) as e:
            err = e
        failed = any(w[0] for w in _exchange_status(ctrl, [0 if err is None else 1]))
        if rank == root:
            new_seg.unlink()  # every rank has mapped it (or given up)
        if failed:
            blk.close()
            _raise_collective(ctrl, err)
        arena.install(gen, seg, rank == root)
        got = _bcast(ctrl, root, arena.alloc(sizes) if rank == root else None)
    else:
        got = plan[1]
    offs, need = got
    seg, gen = arena.seg, arena.gen
    r0, r1 = bounds[rank], bounds[rank + 1]
    base = seg.addr
    err = None
    try:
        blk.download(int(offsets[rank]), base + offs[0] + 8 * r0,
                     base + offs[1] + 8 * int(offsets[rank]),
                     base + offs[2] + 8 * int(offsets[rank]))
    except RuntimeError as e:
        err = e
    mine = blk.choices or []
    blk.close()
    # every slice has landed (this exchange is the barrier)
    if any(w[0] for w in _exchange_status(ctrl, [0 if err is None else 1])):
        if rank == root:
            arena.release(gen, offs[0], need)
        _raise_collective(ctrl, err)
    choices = None
    if stats is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine, group=ctrl)
        choices = [c for part in gathered for c in part]
    t3 = time.perf_counter()
    if timings is not None:
        timings.update(replicate_ms=1e3 * (t1 - t0), compute_ms=1e3 * (t2 - t1),
                       gather_ms=1e3 * (t3 - t2), bounds=bounds, nnz=nnzs)
    if rank != root:
        return None
    release = _Releaser(arena, gen, offs[0], need)
    rp = seg.array(offs[0], a.rows + 1, np.uint64, keepalive=release.one)
    ci = seg.array(offs[1], total_nnz, np.uint64, keepalive=release.one)
    v = seg.array(offs[2], total_nnz, np.float64, keepalive=release.one)
    if stats is not None:
        stats.multiplications += mults
        enum_cls = _choice_enum(strategy)
        stats.row_choices.extend((r, enum_cls.MIN_MAX if mm else enum_cls.SORT)
                                 for r, mm in choices)
    from .formats import make_like

    return make_like(a, a.rows, b.cols, rp, ci, v)


def _bcast(ctrl, root, obj):
    box = [obj]
    dist.broadcast_object_list(box, src=_global_rank(ctrl, root), group=ctrl)
    return box[0]


class _Releaser:
    """Frees the result's arena range when its last array dies."""

    def __init__(self, arena, gen, off, need):
        self.arena, self.gen, self.off, self.need = arena, gen, off, need
        self.count = 3
        self.lock = threading.Lock()

    def one(self):
        with self.lock:
            self.count -= 1
            done = self.count == 0
        if done:
            self.arena.release(self.gen, self.off, self.need)
