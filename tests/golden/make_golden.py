"""Generate the golden fixtures that pin the oracle and the CUDA path to the
reference package itself.

Run HERE (the build container), where the read-only reference lives at
/root/reference; its outputs are committed under tests/golden/ so that the
GPU box (which has no /root/reference) can check against them:

    python tests/golden/make_golden.py small        # -> small_cases.npz  (seconds)
    python tests/golden/make_golden.py full         # -> fingerprints.json (~10 min)
    python tests/golden/make_golden.py formats      # -> formats_cases.npz (seconds)

* small_cases.npz  every operand pair plus the reference's C = A·B
  (`sparsemm.kernels.multiply_rowmajor`, COMBINED), its KernelStats
  (multiplications, row_choices) and estimate_nnz / count_mults, for:
  the known-answer tests of pkg/tests/test_kernels.py (hand 2x2, exact
  cancellation, transient zero, identity), the acceptance corpus of
  pkg/tests/test_acceptance.py:54-63 (200 random pairs + FD grids 1..16),
  rectangular and empty shapes, signed collision-heavy inputs, and long-row
  inputs (thousands of products per row, with exact cancellations) that
  exercise the long-row path.
* formats_cases.npz  for a subset of the small cases: the reference's
  storage-order conversions (csr_to_csc of A and B), its column-major product
  `multiply_colmajor(A_csc, B_csc)` and both mixed products
  `multiply_mixed(A, B_csc)` / `multiply_mixed(A_csc, B)` with their
  KernelStats (multiplications, per-major choices, conversions) and
  `estimate_nnz_csc` (kernels.py:335-363, 417-438; formats.py:292-357).
* fingerprints.json  sha256 fingerprints (genmat.py:154-165 plus separate
  structure/value digests) of the full-size BASELINE configs C1..C5, both
  operands and reference products. C1..C3 operands come from the reference's
  own generators; C4/C5 have no reference generator, so their operands come
  from libspmmm's spmmm_gen_fd3 / spmmm_gen_zipf and only the product is the
  reference's.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from sparsemm.formats import CsrMatrix, estimate_nnz  # noqa: E402
from sparsemm.genmat import SplitMix64, gen_fd, gen_random_k, matrix_fingerprint  # noqa: E402
from sparsemm.kernels import KernelStats, StrategyKind, multiply_rowmajor  # noqa: E402
from sparsemm.perfmodel import count_mults  # noqa: E402


def _genlib():
    path = os.environ.get("SPMMM_LIB", os.path.join(REPO, "paper_1303_1651_b200", "libspmmm.so"))
    lib = ctypes.CDLL(path)
    return lib


def _u64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _f64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def gen_fd3_lib(grid):
    lib = _genlib()
    rows, nnz = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.spmmm_gen_fd3_size(ctypes.c_uint64(grid), ctypes.byref(rows), ctypes.byref(nnz)) == 0
    rp = np.zeros(rows.value + 1, np.uint64)
    ci = np.zeros(nnz.value, np.uint64)
    v = np.zeros(nnz.value, np.float64)
    assert lib.spmmm_gen_fd3(ctypes.c_uint64(grid), _u64p(rp), _u64p(ci), _f64p(v)) == 0
    return CsrMatrix(rows.value, rows.value, rp, ci, v)


def gen_zipf_lib(n, seed, s=2.0, lmax=4096):
    lib = _genlib()
    lib.spmmm_gen_zipf.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    nnz = ctypes.c_uint64()
    assert lib.spmmm_gen_zipf(n, s, lmax, seed, ctypes.byref(nnz), None, None, None) == 0
    rp = np.zeros(n + 1, np.uint64)
    ci = np.zeros(nnz.value, np.uint64)
    v = np.zeros(nnz.value, np.float64)
    assert lib.spmmm_gen_zipf(n, s, lmax, seed, ctypes.byref(nnz), rp.ctypes.data,
                              ci.ctypes.data, v.ctypes.data) == 0
    return CsrMatrix(n, n, rp, ci, v)


def digests(m) -> dict:
    def h(arr, dt):
        return hashlib.sha256(np.ascontiguousarray(arr, dtype=dt).tobytes()).hexdigest()

    return {
        "rows": int(m.rows), "cols": int(m.cols), "nnz": int(m.nnz),
        "fingerprint": matrix_fingerprint(m),
        "row_ptr_sha256": h(m.row_ptr, "<u8"),
        "col_idx_sha256": h(m.col_idx, "<u8"),
        "values_sha256": h(m.values, "<f8"),
        "values_sum": float(np.sum(m.values, dtype=np.float64)),
    }


# ----------------------------------------------------------------------------
# small cases


def csr(dense):
    return CsrMatrix.from_dense(np.asarray(dense, dtype=float))


def random_pair(seed, n_min=4, n_max=64):
    # pkg/tests/conftest.py:49-57
    rng = SplitMix64(seed ^ 0xA5A5A5A5)
    n = n_min + rng.next_below(n_max - n_min + 1)
    k = min(5, n)
    return gen_random_k(n, k, seed), gen_random_k(n, k, seed + 1)


def signed(m, seed):
    """Same structure, values flipped in sign by a splitmix64 coin per entry."""
    rng = SplitMix64(seed)
    flips = np.array([1.0 if rng.next_u64() & 1 else -1.0 for _ in range(m.nnz)])
    return CsrMatrix.from_arrays(m.rows, m.cols, m.row_ptr, m.col_idx, m.values * flips)


def rect_random(rows, cols, density, seed, quantize=False):
    rng = SplitMix64(seed)
    dense = np.zeros((rows, cols))
    for r in range(rows):
        for c in range(cols):
            if (rng.next_u64() >> 11) * 2.0 ** -53 < density:
                u = (rng.next_u64() >> 11) * 2.0 ** -53
                dense[r, c] = (np.floor(u * 8) - 4.0) if quantize else (2 * u - 1)
    return csr(dense)


def long_rows_case(seed):
    """Rows with thousands of products (long-row path), including duplicated B
    rows multiplied by +1/-1 so whole output rows cancel to exact zeros."""
    n = 6000
    b = gen_random_k(n, 6, seed + 1)
    bp, bi, bv = b.row_ptr.tolist(), b.col_idx.tolist(), b.values.tolist()
    # make B row 1 an exact copy of B row 0, and row 3 a copy of row 2
    rows = [list(zip(bi[bp[r]:bp[r + 1]], bv[bp[r]:bp[r + 1]])) for r in range(n)]
    rows[1] = list(rows[0])
    rows[3] = list(rows[2])
    b = _from_rows(n, n, rows)
    rng = SplitMix64(seed)
    arows = []
    lengths = [0, 1, 40, 200, 700, 1500, 3000, 5, 33, 1000, 2500, 2, 129]
    for i, ln in enumerate(lengths):
        cols = set()
        while len(cols) < ln:
            cols.add(rng.next_below(n))
        row = sorted((c, ((rng.next_u64() >> 11) + 1) * 2.0 ** -53) for c in cols)
        if i % 3 == 0:
            # exact cancellation: +v at col 0, -v at col 1 (identical B rows)
            row = [e for e in row if e[0] not in (0, 1, 2, 3)]
            row = sorted(row + [(0, 0.75), (1, -0.75), (2, 1.5), (3, -1.5)])
        arows.append(row)
    return _from_rows(len(lengths), n, arows), b


def _from_rows(nrows, ncols, rows):
    rp = [0]
    ci, v = [], []
    for row in rows:
        for c, x in row:
            ci.append(c)
            v.append(x)
        rp.append(len(ci))
    return CsrMatrix.from_arrays(nrows, ncols, rp, ci, v)


def small_cases():
    cases = {}
    cases["hand_2x2"] = (csr([[1.0, 2.0], [0.0, 1.0]]), csr([[1.0, 0.0], [3.0, 1.0]]))
    cases["cancellation"] = (csr([[1.0, -1.0]]), csr([[5.0, 2.0], [5.0, 0.0]]))
    cases["transient_zero"] = (csr([[1.0, 1.0, 1.0]]), csr([[2.0], [-2.0], [3.0]]))
    cases["clean_after_cancelled"] = (
        CsrMatrix.from_arrays(1, 2, [0, 2], [0, 1], [1.0, -1.0]),
        CsrMatrix.from_arrays(2, 4, [0, 2, 4], [1, 3, 1, 3], [2.0, 1.0, 2.0, -1.0]))
    eye = csr(np.eye(24))
    cases["identity_left"] = (eye, gen_random_k(24, 4, 11))
    cases["identity_right"] = (gen_random_k(24, 4, 11), eye)
    cases["fd3_squared"] = (gen_fd(3), gen_fd(3))
    for seed in range(200):
        cases[f"random_{seed}"] = random_pair(seed)
    for g in range(1, 17):
        cases[f"fd_{g}"] = (gen_fd(g), gen_fd(g))
    # rectangular / empty shapes
    cases["rect_7x13_13x5"] = (rect_random(7, 13, 0.4, 1), rect_random(13, 5, 0.5, 2))
    cases["rect_1x40_40x1"] = (rect_random(1, 40, 0.9, 3), rect_random(40, 1, 0.9, 4))
    cases["rect_40x1_1x40"] = (rect_random(40, 1, 0.9, 5), rect_random(1, 40, 0.9, 6))
    cases["quantized_cancel"] = (rect_random(60, 50, 0.3, 7, True), rect_random(50, 70, 0.3, 8, True))
    cases["all_zero_left"] = (csr(np.zeros((4, 4))), gen_random_k(4, 2, 3))
    cases["all_zero_right"] = (gen_random_k(5, 2, 3), csr(np.zeros((5, 6))))
    cases["empty_rows_mix"] = (rect_random(30, 30, 0.05, 9), rect_random(30, 30, 0.05, 10))
    cases["zero_rows"] = (CsrMatrix.from_arrays(0, 5, [0], [], []), gen_random_k(5, 2, 1))
    cases["zero_inner"] = (CsrMatrix.from_arrays(3, 0, [0, 0, 0, 0], [], []),
                           CsrMatrix.from_arrays(0, 4, [0], [], []))
    cases["zero_cols_out"] = (gen_random_k(6, 2, 4), CsrMatrix.from_arrays(6, 0, [0] * 7, [], []))
    # signed, collision-heavy (a reversed fold fails 1e-12 here)
    a = signed(gen_random_k(300, 40, 21), 1)
    b = signed(gen_random_k(300, 40, 22), 2)
    cases["signed_k40"] = (a, b)
    a = signed(gen_random_k(64, 48, 23), 3)
    cases["signed_dense_rows"] = (a, signed(gen_random_k(64, 48, 24), 4))
    # medium rows (33..768 products) and an A row with > 32 entries but short B rows
    cases["medium_rows"] = (gen_random_k(200, 20, 31), gen_random_k(200, 20, 32))
    cases["wide_a_short_b"] = (gen_random_k(200, 60, 33),
                               _from_rows(200, 200, [[] if r % 2 else [(r, 1.5)] for r in range(200)]))
    cases["long_rows"] = long_rows_case(41)
    return cases


def run_small(out_path):
    t0 = time.time()
    store = {}
    names = []
    for name, (a, b) in small_cases().items():
        stats = KernelStats()
        c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
        choices = np.full(a.rows, -1, np.int8)
        for r, ch in stats.row_choices:
            choices[r] = 0 if ch is StrategyKind.MIN_MAX else 1
        for tag, m in (("a", a), ("b", b), ("c", c)):
            store[f"{name}/{tag}_shape"] = np.array([m.rows, m.cols], np.uint64)
            store[f"{name}/{tag}_rp"] = np.asarray(m.row_ptr, np.uint64)
            store[f"{name}/{tag}_ci"] = np.asarray(m.col_idx, np.uint64)
            store[f"{name}/{tag}_v"] = np.asarray(m.values, np.float64)
        store[f"{name}/mults"] = np.array([stats.multiplications], np.uint64)
        store[f"{name}/estimate_nnz"] = np.array([estimate_nnz(a, b)], np.uint64)
        store[f"{name}/count_mults"] = np.array([count_mults(a, b).multiplications], np.uint64)
        store[f"{name}/row_choices"] = choices
        names.append(name)
    # splitmix64 seed-0 stream (pkg/tests/test_genmat.py:21-28) and a few more
    for seed in (0, 1, 0xA5A5A5A5, 2**64 - 1):
        rng = SplitMix64(seed)
        store[f"splitmix64/{seed}"] = np.array([rng.next_u64() for _ in range(64)], np.uint64)
    store["_names"] = np.array(names)
    np.savez_compressed(out_path, **store)
    print(f"wrote {out_path}: {len(names)} cases in {time.time() - t0:.1f}s")


# ----------------------------------------------------------------------------
# storage-order fixtures


def formats_subset(cases):
    keep = ["hand_2x2", "cancellation", "transient_zero", "clean_after_cancelled",
            "identity_left", "identity_right", "fd3_squared", "rect_7x13_13x5",
            "rect_1x40_40x1", "rect_40x1_1x40", "quantized_cancel", "all_zero_left",
            "all_zero_right", "empty_rows_mix", "zero_rows", "zero_inner", "zero_cols_out",
            "wide_a_short_b"]
    keep += [f"random_{s}" for s in range(0, 200, 5)] + [f"fd_{g}" for g in (1, 2, 5, 8, 13)]
    return {k: cases[k] for k in keep}


def run_formats(out_path):
    from sparsemm.formats import csr_to_csc, estimate_nnz_csc
    from sparsemm.kernels import multiply_colmajor, multiply_mixed

    t0 = time.time()
    store = {}
    names = []

    def put_csc(prefix, m):
        store[f"{prefix}_shape"] = np.array([m.rows, m.cols], np.uint64)
        store[f"{prefix}_ptr"] = np.asarray(m.col_ptr, np.uint64)
        store[f"{prefix}_idx"] = np.asarray(m.row_idx, np.uint64)
        store[f"{prefix}_v"] = np.asarray(m.values, np.float64)

    def put_csr(prefix, m):
        store[f"{prefix}_shape"] = np.array([m.rows, m.cols], np.uint64)
        store[f"{prefix}_ptr"] = np.asarray(m.row_ptr, np.uint64)
        store[f"{prefix}_idx"] = np.asarray(m.col_idx, np.uint64)
        store[f"{prefix}_v"] = np.asarray(m.values, np.float64)

    def put_stats(prefix, stats, n_major):
        ch = np.full(n_major, -1, np.int8)
        for r, c in stats.row_choices:
            ch[r] = 0 if c is StrategyKind.MIN_MAX else 1
        store[f"{prefix}_mults"] = np.array([stats.multiplications], np.uint64)
        store[f"{prefix}_conv"] = np.array([stats.conversions], np.uint64)
        store[f"{prefix}_choices"] = ch

    for name, (a, b) in formats_subset(small_cases()).items():
        a_csc, b_csc = csr_to_csc(a), csr_to_csc(b)
        put_csr(f"{name}/a", a)
        put_csr(f"{name}/b", b)
        put_csc(f"{name}/a_csc", a_csc)
        put_csc(f"{name}/b_csc", b_csc)
        st = KernelStats()
        put_csc(f"{name}/col", multiply_colmajor(a_csc, b_csc, StrategyKind.COMBINED, st))
        put_stats(f"{name}/col", st, b.cols)
        st = KernelStats()
        put_csr(f"{name}/mix_rc", multiply_mixed(a, b_csc, StrategyKind.COMBINED, st))
        put_stats(f"{name}/mix_rc", st, a.rows)
        st = KernelStats()
        put_csc(f"{name}/mix_cr", multiply_mixed(a_csc, b, StrategyKind.COMBINED, st))
        put_stats(f"{name}/mix_cr", st, b.cols)
        store[f"{name}/estimate_csc"] = np.array([estimate_nnz_csc(a_csc, b_csc)], np.uint64)
        names.append(name)
    store["_names"] = np.array(names)
    np.savez_compressed(out_path, **store)
    print(f"wrote {out_path}: {len(names)} cases in {time.time() - t0:.1f}s")


# ----------------------------------------------------------------------------
# full-size fingerprints


def run_full(out_path, only=None):
    results = {}
    if os.path.exists(out_path):
        with open(out_path) as f:
            results = json.load(f)

    def save():
        with open(out_path, "w") as f:
            json.dump(results, f, indent=1, sort_keys=True)

    def product(label, a, b, a_src, b_src):
        if only and label not in only:
            return
        t0 = time.time()
        stats = KernelStats()
        c = multiply_rowmajor(a, b, StrategyKind.COMBINED, stats)
        dt = time.time() - t0
        results[label] = {
            "a": digests(a), "b": digests(b), "c": digests(c),
            "multiplications": int(stats.multiplications),
            "a_source": a_src, "b_source": b_src,
            "reference_seconds": round(dt, 2),
        }
        save()
        print(f"{label}: nnz(C)={c.nnz} mults={stats.multiplications} ref {dt:.1f}s", flush=True)

    a = gen_fd(100)
    product("C1_fd100", a, a, "sparsemm.genmat.gen_fd(100)", "same as a")
    for g in (32, 64, 128, 256, 512, 1024, 2048):
        if only and f"C2_fd{g}" not in only:
            continue
        a = gen_fd(g)
        product(f"C2_fd{g}", a, a, f"sparsemm.genmat.gen_fd({g})", "same as a")
    if not only or "C3_random2M" in only:
        a = gen_random_k(2_000_000, 5, 0)
        b = gen_random_k(2_000_000, 5, 1)
        product("C3_random2M", a, b, "sparsemm.genmat.gen_random_k(2000000, 5, 0)",
                "sparsemm.genmat.gen_random_k(2000000, 5, 1)")
    if not only or "C4_fd3_100" in only:
        a = gen_fd3_lib(100)
        product("C4_fd3_100", a, a, "libspmmm spmmm_gen_fd3(100)", "same as a")
    if not only or "C5_zipf2M" in only:
        a = gen_zipf_lib(2_000_000, 0)
        b = gen_zipf_lib(2_000_000, 1)
        product("C5_zipf2M", a, b, "libspmmm spmmm_gen_zipf(2000000, s=2, lmax=4096, seed=0)",
                "libspmmm spmmm_gen_zipf(2000000, s=2, lmax=4096, seed=1)")


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "small"
    if mode == "small":
        run_small(os.path.join(HERE, "small_cases.npz"))
    elif mode == "full":
        run_full(os.path.join(HERE, "fingerprints.json"), set(sys.argv[2:]) or None)
    elif mode == "formats":
        run_formats(os.path.join(HERE, "formats_cases.npz"))
    else:
        raise SystemExit("usage: make_golden.py small|full|formats [labels...]")
