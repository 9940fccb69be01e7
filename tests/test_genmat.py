"""The native generators against the reference's own outputs: the splitmix64
stream (pkg/tests/test_genmat.py:21-28), gen_fd / gen_random_k operands of
the golden corpus, and the full-size operand fingerprints of C1..C3. C4/C5
generators have no reference counterpart; their structural properties and
determinism are checked."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import fingerprints, golden_case, golden_splitmix
from paper_1303_1651_b200 import genmat
from paper_1303_1651_b200.formats import validate_csr


def test_splitmix64_seed0_known_answers():
    s = genmat.splitmix64(0, 3)
    assert s.tolist() == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("seed", [0, 1, 0xA5A5A5A5, 2**64 - 1])
def test_splitmix64_streams_match_reference(seed):
    assert np.array_equal(genmat.splitmix64(seed, 64), golden_splitmix(seed))


def test_gen_fd_matches_reference_corpus():
    for g in range(1, 17):
        a, _, _, _, _ = golden_case(f"fd_{g}")
        m = genmat.gen_fd(g)
        assert m.row_ptr.tobytes() == a.row_ptr.tobytes()
        assert m.col_idx.tobytes() == a.col_idx.tobytes()
        assert m.values.tobytes() == a.values.tobytes()
    assert genmat.gen_fd(32).values.size == 4992  # test_genmat.py:65-70


def test_gen_random_k_matches_reference_corpus():
    rng_seeds = [0, 1, 7, 23, 199]
    from paper_1303_1651_b200.genmat import splitmix64

    for seed in rng_seeds:
        a, b, _, _, _ = golden_case(f"random_{seed}")
        n = a.rows
        k = min(5, n)
        assert int(4 + splitmix64(seed ^ 0xA5A5A5A5, 1)[0] % 61) == n
        for m_ref, s in ((a, seed), (b, seed + 1)):
            m = genmat.gen_random_k(n, k, s)
            assert m.col_idx.tobytes() == m_ref.col_idx.tobytes()
            assert m.values.tobytes() == m_ref.values.tobytes()


@pytest.mark.parametrize("label", ["C1_fd100", "C2_fd512", "C2_fd2048", "C3_random2M"])
def test_full_size_operands_match_reference_fingerprints(label):
    fp = fingerprints().get(label)
    if fp is None:
        pytest.skip("fingerprint missing")
    if label.startswith("C3"):
        a, b = genmat.gen_random_k(2_000_000, 5, 0), genmat.gen_random_k(2_000_000, 5, 1)
    else:
        grid = int(label.split("fd")[1])
        a = b = genmat.gen_fd(grid)
    assert genmat.digests(a)["fingerprint"] == fp["a"]["fingerprint"]
    assert genmat.digests(b)["fingerprint"] == fp["b"]["fingerprint"]


def test_fd3_structure():
    m = genmat.gen_fd3(5)
    validate_csr(m)
    assert m.rows == 125
    d = m.to_dense()
    assert np.array_equal(d, d.T)
    assert np.all(np.diag(d) == 26.0)
    interior = 2 + 5 * 2 + 25 * 2  # (2,2,2)
    assert int(m.row_ptr[interior + 1] - m.row_ptr[interior]) == 27
    rows, nnz = m.rows, m.values.size
    assert nnz == (3 * 5 - 2) ** 3
    fp = fingerprints().get("C4_fd3_100")
    if fp:
        assert fp["a"]["nnz"] == 26_463_592


def test_zipf_structure_and_determinism():
    a = genmat.gen_zipf(50_000, 0)
    validate_csr(a)
    lens = np.diff(a.row_ptr.astype(np.int64))
    assert lens.min() >= 1 and lens.max() <= 4096
    # Zipf(2): P(L=1) = 1/zeta(2) ~ 0.608
    assert abs(np.mean(lens == 1) - 6 / np.pi**2) < 0.01
    assert np.all((a.values >= -1.0) & (a.values < 1.0))
    b = genmat.gen_zipf(50_000, 0)
    assert genmat.matrix_fingerprint(a) == genmat.matrix_fingerprint(b)
    assert genmat.matrix_fingerprint(genmat.gen_zipf(50_000, 1)) != genmat.matrix_fingerprint(a)


def test_config_operands_c5_fingerprint():
    fp = fingerprints().get("C5_zipf2M")
    if fp is None:
        pytest.skip("fingerprint missing")
    a, b, _ = genmat.config_operands("C5")
    assert genmat.digests(a)["fingerprint"] == fp["a"]["fingerprint"]
    assert genmat.digests(b)["fingerprint"] == fp["b"]["fingerprint"]


# --- the oracle's generators (gen_oracle.c), used by bench.py's reference arm


def test_oracle_splitmix64_matches_reference():
    import oracle

    for seed in (0, 1, 0xA5A5A5A5, 2**64 - 1):
        assert np.array_equal(oracle.splitmix64(seed, 64), golden_splitmix(seed))


@pytest.mark.parametrize("label", ["C1", "C3", "C4", "C5"])
def test_oracle_config_operands_match_reference_fingerprints(label):
    """The reference arm's operands are the reference's own (C1, C3) and the
    same bytes as the product's generators (C4, C5; fingerprints the
    reference computed over them)."""
    import oracle

    key = {"C1": "C1_fd100", "C3": "C3_random2M", "C4": "C4_fd3_100", "C5": "C5_zipf2M"}[label]
    fp = fingerprints().get(key)
    if fp is None:
        pytest.skip("fingerprint missing")
    a, b, _ = oracle.config_operands(label)
    assert genmat.digests(a)["fingerprint"] == fp["a"]["fingerprint"]
    assert genmat.digests(b)["fingerprint"] == fp["b"]["fingerprint"]


def test_oracle_c2_sweep_operand_matches_reference():
    import oracle

    for g in (32, 512):
        fp = fingerprints().get(f"C2_fd{g}")
        if fp is None:
            pytest.skip("fingerprint missing")
        a, b, _ = oracle.config_operands("C2", grid=g)
        assert b is a and genmat.digests(a)["fingerprint"] == fp["a"]["fingerprint"]
