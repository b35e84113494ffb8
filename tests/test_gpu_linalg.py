"""Device dense linear algebra vs the reference's known answers
(pkg/tests/test_linalg.py) and the golden fixtures."""
import ctypes

import numpy as np
import pytest
from numpy.testing import assert_allclose

from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [0, 2, 3, 4, 5])
def test_dgemm_all_transposes_vs_numpy(rng, cfg):
    """em_config debug key 96 selects the tile configuration: 0 the default (64x64 tiles,
    three CTAs per SM for a transposed A, four otherwise), 2 64x64 / four CTAs, 3 128x64,
    4 64x64 / three CTAs, 5 the paired-fragment tiles (16-byte operands: the even leading
    dimensions below); (40, 70, 6000) takes split-K."""
    from paper_2407_11993_b200 import _native as nat
    ctx = nat.context()
    lib = nat.load_library()
    nat.check(lib.em_config(ctx, 96, cfg))
    try:
        _dgemm_cases(rng, nat, ctx, lib)
    finally:
        nat.check(lib.em_config(ctx, 96, 0))


def _dgemm_cases(rng, nat, ctx, lib):
    for (m, n, k) in ((1, 1, 1), (37, 129, 300), (257, 131, 17), (300, 300, 300),
                      (130, 200, 1100), (40, 70, 6000), (256, 192, 64), (200, 330, 146)):
        for ta in (0, 1):
            for tb in (0, 1):
                a = rng.standard_normal((k, m) if ta else (m, k))
                b = rng.standard_normal((n, k) if tb else (k, n))
                c0 = rng.standard_normal((m, n))
                da, db, dc = nat.device_colmajor(a), nat.device_colmajor(b), nat.device_colmajor(c0)
                lda, ldb = a.shape[0], b.shape[0]
                nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 0.5, nat.ptr(da), lda, nat.ptr(db),
                                       ldb, -2.0, nat.ptr(dc), m))
                ref = 0.5 * (a.T if ta else a) @ (b.T if tb else b) - 2.0 * c0
                got = nat.host_colmajor(dc, m, n)
                assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_cholesky_known_answers_match_reference():
    from paper_2407_11993_b200.linalg import cholesky
    g = golden("kat_linalg")
    for n in (1, 2, 5, 17, 40):
        a = g[f"chol_a_{n}"]
        c = cholesky(a).c
        assert_allclose(c, g[f"chol_c_{n}"], rtol=1e-13, atol=1e-13 * np.abs(a).max())
        assert np.linalg.norm(c @ c.T - a) <= 1e-12 * np.linalg.norm(a)
        assert np.array_equal(c, np.tril(c))


def test_cholesky_identity_and_indefinite_pivot():
    from paper_2407_11993_b200.errors import NotPositiveDefinite
    from paper_2407_11993_b200.linalg import cholesky
    assert_allclose(cholesky(np.eye(3)).c, np.eye(3))
    with pytest.raises(NotPositiveDefinite) as exc:
        cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]), what="modal resistance matrix")
    assert exc.value.pivot == 1
    assert "modal resistance matrix" in str(exc.value)


@pytest.mark.parametrize("n,bad", [(200, 0), (300, 131), (400, 255), (700, 699)])
def test_cholesky_failing_pivot_index_across_blocks(rng, n, bad):
    """The first non-positive pivot is reported with the reference's index, also
    when it lies in a later 128-block of the blocked factorisation."""
    from oracle import oracle as O
    from paper_2407_11993_b200.errors import NotPositiveDefinite
    from paper_2407_11993_b200.linalg import cholesky
    b = rng.standard_normal((n, n)) / np.sqrt(n)
    a = b @ b.T + np.eye(n)
    a[bad, bad] = -1.0
    with pytest.raises(NotPositiveDefinite) as exc:
        cholesky(a)
    with pytest.raises(O.OracleNotPositiveDefinite) as ref:
        O.cholesky(a)
    assert exc.value.pivot == ref.value.pivot == bad


@pytest.mark.parametrize("n", [1, 5, 64, 129, 500, 1000])
def test_cholesky_reconstruction_many_sizes(rng, n):
    from paper_2407_11993_b200.linalg import cholesky
    b = rng.standard_normal((n, n))
    a = b.T @ b + n * np.eye(n)
    c = cholesky(a).c
    assert np.linalg.norm(c @ c.T - a) <= 1e-12 * np.linalg.norm(a)


def test_solve_cholesky_residual_and_linearity(rng):
    from paper_2407_11993_b200.errors import DimensionMismatch
    from paper_2407_11993_b200.linalg import LowerTriangular, cholesky, solve_cholesky
    assert_allclose(solve_cholesky(LowerTriangular(np.eye(3)), np.array([1.0, 2.0, 3.0])),
                    [1, 2, 3])
    n = 300
    b = rng.standard_normal((n, n))
    a = b.T @ b + n * np.eye(n)
    c = cholesky(a)
    rhs = rng.standard_normal(n)
    x = solve_cholesky(c, rhs)
    assert np.linalg.norm(a @ x - rhs) / np.linalg.norm(rhs) < 1e-12
    b1, b2 = rng.standard_normal(n), rng.standard_normal(n)
    lhs = solve_cholesky(c, 2.5 * b1 - 1.25 * b2)
    r2 = 2.5 * solve_cholesky(c, b1) - 1.25 * solve_cholesky(c, b2)
    assert np.linalg.norm(lhs - r2) <= 1e-12 * max(np.linalg.norm(lhs), 1.0)
    with pytest.raises(DimensionMismatch):
        solve_cholesky(cholesky(np.eye(3)), np.ones(4))


def test_trsm_both_directions_vs_oracle(rng):
    from oracle import oracle as O
    from paper_2407_11993_b200 import _native as nat
    n, m = 333, 77
    b0 = rng.standard_normal((n, n)) / np.sqrt(n)
    c = np.linalg.cholesky(b0 @ b0.T + np.eye(n))
    rhs = rng.standard_normal((n, m))
    ctx = nat.context()
    lib = nat.load_library()
    for trans in (0, 1):
        dc, db = nat.device_colmajor(c), nat.device_colmajor(rhs)
        nat.check(lib.em_trsm_lower(ctx, trans, n, m, nat.ptr(dc), n, nat.ptr(db), n))
        got = nat.host_colmajor(db, n, m)
        ref = np.ascontiguousarray(rhs.copy())
        if trans:
            O.lib().orc_tri_lower_t_solve_mat(O._p(np.ascontiguousarray(c)), O._p(ref), n, m)
        else:
            O.lib().orc_tri_lower_solve_mat(O._p(np.ascontiguousarray(c)), O._p(ref), n, m)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_sym_eig_known_answers():
    from paper_2407_11993_b200.linalg import sym_eig
    g = golden("kat_linalg")
    lam, u = sym_eig(np.diag([3.0, 1.0, 2.0]))
    assert_allclose(lam, [3.0, 2.0, 1.0])
    assert_allclose(np.abs(u), np.eye(3)[:, [0, 2, 1]], atol=1e-14)
    lam, u = sym_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert_allclose(lam, [3.0, 1.0], rtol=1e-14)
    assert u[0, 1] * u[1, 1] < 0
    a = g["eig_a_seeded"]
    lam, u = sym_eig(a)
    assert_allclose(lam, g["eig_lam_seeded"], rtol=1e-12, atol=1e-13)
    assert np.linalg.norm(a @ u - u @ np.diag(lam)) <= 1e-10 * np.linalg.norm(a)
    assert np.abs(u.T @ u - np.eye(12)).max() < 1e-12


@pytest.mark.parametrize("n", [63, 64, 65, 130, 257, 1000, 2000])
def test_sym_eig_divide_and_conquer_sizes(rng, n):
    from paper_2407_11993_b200.linalg import sym_eig
    a = rng.standard_normal((n, n))
    a = (a + a.T) / 2
    lam, u = sym_eig(a)
    ref = np.linalg.eigvalsh(a)[::-1]
    assert np.abs(lam - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.linalg.norm(a @ u - u * lam) <= 1e-11 * np.linalg.norm(a)
    assert np.abs(u.T @ u - np.eye(n)).max() < 1e-11
    assert np.all(np.diff(lam) <= 0)


def test_sym_eig_degenerate_spectrum(rng):
    """Exactly repeated eigenvalues (heavy deflation): clusters of 1, 3, 10, 40."""
    from paper_2407_11993_b200.linalg import sym_eig
    n = 300
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.concatenate([np.full(40, 2.0), np.full(10, -1.0), np.full(3, 0.5),
                        rng.standard_normal(n - 53)])
    a = (q * w) @ q.T
    a = (a + a.T) / 2
    lam, u = sym_eig(a)
    assert np.abs(np.sort(lam) - np.sort(w)).max() < 1e-12 * np.abs(w).max() * n
    assert np.linalg.norm(a @ u - u * lam) <= 1e-11 * np.linalg.norm(a)
    assert np.abs(u.T @ u - np.eye(n)).max() < 1e-11


@pytest.mark.parametrize("n", [1, 63, 64, 65, 1000, 1111])
def test_symv_lower_reads_only_lower_triangle(rng, n):
    """em_symv_lower == A_sym x with garbage in the upper triangle (td1_step_kernel's R @ state)."""
    from paper_2407_11993_b200 import _native as nat
    a = rng.standard_normal((n, n))
    sym = np.tril(a) + np.tril(a, -1).T
    garbage = sym.copy()
    garbage[np.triu_indices(n, 1)] = 1e300  # must never be read
    x = rng.standard_normal(n)
    y0 = rng.standard_normal(n)
    ad = nat.device_colmajor(garbage)
    xd, yd = nat.device_vector(x), nat.device_vector(y0)
    nat.check(nat.load_library().em_symv_lower(nat.context(), n, -0.5, nat.ptr(ad), n,
                                                nat.ptr(xd), 2.0, nat.ptr(yd)))
    ref = -0.5 * sym @ x + 2.0 * y0
    assert np.abs(yd.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.fixture
def two_stage():
    """Force the two-stage (dense -> band -> tridiagonal) reduction for every n > 128."""
    from paper_2407_11993_b200 import _native as nat
    nat.set_two_stage_min(0)
    yield
    nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)


@pytest.mark.parametrize("n", [129, 200, 257, 700, 1500])
def test_two_stage_sym_eig(rng, n, two_stage):
    from paper_2407_11993_b200.linalg import sym_eig
    a = rng.standard_normal((n, n))
    a = (a + a.T) / 2
    lam, u = sym_eig(a)
    ref = np.linalg.eigvalsh(a)[::-1]
    assert np.abs(lam - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.linalg.norm(a @ u - u * lam) <= 1e-11 * np.linalg.norm(a)
    assert np.abs(u.T @ u - np.eye(n)).max() < 1e-11


def test_two_stage_degenerate_spectrum(rng, two_stage):
    from paper_2407_11993_b200.linalg import sym_eig
    n = 400
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.concatenate([np.full(70, 2.0), np.full(10, -1.0), rng.standard_normal(n - 80)])
    a = (q * w) @ q.T
    a = (a + a.T) / 2
    lam, u = sym_eig(a)
    assert np.abs(np.sort(lam) - np.sort(w)).max() < 1e-12 * np.abs(w).max() * n
    assert np.linalg.norm(a @ u - u * lam) <= 1e-11 * np.linalg.norm(a)
    assert np.abs(u.T @ u - np.eye(n)).max() < 1e-11


@pytest.mark.parametrize("name", ["plate_200", "tube_ref"])
def test_two_stage_generalized_eig_matches_reference(name, two_stage):
    from tests.conftest import modal_directions_match
    from paper_2407_11993_b200.modal import generalized_eig
    g = golden(name)
    mb = generalized_eig(g["l_i"], g["r_i"])
    assert np.max(np.abs(mb.tau - g["tau"]) / g["tau"]) < 1e-10
    assert modal_directions_match(g["v"], g["tau"], mb.v, tol=1e-7)
