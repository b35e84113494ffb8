"""Implicit-V eigensolve (em_sygv_implicit / em_sygv_implicit_band, modal.implicit_eig):
tau and V^T Y without forming V, U or the Q back-transforms (divide and conquer carries
U^T Y through its merges, csrc/stedc.cu stedc_apply). Each row of V^T Y is fixed up to the
mode's sign, so the checks are the sign- and rotation-invariant identities of the reference
basis (modal.py:46-81: V^T R V = I, V^T L V = diag(tau)):
  (V^T Y)^T (V^T Y) = Y^T R^-1 Y,   (V^T Y)^T diag(tau) (V^T Y) = Y^T R^-1 L R^-1 Y,
plus tau against the explicit solve and |V^T Y| row by row where the spectrum is simple."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plate(nx, ny, nz):
    from paper_2407_11993_b200 import synth
    m = synth.plate_model(nx, ny, nz, n_ports=0, n_sources=0, n_obs=1)
    return m["l_i"].full if hasattr(m["l_i"], "full") else m["l_i"], \
        m["r_i"].full if hasattr(m["r_i"], "full") else m["r_i"]


def _check_identities(l, r, y, tau, vy, tol=1e-9):
    ry = np.linalg.solve(r, y)
    g1 = vy.T @ vy
    g2 = vy.T @ (tau[:, None] * vy)
    e1 = y.T @ ry
    e2 = ry.T @ l @ ry
    assert np.max(np.abs(g1 - e1)) < tol * np.max(np.abs(e1))
    assert np.max(np.abs(g2 - e2)) < tol * np.max(np.abs(e2))


@pytest.mark.parametrize("grid,two_stage", [((10, 8, 2), False), ((10, 8, 2), True),
                                            ((30, 20, 4), False), ((30, 20, 4), True),
                                            ((45, 25, 4), True)])
def test_implicit_eig_identities_and_explicit_tau(grid, two_stage):
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal
    l, r = _plate(*grid)
    n = l.shape[0]
    rng = np.random.default_rng(7)
    y = rng.standard_normal((n, 9))
    if two_stage:
        nat.set_two_stage_min(0)
    try:
        tau, vy = modal.implicit_eig(l, r, y)
        basis = modal.generalized_eig(l, r)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    assert np.max(np.abs(tau - basis.tau) / basis.tau) < 1e-12
    _check_identities(l, r, y, tau, vy)
    # row by row up to sign against the explicit basis (simple spectrum)
    ve = basis.v.T @ y
    s = np.sign(np.sum(ve * vy, axis=1))
    s[s == 0] = 1
    assert np.max(np.abs(vy - s[:, None] * ve)) < 1e-8 * np.max(np.abs(ve))


@pytest.mark.parametrize("two_stage", [False, True])
def test_implicit_eig_degenerate_pencil(two_stage):
    """L = 3 R + a rank-2 term: all but two eigenvalues equal, so almost every secular
    pole deflates (rotations of close poles); the identities still hold."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal
    _, r = _plate(12, 10, 2)
    n = r.shape[0]
    rng = np.random.default_rng(3)
    u = rng.standard_normal((n, 2))
    l = 3.0 * r + r @ u @ u.T @ r * 1e-3
    l = 0.5 * (l + l.T)
    y = rng.standard_normal((n, 5))
    if two_stage:
        nat.set_two_stage_min(0)
    try:
        tau, vy = modal.implicit_eig(l, r, y)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    assert np.sum(np.abs(tau - 3.0) < 1e-9) == n - 2
    _check_identities(l, r, y, tau, vy, tol=1e-8)


def test_implicit_band_in_place_equals_dense():
    """R in band storage + L reduced in place (em_sygv_implicit_band, EM_SYGV_L_WORKSPACE:
    the memory plan of the N = 120,000 run) against the dense-R, copied-L solve."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal
    l, r = _plate(32, 16, 4)  # n = 2048: ld a multiple of 32, L is reduced in place
    n = l.shape[0]
    bw = 16 * 4
    assert np.all(np.tril(r, -bw - 1) == 0)
    y = np.random.default_rng(11).standard_normal((n, 6))
    for ts in (False, True):
        if ts:
            nat.set_two_stage_min(0)
        try:
            tau0, vy0 = modal.implicit_eig(l, r, y)
            tau1, vy1 = modal.implicit_eig(l, r, y, r_band=bw, l_workspace=True)
        finally:
            nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
        np.testing.assert_allclose(tau1, tau0, rtol=1e-13, atol=0)
        assert np.max(np.abs(np.abs(vy1) - np.abs(vy0))) < 1e-10 * np.max(np.abs(vy0))
        _check_identities(l, r, y, tau1, vy1)
