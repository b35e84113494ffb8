"""Device generalized eigensolve vs the reference (golden fixtures produced by
the unmodified reference) and the reference's own modal tests
(pkg/tests/test_modal.py). North-star tolerance: eigenvalues 1e-10 relative."""
import numpy as np
import pytest
from numpy.testing import assert_allclose

from tests.conftest import golden, modal_directions_match, rel_l2

pytestmark = pytest.mark.gpu


def random_spd(rng, n, shift=None):
    b = rng.standard_normal((n, n))
    return b @ b.T + (shift if shift is not None else n) * np.eye(n)


@pytest.mark.parametrize("name", ["plate_small", "plate_200", "tube_small", "tube_ref"])
def test_generalized_eig_matches_reference(name):
    from paper_2407_11993_b200.linalg import SymMatrix
    from paper_2407_11993_b200.modal import generalized_eig
    g = golden(name)
    mb = generalized_eig(SymMatrix(g["l_i"]), SymMatrix(g["r_i"]))
    assert np.max(np.abs(mb.tau - g["tau"]) / g["tau"]) < 1e-10
    assert np.all(np.diff(mb.tau) <= 0)
    assert_allclose(mb.l_n, g["l_n"], rtol=1e-10)
    assert_allclose(mb.r_n, g["r_n"], rtol=1e-10)
    # same invariant subspaces (tube modes are exactly degenerate in groups)
    assert modal_directions_match(g["v"], g["tau"], mb.v, tol=1e-7)
    # R-orthonormality and sign convention
    r = g["r_i"]
    gram = mb.v.T @ r @ mb.v
    assert np.abs(gram - np.eye(len(mb.tau))).max() < 1e-10
    idx = np.argmax(np.abs(mb.v), axis=0)
    assert np.all(mb.v[idx, np.arange(mb.v.shape[1])] > 0)
    assert_allclose(mb.vt_r, mb.v.T @ r, rtol=0, atol=1e-12 * np.abs(mb.vt_r).max())


def test_identity_and_diagonal_pairs():
    from paper_2407_11993_b200.modal import generalized_eig
    mb = generalized_eig(np.eye(3), np.eye(3))
    assert_allclose(mb.tau, 1.0)
    assert_allclose(np.abs(mb.v.T @ mb.v), np.eye(3), atol=1e-12)
    mb = generalized_eig(np.diag([2.0, 1.0]), np.eye(2))
    assert_allclose(mb.tau, [2.0, 1.0])
    assert_allclose(mb.l_n, mb.tau, rtol=1e-14)
    assert_allclose(mb.r_n, 1.0, rtol=1e-14)


@pytest.mark.parametrize("n", [10, 100, 333])
def test_seeded_pair_residual_and_gram(rng, n):
    from paper_2407_11993_b200.modal import generalized_eig
    l = random_spd(rng, n)
    r = random_spd(rng, n)
    mb = generalized_eig(l, r)
    resid = np.linalg.norm(l @ mb.v - r @ mb.v @ np.diag(mb.tau))
    assert resid <= 1e-9 * np.linalg.norm(l)
    for gram in (mb.v.T @ l @ mb.v, mb.v.T @ r @ mb.v):
        off = np.abs(gram - np.diag(np.diag(gram))).max()
        assert off < 1e-10 * np.abs(np.diag(gram)).min()
    assert np.all(np.diff(mb.tau) <= 1e-12 * mb.tau[0])
    assert np.all(mb.tau > 0)


def test_non_spd_rejected_with_reference_messages():
    from paper_2407_11993_b200.errors import NotPositiveDefinite
    from paper_2407_11993_b200.modal import generalized_eig
    with pytest.raises(NotPositiveDefinite) as exc:
        generalized_eig(np.eye(2), np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert "modal resistance matrix" in str(exc.value) and exc.value.pivot == 1
    with pytest.raises(NotPositiveDefinite) as exc:
        generalized_eig(np.array([[1.0, 2.0], [2.0, 1.0]]), np.eye(2))
    assert "modal inductance matrix" in str(exc.value) and exc.value.pivot == 1


def test_doubling_resistivity_halves_every_tau():
    """test_modal.py:68-75 on the tube fixture: R -> 2R halves tau, same directions."""
    from paper_2407_11993_b200.modal import generalized_eig
    g = golden("tube_small")
    mb1 = generalized_eig(g["l_i"], g["r_i"])
    mb2 = generalized_eig(g["l_i"], 2.0 * g["r_i"])
    assert_allclose(mb2.tau, mb1.tau / 2, rtol=1e-12)
    assert modal_directions_match(mb1.v, mb1.tau, mb2.v, tol=1e-10)


def test_monotonicity_under_resistance_increase(rng):
    """test_modal.py:77-93 restated on plates: raising R elementwise-diagonally
    never raises any time constant."""
    from paper_2407_11993_b200.modal import generalized_eig
    g = golden("plate_small")
    t1 = generalized_eig(g["l_i"], g["r_i"]).tau
    for _ in range(3):
        bump = np.diag(rng.uniform(0.0, 3.0, size=g["r_i"].shape[0]) * 1e-3)
        t2 = generalized_eig(g["l_i"], g["r_i"] + bump).tau
        assert np.all(t2 <= t1 * (1 + 1e-10))


def test_modal_transform_round_trips(rng):
    from paper_2407_11993_b200.errors import DimensionMismatch
    from paper_2407_11993_b200.modal import from_modal, generalized_eig, to_modal
    for name in ("tube_small", "tube_ref"):
        g = golden(name)
        mb = generalized_eig(g["l_i"], g["r_i"])
        assert_allclose(from_modal(mb, to_modal(mb, np.zeros(mb.n_modes))), 0.0)
        m = to_modal(mb, mb.v[:, 0].copy())
        expected = np.zeros(mb.n_modes)
        expected[0] = mb.r_n[0]
        assert_allclose(m, expected, atol=1e-10)
        x = rng.standard_normal(mb.n_modes)
        y = from_modal(mb, to_modal(mb, x))
        assert np.linalg.norm(y - x) < 1e-10 * np.linalg.norm(x)
        with pytest.raises(DimensionMismatch):
            to_modal(mb, np.zeros(mb.n_modes + 1))


def test_modal_forcing_scalar_case_and_projection(rng):
    from paper_2407_11993_b200 import reduction
    from paper_2407_11993_b200.linalg import SymMatrix
    from paper_2407_11993_b200.modal import ModalBasis, drive_rhs, generalized_eig, modal_forcing
    rm = reduction.ReducedModel(r_i=SymMatrix(np.eye(1)), l_i=SymMatrix(np.eye(1)),
                                r_d=np.zeros((1, 1)), l_d=np.ones((1, 1)), m0=np.zeros((1, 0)),
                                lift=np.ones((1, 1)), k=np.eye(1), port_names=("p",))
    mb = ModalBasis(v=np.eye(1), tau=np.ones(1), l_n=np.ones(1), r_n=np.ones(1), vt_r=np.eye(1))
    f = modal_forcing(mb, rm, i_d=np.zeros(1), delta_i_d=np.ones(1), delta_i0=np.zeros(0),
                      dt=0.1, theta=1.0)
    assert_allclose(f, [-1.0])
    g = golden("tube_small")
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], None, port_names=("p",))
    mb = generalized_eig(rm.l_i, rm.r_i)
    i_d, d_id = rng.standard_normal(1), rng.standard_normal(1)
    f = modal_forcing(mb, rm, i_d, d_id, np.zeros(0), 1 / 30000, 0.7)
    rhs = drive_rhs(rm, i_d, d_id, np.zeros(0), 1 / 30000, 0.7)
    assert_allclose(f, mb.v.T @ rhs, rtol=1e-12, atol=1e-18 + 1e-13 * np.abs(f).max())


@pytest.mark.skipif(not __import__("os").path.exists(
    __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "c1.npz")),
    reason="c1 golden absent")
def test_c1_eigenvalues_match_reference_jacobi():
    """Config C1 (N=2000): device eigenvalues vs the reference's Jacobi, 1e-10."""
    from paper_2407_11993_b200.modal import generalized_eig
    from paper_2407_11993_b200.synth import plate_model
    g = golden("c1")
    m = plate_model(40, 25, 2, n_ports=0, n_sources=1, n_obs=16)
    mb = generalized_eig(m["l_i"], m["r_i"])
    assert np.max(np.abs(mb.tau - g["tau"]) / g["tau"]) < 1e-10
    assert_allclose(mb.l_n, g["l_n"], rtol=1e-10)
    assert rel_l2(mb.v[:, :4], g["v_lead"]) < 1e-8


def test_certificate_deferred_only_when_provably_redundant():
    """EM_CFG_L_CERTIFICATE (modal.py:69-70): by default the Cholesky of L is skipped when
    the solved spectrum proves it succeeds (plate: tau > 0, R diagonally dominant, well
    conditioned) — same basis as with the certificate forced; a non-SPD L still raises the
    reference's error with the reference's pivot (then after the eigensolve)."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal, reduction
    from paper_2407_11993_b200.errors import NotPositiveDefinite
    from oracle import oracle as O
    g = golden("plate_200")
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], g["m0"])
    lib, ctx = nat.load_library(), nat.context()
    nat.profile(1)
    b0 = modal.generalized_eig(rm.l_i, rm.r_i)
    st0 = nat.stage_times()
    nat.check(lib.em_config(ctx, 5, 1))
    try:
        nat.profile(1)
        b1 = modal.generalized_eig(rm.l_i, rm.r_i)
        st1 = nat.stage_times()
    finally:
        nat.check(lib.em_config(ctx, 5, 0))
        nat.profile(0)
    assert "potrf_L" not in st0 and "potrf_L" in st1
    np.testing.assert_array_equal(b0.tau, b1.tau)
    # an indefinite L: the deferred certificate names the reference's pivot
    lbad = g["l_i"].copy()
    lbad[7, 7] = -1.0
    with pytest.raises(O.OracleNotPositiveDefinite) as ref:
        O.cholesky(O.sym_mirror(lbad), what="modal inductance matrix")
    with pytest.raises(NotPositiveDefinite) as e:
        modal.generalized_eig(lbad, g["r_i"])
    assert e.value.pivot == ref.value.pivot and "inductance" in str(e.value)


@pytest.mark.parametrize("dense_r", [False, True])
def test_device_inputs_read_only_the_lower_triangles(dense_r):
    """SymMatrix semantics on the device path (E/linalg.py:24-59, modal.py:46-81): L and R
    given as device tensors with garbage above the diagonal give the same basis as the
    clean symmetric inputs (the library reads lower triangles only: band detection, the
    factor, the reduction, the CSR copy behind r_n); em_sym_mirror_lower restores
    symmetry in place."""
    import torch
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal
    from paper_2407_11993_b200.synth import plate_model
    m = plate_model(30, 12, 2, n_ports=0, n_sources=1, n_obs=4)  # N = 720, band 24
    l, r = m["l_i"], m["r_i"]
    n = l.shape[0]
    rng = np.random.default_rng(4)
    junk = np.triu(rng.standard_normal((n, n)), 1)
    # column-major device buffers: element (i, j) at j*n + i, i.e. the transpose's bytes;
    # garbage strictly above the diagonal
    lg = torch.from_numpy(np.ascontiguousarray((l + junk).T)).cuda()
    rg = torch.from_numpy(np.ascontiguousarray((r + 1e-3 * junk).T)).cuda()
    lib, ctx = nat.load_library(), nat.context()
    if dense_r:
        nat.check(lib.em_config(ctx, 2, 1))
    try:
        clean = modal.generalized_eig(torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda())
        dirty = modal.generalized_eig(lg, rg)
    finally:
        nat.check(lib.em_config(ctx, 2, 0))
    np.testing.assert_array_equal(dirty.tau, clean.tau)
    np.testing.assert_array_equal(dirty.l_n, clean.l_n)
    assert np.abs(dirty.r_n - clean.r_n).max() < 1e-14
    assert np.abs(dirty.v - clean.v).max() <= 1e-12 * np.abs(clean.v).max()
    nat.check(lib.em_sym_mirror_lower(ctx, n, nat.ptr(lg), n), "em_sym_mirror_lower")
    np.testing.assert_array_equal(lg.cpu().numpy(), l.T)
