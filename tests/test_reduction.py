"""External-model reduction against the unmodified reference's
outputs (tests/golden/reduction.npz, tests/golden/make_golden.py case_reduction):
integer_kernel bit for bit (reduction.py:60-99), the lift E^T (E E^T)^-1 and its
rank checks (reduction.py:21-57) on CPU; project_external (reduction.py:143-183), whose
products run on the device GEMM, on the GPU."""
import numpy as np
import pytest

from tests.conftest import golden


def test_integer_kernel_equals_reference():
    from paper_2407_11993_b200.reduction import integer_kernel
    g = golden("reduction")
    cases = sorted({k.split("_")[-1] for k in g.files if k.startswith("ik_e_")}, key=int)
    assert len(cases) >= 10
    for t in cases:
        e, k_ref = g[f"ik_e_{t}"], g[f"ik_k_{t}"]
        k = integer_kernel(e)
        assert k.dtype == np.int64 and np.array_equal(k, k_ref), t
        assert not np.any(e @ k)  # exact null space


def test_integer_kernel_identity_block():
    """E = [0 .. 0 | I] (the plates' electrode coordinate) gives K = [I; 0]."""
    from paper_2407_11993_b200.reduction import integer_kernel
    n, p = 9, 2
    e = np.zeros((p, n + p), dtype=np.int64)
    e[:, n:] = np.eye(p, dtype=np.int64)
    k = integer_kernel(e)
    assert np.array_equal(k, np.vstack([np.eye(n, dtype=np.int64), np.zeros((p, n), np.int64)]))


@pytest.mark.gpu
def test_lift_matrix_and_rank_checks():
    """(linalg.cholesky / solve_cholesky run on the device)"""
    from paper_2407_11993_b200.errors import DimensionMismatch, RankDeficient
    from paper_2407_11993_b200.reduction import lift_electrode_currents, lift_matrix
    g = golden("reduction")
    lift = lift_matrix(g["lift_e"])
    assert np.abs(lift - g["lift_m"]).max() <= 1e-14 * np.abs(g["lift_m"]).max()
    i_d = np.array([0.3, -1.2])
    np.testing.assert_allclose(lift_electrode_currents(g["lift_e"], i_d), lift @ i_d,
                               rtol=1e-13, atol=1e-15)
    with pytest.raises(RankDeficient):
        lift_matrix(np.array([[1, 0, 1], [2, 0, 2]]))  # duplicated electrode
    with pytest.raises(DimensionMismatch):
        lift_electrode_currents(g["lift_e"], np.ones(3))
    assert lift_matrix(np.zeros((0, 4))).shape == (4, 0)


@pytest.mark.gpu
def test_project_external_matches_reference():
    from paper_2407_11993_b200.reduction import project_external
    g = golden("reduction")
    rm = project_external(g["px_r_x"], g["px_l_x"], g["px_e"], port_names=("a", "b"))
    assert np.array_equal(rm.k, g["px_k"])
    for ours, ref in ((rm.r_i.full, g["px_r_i"]), (rm.l_i.full, g["px_l_i"]),
                      (rm.r_d, g["px_r_d"]), (rm.l_d, g["px_l_d"]), (rm.lift, g["px_lift"])):
        assert ours.shape == ref.shape
        assert np.abs(ours - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0)
    assert rm.port_names == ("a", "b") and rm.n_internal == g["px_k"].shape[1]
