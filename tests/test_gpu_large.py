"""Large-order eigensolve on the device: N = 46,400 > 46,341, so N^2 exceeds 2^31 and
every N x N index in the eigensolver must be 64-bit. Checked through properties that
do not need a CPU eigensolve at this size (LAPACK would take hours):
R-orthonormality V^T R V = I, the residual L V - R V diag(tau), descending order,
the sign convention (largest-|.| entry positive, modal.py:74-78), l_n = diag(V^T L V)
and r_n = diag(V^T R V). Also covers the memory-lean buffer plan (eigenvectors formed
in the output buffer, no V^T R) that lets C3 (N = 50,000) fit one B200.

The residual/Gram products use torch matmul: test infrastructure, not the product."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_lazy_vt_r_matches_eager():
    from paper_2407_11993_b200.linalg import SymMatrix
    from paper_2407_11993_b200.modal import generalized_eig
    from tests.conftest import golden
    g = golden("plate_200")
    a = generalized_eig(SymMatrix(g["l_i"]), SymMatrix(g["r_i"]), vt_r="eager")
    b = generalized_eig(SymMatrix(g["l_i"]), SymMatrix(g["r_i"]), vt_r="lazy")
    assert np.array_equal(a.tau, b.tau)
    assert np.array_equal(a.v, b.v)
    np.testing.assert_allclose(b.vt_r, a.vt_r, rtol=0, atol=1e-13 * np.abs(a.vt_r).max())


@pytest.mark.parametrize("two_stage", [True, False])
def test_eigensolve_beyond_int32_squared(two_stage):
    """Both tridiagonalisations at N = 46,400: the two-stage path (the default from
    N = 40,000 when its storage fits) and the one-stage path."""
    import torch
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model
    # the previous case's N x N tensors sit in torch's cache and the eigensolver's
    # workspace in the library's pool (em_config debug key 99 trims it)
    torch.cuda.empty_cache()
    nat.check(nat.load_library().em_config(nat.context(), 99, 0))
    free = torch.cuda.mem_get_info()[0]
    m = device_plate_model(116, 100, 4, n_ports=0, n_sources=0, n_obs=1)
    L, R = m["l_i"], m["r_i"]
    n = L.shape[0]
    assert n * n > 2 ** 31
    if free < 7.5 * 8.0 * n * n:
        pytest.skip("device too small for the 7 N^2 eigensolve at N = 46,400")
    lib, ctx = nat.load_library(), nat.context()
    tau, ln, rn = nat.empty(n), nat.empty(n), nat.empty(n)
    V = nat.empty(n, n)
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    nat.set_two_stage_min(0 if two_stage else 2**62)
    try:
        nat.profile(2)
        nat.check(lib.em_sygv(ctx, n, nat.ptr(L), n, nat.ptr(R), n, nat.ptr(tau), nat.ptr(V),
                              n, nat.ptr(ln), nat.ptr(rn), None, n, ctypes.byref(piv),
                              ctypes.byref(which)), "em_sygv")
        torch.cuda.synchronize()
        stages = nat.stage_times()
        nat.profile(0)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    # the requested path ran (stage 2 of the two-stage reduction is timed as sb2st)
    assert ("sb2st" in stages) == two_stage, sorted(stages)
    # column-major V: row j of the torch tensor is mode j
    Vt = V
    assert bool(torch.all(tau[1:] <= tau[:-1]))
    assert bool(torch.all(tau > 0))
    # sign convention on every mode
    idx = Vt.abs().argmax(dim=1)
    assert bool(torch.all(Vt.gather(1, idx[:, None]) > 0))
    worst_gram = worst_res = 0.0
    lnorm = torch.linalg.matrix_norm(L).item()
    cb = 4096
    for c0 in range(0, n, cb):
        blk = Vt[c0:c0 + cb]                  # (b, n): modes c0.. as rows
        rv = blk @ R                           # (R v)^T, R symmetric
        gram = rv @ Vt.T                       # (b, n) block of V^T R V
        gram[:, c0:c0 + cb] -= torch.eye(blk.shape[0], device=gram.device, dtype=gram.dtype)
        worst_gram = max(worst_gram, gram.abs().max().item())
        lv = blk @ L
        res = lv - tau[c0:c0 + cb, None] * rv
        worst_res = max(worst_res, torch.linalg.norm(res, dim=1).max().item())
        # l_n, r_n against the direct quadratic forms
        torch.testing.assert_close(ln[c0:c0 + cb], (lv * blk).sum(dim=1), rtol=1e-10, atol=0)
        torch.testing.assert_close(rn[c0:c0 + cb], (rv * blk).sum(dim=1), rtol=1e-10, atol=0)
        del rv, gram, lv, res
    assert worst_gram < 1e-9, worst_gram
    assert worst_res < 1e-9 * lnorm, (worst_res, lnorm)


@pytest.mark.parametrize("sparse_r", [True, False])
def test_r_workspace_mode_identical_and_restores_r(sparse_r):
    """EM_SYGV_R_WORKSPACE: the stencil R holds its own factor during the solve and is
    restored bit for bit from the CSR copy; results identical to the default mode. A
    dense R (no CSR) silently takes the copy path."""
    import torch
    from paper_2407_11993_b200 import _native as nat
    from tests.conftest import golden
    g = golden("plate_200")
    r = g["r_i"] if sparse_r else g["r_i"] + 1e-12 * np.ones_like(g["r_i"])
    n = r.shape[0]
    lib, ctx = nat.load_library(), nat.context()
    L = nat.device_symmetric(g["l_i"])
    outs = []
    for flags in (0, 1):
        R = nat.device_symmetric(r)
        R0 = R.clone()
        tau, ln, rn, V, VtR = (nat.empty(n), nat.empty(n), nat.empty(n), nat.empty(n, n),
                               nat.empty(n, n))
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        nat.check(lib.em_sygv_ex(ctx, n, nat.ptr(L), n, nat.ptr(R), n, nat.ptr(tau), nat.ptr(V),
                                 n, nat.ptr(ln), nat.ptr(rn), nat.ptr(VtR), n, flags,
                                 ctypes.byref(piv), ctypes.byref(which)), "em_sygv_ex")
        torch.cuda.synchronize()
        assert torch.equal(R, R0)
        outs.append([x.cpu().numpy() for x in (tau, ln, rn, V, VtR)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def _sygv_dev(L, R, n, flags=0):
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    tau, ln, rn, V = nat.empty(n), nat.empty(n), nat.empty(n), nat.empty(n, n)
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    rc = lib.em_sygv_ex(ctx, n, nat.ptr(L), n, nat.ptr(R), n, nat.ptr(tau), nat.ptr(V), n,
                        nat.ptr(ln), nat.ptr(rn), None, n, flags, ctypes.byref(piv),
                        ctypes.byref(which))
    return rc, piv.value, which.value, [x.cpu().numpy() for x in (tau, ln, rn, V)]


@pytest.mark.parametrize("grid", [(32, 16, 4), (21, 13, 5)])
def test_banded_r_path_matches_dense_path(grid):
    """Banded Cholesky of the stencil R + banded two-sided reduction (the reference's
    G^-1 (G^-1 L)^T, (B + B^T)/2 sequence) + banded back-transform against the dense
    path (EM_CFG_BAND_OFF) on the same plate; a ragged last block (N = 1365)."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model
    m = device_plate_model(*grid, n_ports=0, n_sources=0, n_obs=1)
    L, R = m["l_i"], m["r_i"]
    n = L.shape[0]
    lib, ctx = nat.load_library(), nat.context()
    outs = []
    for off in (1, 0):
        nat.check(lib.em_config(ctx, 2, off))
        rc, _, _, o = _sygv_dev(L, R, n)
        nat.check(rc)
        outs.append(o)
    nat.check(lib.em_config(ctx, 2, 0))
    (t0, l0, r0, v0), (t1, l1, r1, v1) = outs
    assert np.max(np.abs(t1 - t0) / t0) < 1e-12
    np.testing.assert_allclose(l1, l0, rtol=1e-11)
    np.testing.assert_allclose(r1, r0, rtol=1e-11)
    # modes of well-separated eigenvalues agree column by column (sign-fixed)
    gap = np.minimum(np.abs(np.diff(t0, prepend=np.inf)), np.abs(np.diff(t0, append=-np.inf)))
    sep = gap > 1e-6 * t0
    err = np.abs(v1 - v0).max(axis=1)  # host (n, n) rows = modes
    assert np.all(err[sep] < 1e-7 * np.abs(v0).max())


@pytest.mark.parametrize("two_stage", [False, True])
def test_banded_r_workspace_holds_reduced_matrix_and_is_restored(two_stage):
    """EM_SYGV_R_WORKSPACE with a BANDED stencil R (factor in band storage of its own): R's
    dense storage holds the reduced matrix during the eigensolve (N = 2,048: columns
    256-byte aligned) and comes back bit for bit from the CSR copy; tau, l_n, r_n, V are
    identical to the default mode, on the one-stage and the two-stage tridiagonalisation."""
    import torch
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model
    m = device_plate_model(32, 16, 4, n_ports=0, n_sources=0, n_obs=1)
    L, R = m["l_i"], m["r_i"]
    n = L.shape[0]
    assert n % 32 == 0
    R0 = R.clone()
    if two_stage:
        nat.set_two_stage_min(0)
    try:
        rc0, _, _, o0 = _sygv_dev(L, R, n, flags=0)
        rc1, _, _, o1 = _sygv_dev(L, R, n, flags=nat.EM_SYGV_R_WORKSPACE)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    nat.check(rc0)
    nat.check(rc1)
    torch.cuda.synchronize()
    assert torch.equal(R, R0)
    for a, b in zip(o0, o1):
        assert np.array_equal(a, b)


def test_banded_r_not_pd_reports_the_dense_pivot():
    """A banded R that is not positive definite: same failing pivot (the reference's
    first failing Crout column, cholesky_kernel _kernels.py:18-36) on both paths."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model
    m = device_plate_model(32, 16, 4, n_ports=0, n_sources=0, n_obs=1)
    L, R = m["l_i"], m["r_i"].clone()
    n = L.shape[0]
    R[700, 700] = -1.0  # column 700 of the lower triangle (row-major == column-major)
    lib, ctx = nat.load_library(), nat.context()
    res = []
    for off in (1, 0):
        nat.check(lib.em_config(ctx, 2, off))
        rc, piv, which, _ = _sygv_dev(L, R, n)
        res.append((rc, piv, which))
    nat.check(lib.em_config(ctx, 2, 0))
    assert res[0] == res[1] == (nat.EM_ERR_NOT_PD, 700, 0)


def test_banded_path_l_certificate_errors_and_order():
    """With a banded R (banded factor, dense L certificate): a non-SPD L
    still reports the dense path's pivot with which = 1, and a non-SPD R still wins
    (the reference checks R first, modal.py:61-70)."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model
    m = device_plate_model(32, 16, 4, n_ports=0, n_sources=0, n_obs=1)
    n = m["l_i"].shape[0]
    L = m["l_i"].clone()
    L[900, 900] = -1.0
    lib, ctx = nat.load_library(), nat.context()
    res = []
    for off in (1, 0):
        nat.check(lib.em_config(ctx, 2, off))
        rc, piv, which, _ = _sygv_dev(L, m["r_i"], n)
        res.append((rc, piv, which))
    assert res[0] == res[1] and res[1][0] == nat.EM_ERR_NOT_PD and res[1][2] == 1
    R = m["r_i"].clone()
    R[300, 300] = -1.0
    rc, piv, which, _ = _sygv_dev(L, R, n)
    nat.check(lib.em_config(ctx, 2, 0))
    assert (rc, piv, which) == (nat.EM_ERR_NOT_PD, 300, 0)
    # and a clean solve right after the failed calls
    rc, _, _, (tau, _, _, _) = _sygv_dev(m["l_i"], m["r_i"], n)
    nat.check(rc)
    assert np.all(tau > 0)
