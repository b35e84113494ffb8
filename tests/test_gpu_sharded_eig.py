"""Column-sharded generalized eigensolve (em_sygv_range, the multi-GPU layout of
parallel.py): a rank's modes m_lo .. m_hi - 1 must equal the corresponding columns of the
single-device em_sygv_ex solve (same arithmetic per column: only the back-transforms are
restricted), for the banded (stencil) R and a dense R, the one-stage and the two-stage
tridiagonalisation, ragged ranges and empty ranges."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(l, r, lo=None, hi=None):
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    n = l.shape[0]
    dl, dr = nat.device_symmetric(l), nat.device_symmetric(r)
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    tau = nat.empty(n)
    if lo is None:
        v, ln, rn = nat.empty(n, n), nat.empty(n), nat.empty(n)
        nat.check(lib.em_sygv_ex(ctx, n, nat.ptr(dl), n, nat.ptr(dr), n, nat.ptr(tau), nat.ptr(v),
                                 n, nat.ptr(ln), nat.ptr(rn), None, n, 0, ctypes.byref(piv),
                                 ctypes.byref(which)), "em_sygv_ex")
        m = n
    else:
        m = hi - lo
        v, ln, rn = nat.empty(max(m, 1), n), nat.empty(max(m, 1)), nat.empty(max(m, 1))
        nat.check(lib.em_sygv_range(ctx, n, nat.ptr(dl), n, nat.ptr(dr), n, lo, hi, nat.ptr(tau),
                                    nat.ptr(v), n, nat.ptr(ln), nat.ptr(rn), None, n, 0,
                                    ctypes.byref(piv), ctypes.byref(which)), "em_sygv_range")
    return (tau.cpu().numpy(), v.cpu().numpy()[:m].T.copy(), ln.cpu().numpy()[:m],
            rn.cpu().numpy()[:m])


@pytest.mark.parametrize("two_stage", [False, True])
@pytest.mark.parametrize("dense_r", [False, True])
def test_range_columns_equal_full_solve(two_stage, dense_r):
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import plate_model
    lib, ctx = nat.load_library(), nat.context()
    m = plate_model(24, 10, 2, n_ports=1, n_sources=1, n_obs=4)  # N = 480, b = 20
    l, r = m["l_i"], m["r_i"]
    n = l.shape[0]
    if two_stage:
        nat.set_two_stage_min(0)
    if dense_r:
        nat.check(lib.em_config(ctx, 2, 1))
    try:
        tau, v, ln, rn = _solve(l, r)
        for lo, hi in ((0, n), (0, 161), (161, 320), (320, n), (0, 1), (n - 1, n), (7, 7)):
            t2, v2, l2, r2 = _solve(l, r, lo, hi)
            np.testing.assert_array_equal(t2, tau)
            if hi == lo:
                continue
            scale = np.abs(v).max()
            assert np.abs(v2 - v[:, lo:hi]).max() <= 1e-12 * scale, (lo, hi)
            assert np.max(np.abs(l2 - ln[lo:hi]) / ln[lo:hi]) < 1e-12
            assert np.max(np.abs(r2 - rn[lo:hi])) < 1e-12
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
        nat.check(lib.em_config(ctx, 2, 0))


def test_range_arguments_rejected():
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.errors import DeviceError
    n = 8
    a = np.eye(n)
    for lo, hi in ((-1, 3), (2, 9), (5, 4)):
        with pytest.raises(DeviceError):
            _solve(a, a, lo, hi)
    assert nat is not None
