"""The tridiagonalisation's alternative code paths (em_config debug key 98: bit0 the
non-TMA symv, bit1 no programmatic dependent launch, bit2 no CUDA graph, bit3 the
4-launch column chain) against LAPACK on awkward sizes, including an odd leading
dimension (no TMA) and orders that are not multiples of the 64/128 tiles."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _syev(a, lda=None):
    import torch
    from paper_2407_11993_b200 import _native as nat
    n = a.shape[0]
    lda = lda or n
    buf = np.zeros((n, lda))  # column-major n x n with leading dimension lda
    buf[:, :n] = a.T
    ad = nat.device_vector(buf.reshape(-1))
    w = torch.empty(max(n, 1), device="cuda", dtype=torch.float64)
    u = torch.empty(max(n * n, 1), device="cuda", dtype=torch.float64)
    lib, ctx = nat.load_library(), nat.context()
    nat.check(lib.em_syev(ctx, n, nat.ptr(ad), lda, nat.ptr(w), nat.ptr(u), n), "em_syev")
    return w.cpu().numpy()[:n], u.cpu().numpy()[:n * n].reshape(n, n).T


@pytest.mark.parametrize("flags", [0, 1, 2, 4, 8, 15])
@pytest.mark.parametrize("n", [1, 2, 3, 65, 130, 333, 1100])
def test_sytrd_paths_match_lapack(flags, n):
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    nat.check(lib.em_config(ctx, 98, flags))
    try:
        rng = np.random.default_rng(n * 31 + flags)
        b = rng.standard_normal((n, n))
        a = b + b.T
        w, u = _syev(a)
        ref = np.sort(np.linalg.eigvalsh(a))[::-1]
        scale = max(1.0, np.abs(ref).max())
        assert np.max(np.abs(w - ref)) < 1e-12 * scale * max(n, 1)
        assert np.max(np.abs(u.T @ u - np.eye(n))) < 1e-12 * max(n, 1)
        assert np.max(np.abs(a @ u - u * w)) < 1e-11 * scale * max(n, 1)
    finally:
        nat.check(lib.em_config(ctx, 98, 0))


def test_sytrd_odd_leading_dimension():
    """lda odd: the TMA map is refused (stride not a multiple of 16 B) and the
    register-prefetch symv runs instead."""
    rng = np.random.default_rng(5)
    n = 300
    b = rng.standard_normal((n, n))
    a = b + b.T
    w, u = _syev(a, lda=n + 1)
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    assert np.max(np.abs(w - ref)) < 1e-12 * np.abs(ref).max() * n


@pytest.mark.parametrize("n", [2500, 4097])
def test_sytrd_larger_orders(n):
    """Several panels with trailing orders past one tile wave (every CTA of the symv busy)
    and the L2 policy switch (EM_CFG_SYMV_L2_KEEP_MB: no hints vs evict_first + keep)."""
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    a = b + b.T
    w, u = _syev(a)
    nat.check(lib.em_config(ctx, 3, -1))
    try:
        w2, _ = _syev(a)
    finally:
        nat.check(lib.em_config(ctx, 3, 32))
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    assert np.max(np.abs(w - ref)) < 1e-12 * np.abs(ref).max() * n
    assert np.array_equal(w, w2)  # cache hints do not change the arithmetic
    assert np.max(np.abs(a @ u - u * w)) < 1e-11 * np.abs(ref).max() * n


@pytest.mark.parametrize("n,lda", [(129, 129), (300, 301), (1000, 1000), (2049, 2051),
                                   (4500, 4503), (6000, 6000), (9800, 9800)])
def test_two_stage_q2_forms_agree(n, lda):
    """Two-stage reduction: the register-resident Q2 back-transform (debug key 97 = 0, the
    default), the wavefront grouped-GEMM form (97 = 1) and the shared-memory column strips
    (97 = 2) give the same eigenvectors up to rounding, and all satisfy the eigen-equation;
    orders with a partial last sweep group and strip, odd leading dimensions (4500 / 4503:
    sy2sb's blocked symmetric product with lda != n); n = 9800 has more strips than SMs."""
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    a = b + b.T
    nat.set_two_stage_min(0)
    try:
        out = {}
        for mode in (0, 1, 2):
            nat.check(lib.em_config(ctx, 97, mode))
            out[mode] = _syev(a, lda=lda)
    finally:
        nat.check(lib.em_config(ctx, 97, 0))
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    scale = np.abs(ref).max()
    for w, u in out.values():
        assert np.max(np.abs(w - ref)) < 1e-12 * scale * n
        assert np.max(np.abs(u.T @ u - np.eye(n))) < 1e-12 * n
        assert np.max(np.abs(a @ u - u * w)) < 1e-11 * scale * n
    for mode in (1, 2):
        np.testing.assert_array_equal(out[0][0], out[mode][0])  # Q2 does not touch the spectrum
        # same eigenvectors (well separated random spectrum; sign fixed by the solver)
        d = np.abs(np.abs(np.sum(out[0][1] * out[mode][1], axis=0)) - 1.0)
        assert d.max() < 1e-9


@pytest.mark.parametrize("n", [130, 1000, 3001])
def test_panel_qr_global_memory_form(n):
    """The band reduction's panel QR (one grid barrier per column) in its global-memory
    form (debug key 92: the form panels taller than the CTAs' shared memory take, N > ~59,000)
    runs the same arithmetic in the same order as the shared-memory form: identical
    eigenvalues and eigenvectors, bit for bit, and both match LAPACK. Orders with a last
    panel shorter than 64 rows (130, 3001)."""
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    rng = np.random.default_rng(7 * n)
    b = rng.standard_normal((n, n))
    a = b + b.T
    nat.set_two_stage_min(0)
    try:
        w0, u0 = _syev(a)
        nat.check(lib.em_config(ctx, 92, 1))
        w1, u1 = _syev(a)
    finally:
        nat.check(lib.em_config(ctx, 92, 0))
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    scale = np.abs(ref).max()
    assert np.max(np.abs(w0 - ref)) < 1e-12 * scale * n
    assert np.max(np.abs(a @ u0 - u0 * w0)) < 1e-11 * scale * n
    np.testing.assert_array_equal(w0, w1)
    np.testing.assert_array_equal(u0, u1)


def test_eig_path_reported_and_pool_trim():
    """em_info(EM_INFO_EIG_PATH) says which tridiagonalisation ran; em_trim releases the
    library's cached pool memory (ADVICE: the path may depend on free memory, so it is
    observable, and the cache is releasable)."""
    from paper_2407_11993_b200 import _native as nat
    rng = np.random.default_rng(3)
    b = rng.standard_normal((300, 300))
    a = b + b.T
    _syev(a)
    assert nat.last_eig_path() == 1
    nat.set_two_stage_min(0)
    try:
        w2, _ = _syev(a)
        assert nat.last_eig_path() == 2
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    nat.trim()
    w1, _ = _syev(a)
    assert np.max(np.abs(w1 - w2)) < 1e-11 * np.abs(w1).max()
