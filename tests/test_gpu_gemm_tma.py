"""The TMA-fed persistent DGEMM (csrc/gemm_tma.cu) against numpy on every operand layout,
ragged edges, beta, split-k and the lower-triangle output mode. The reference does these
products with numpy (E/modal.py:64-81, E/transient.py:140-154); FP64 tolerance 1e-12
relative to the largest entry (summation order differs from BLAS)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = ((256, 192, 64), (300, 333, 146), (130, 64, 1100), (517, 260, 33), (128, 128, 16),
          (1, 1, 1), (37, 129, 300), (96, 2000, 2100))


def _off8(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr() + 8)


def _lib():
    from paper_2407_11993_b200 import _native as nat
    return nat, nat.context(), nat.load_library()


@pytest.mark.parametrize("cfg", [2, 4, 5])
def test_dgemm_tma_all_layouts(cfg):
    nat, ctx, lib = _lib()
    rng = np.random.default_rng(11 + cfg)
    nat.check(lib.em_config(ctx, 95, cfg))
    try:
        for (m, n, k) in SHAPES:
            for ta in (0, 1):
                for tb in (0, 1):
                    a = rng.standard_normal((k, m) if ta else (m, k))
                    b = rng.standard_normal((n, k) if tb else (k, n))
                    c0 = rng.standard_normal((m, n))
                    # even leading dimensions (TMA strides are multiples of 16 bytes)
                    lda, ldb = a.shape[0] + (a.shape[0] & 1), b.shape[0] + (b.shape[0] & 1)
                    ap = np.zeros((lda, a.shape[1]))
                    ap[:a.shape[0]] = a
                    bp = np.zeros((ldb, b.shape[1]))
                    bp[:b.shape[0]] = b
                    da, db, dc = (nat.device_colmajor(ap), nat.device_colmajor(bp),
                                  nat.device_colmajor(c0))
                    for beta in (0.0, -2.0):
                        dc = nat.device_colmajor(c0)
                        nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 0.5, nat.ptr(da), lda,
                                               nat.ptr(db), ldb, beta, nat.ptr(dc), m))
                        ref = 0.5 * (a.T if ta else a) @ (b.T if tb else b) + beta * c0
                        got = nat.host_colmajor(dc, m, n)
                        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), \
                            (cfg, m, n, k, ta, tb, beta)
    finally:
        nat.check(lib.em_config(ctx, 95, 1))


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_dgemm_lower_output(cfg):
    """Only entries with r + diag_off >= c are written; the rest of C is untouched."""
    nat, ctx, lib = _lib()
    rng = np.random.default_rng(5)
    nat.check(lib.em_config(ctx, 95, cfg))
    try:
        for (m, n, k, off) in ((400, 400, 96, 0), (333, 290, 64, 17), (512, 640, 130, -64),
                               (2304, 2304, 128, 0)):
            for ta, tb in ((0, 1), (1, 0), (0, 0)):
                a = rng.standard_normal((k, m) if ta else (m, k))
                b = rng.standard_normal((n, k) if tb else (k, n))
                c0 = rng.standard_normal((m, n))
                da, db, dc = nat.device_colmajor(a), nat.device_colmajor(b), nat.device_colmajor(c0)
                nat.check(lib.em_dgemm_lower(ctx, ta, tb, m, n, k, -1.0, nat.ptr(da), a.shape[0],
                                             nat.ptr(db), b.shape[0], 1.0, nat.ptr(dc), m, off))
                full = c0 - (a.T if ta else a) @ (b.T if tb else b)
                r, c = np.indices((m, n))
                ref = np.where(r + off >= c, full, c0)
                got = nat.host_colmajor(dc, m, n)
                assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), \
                    (cfg, m, n, k, off, ta, tb)
                assert np.array_equal(got[r + off < c], c0[r + off < c])
    finally:
        nat.check(lib.em_config(ctx, 95, 1))


def test_dgemm_tma_auto_large_and_repeatable():
    """The automatic selection (large aligned products) gives bitwise-repeatable results
    (every tile is one CTA's fixed-order sum, whichever CTA claims it) and matches the
    cp.async path to rounding."""
    import torch
    nat, ctx, lib = _lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    for (m, n, k, ta, tb) in ((4096, 2048, 512, 0, 0), (256, 8192, 4096, 1, 0),
                              (3072, 3072, 128, 0, 1)):
        a = torch.randn((m, k) if ta else (k, m), device="cuda", dtype=torch.float64, generator=g)
        b = torch.randn((k, n) if tb else (n, k), device="cuda", dtype=torch.float64, generator=g)
        outs = []
        for mode in (1, 1, 0):
            nat.check(lib.em_config(ctx, 95, mode))
            c = torch.zeros(n, m, device="cuda", dtype=torch.float64)
            nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 1.0, nat.ptr(a), a.shape[1], nat.ptr(b),
                                   b.shape[1], 0.0, nat.ptr(c), m))
            outs.append(c)
        nat.check(lib.em_config(ctx, 95, 1))
        assert torch.equal(outs[0], outs[1])
        scale = float(outs[2].abs().max())
        assert float((outs[0] - outs[2]).abs().max()) <= 1e-12 * scale


@pytest.mark.parametrize("cfg", [2, 4])
def test_dgemm_tma_operands_on_odd_elements(cfg):
    """Operands starting 8 bytes past a 16-byte boundary (sub-blocks at odd row offsets, as
    the divide-and-conquer merges pass them): the tensor map starts one element lower and
    the contiguous coordinate moves up by one."""
    nat, ctx, lib = _lib()
    rng = np.random.default_rng(3)
    nat.check(lib.em_config(ctx, 95, cfg))
    try:
        for (m, n, k) in ((300, 333, 146), (256, 192, 64), (129, 70, 2100)):
            for ta in (0, 1):
                for tb in (0, 1):
                    a = rng.standard_normal((k, m) if ta else (m, k))
                    b = rng.standard_normal((n, k) if tb else (k, n))
                    c0 = rng.standard_normal((m, n))
                    # one garbage row above each operand; even leading dimensions
                    lda = a.shape[0] + 1 + ((a.shape[0] + 1) & 1)
                    ldb = b.shape[0] + 1 + ((b.shape[0] + 1) & 1)
                    ap = np.full((lda, a.shape[1]), np.nan)
                    ap[1:1 + a.shape[0]] = a
                    ap[1 + a.shape[0]:] = 7.0
                    bp = np.full((ldb, b.shape[1]), np.nan)
                    bp[1:1 + b.shape[0]] = b
                    bp[1 + b.shape[0]:] = -3.0
                    da, db, dc = (nat.device_colmajor(ap), nat.device_colmajor(bp),
                                  nat.device_colmajor(c0))
                    nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 1.0, _off8(da), lda,
                                           _off8(db), ldb, 1.0, nat.ptr(dc), m))
                    ref = (a.T if ta else a) @ (b.T if tb else b) + c0
                    got = nat.host_colmajor(dc, m, n)
                    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), \
                        (cfg, m, n, k, ta, tb)
    finally:
        nat.check(lib.em_config(ctx, 95, 1))


def test_dsymm_band_lower_reads_only_lower_and_band():
    """C = A B for symmetric A from its lower triangle plus 127 diagonals above it: entries
    further above the diagonal are poisoned with NaN and must not be read; ragged sizes,
    the 64- and 128-column tile configurations, split-k."""
    nat, ctx, lib = _lib()
    rng = np.random.default_rng(9)
    for (m, n) in ((1000, 64), (4436, 64), (2050, 33), (3000, 192), (130, 64), (6000, 64)):
        s = rng.standard_normal((m, m))
        a = s + s.T
        b = rng.standard_normal((m, n))
        r, c = np.indices((m, m))
        ap = np.where(c - r > 127, np.nan, a)
        lda = m + (m & 1)
        app = np.zeros((lda, m))
        app[:m] = ap
        bp = np.zeros((lda, n))
        bp[:m] = b
        da, db = nat.device_colmajor(app), nat.device_colmajor(bp)
        dc = nat.device_colmajor(np.full((m, n), np.nan))
        nat.check(lib.em_dsymm_band_lower(ctx, m, n, nat.ptr(da), lda, nat.ptr(db), lda,
                                          nat.ptr(dc), m))
        got = nat.host_colmajor(dc, m, n)
        ref = a @ b
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max() * np.sqrt(m), (m, n)


@pytest.mark.parametrize("cfg", [2, 4])
def test_dgemm_tma_accumulate_many_tiles_per_cta_repeated(cfg):
    """beta != 0 with several tiles per CTA, repeated: the configuration in which a ring
    stage released right behind its last fragment load was overwritten by the next TMA box
    while other warps' epilogue traffic delayed the load (wrong 16 x 64 blocks in ~40% of
    the runs before the stage release moved behind the consuming DMMAs)."""
    import torch
    nat, ctx, lib = _lib()
    rng = np.random.default_rng(0)
    m = n = 4436
    k = 128
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((n, k))
    c0 = rng.standard_normal((m, n))
    ref = c0 - a @ b.T
    A = torch.from_numpy(a.T.copy()).cuda()
    B = torch.from_numpy(b.T.copy()).cuda()
    nat.check(lib.em_config(ctx, 95, cfg))
    try:
        for _ in range(8):
            C = torch.from_numpy(c0.T.copy()).cuda()
            nat.check(lib.em_dgemm(ctx, 0, 1, m, n, k, -1.0, nat.ptr(A), m, nat.ptr(B), n, 1.0,
                                   nat.ptr(C), m))
            got = C.t().cpu().numpy()
            assert np.abs(got - ref).max() <= 1e-11
    finally:
        nat.check(lib.em_config(ctx, 95, 1))
