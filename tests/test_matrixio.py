"""Model / eigenbasis storage: the reference's text cache read and
written byte for byte (tests/golden/cache_tube.txt from the unmodified reference's
write_cache), the binary model cache, and the device eigenbasis file."""
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

CACHE = os.path.join(GOLDEN, "cache_tube.txt")


def _read_e(path):
    lines = open(path).read().splitlines()
    for i, line in enumerate(lines):
        if line.startswith("matrix E "):
            rows, cols = int(line.split()[2]), int(line.split()[3])
            return np.array([[int(v) for v in lines[i + 1 + r].split()] for r in range(rows)])
    return None


def test_text_cache_roundtrip_is_byte_identical(tmp_path):
    from paper_2407_11993_b200 import matrixio
    rm, net = matrixio.read_cache(CACHE)
    assert net is None
    assert rm.n_internal == 11 and rm.port_names == ("drive",) and rm.source_names == ()
    assert rm.basis.n_cycles == 11 and rm.basis.n_paths == 1 and rm.basis.w.dtype == np.int64
    out = tmp_path / "cache.txt"
    matrixio.write_cache(out, rm, None, e=_read_e(CACHE),
                         header_lines=("golden: reference write_cache",))
    assert out.read_bytes() == open(CACHE, "rb").read()


def test_binary_cache_roundtrip(tmp_path):
    from paper_2407_11993_b200 import matrixio
    rm, _ = matrixio.read_cache(CACHE)
    e = _read_e(CACHE)
    p = tmp_path / "cache.emb"
    matrixio.write_cache_binary(p, rm, e=e)
    rm2, _ = matrixio.read_cache_binary(p)
    for f in ("r_d", "l_d", "m0", "lift", "k"):
        assert np.array_equal(getattr(rm, f), getattr(rm2, f)), f
    assert np.array_equal(rm.r_i.full, rm2.r_i.full) and np.array_equal(rm.l_i.full, rm2.l_i.full)
    assert rm2.port_names == rm.port_names and rm2.source_names == rm.source_names
    assert np.array_equal(rm2.basis.w, rm.basis.w) and rm2.basis.n_paths == rm.basis.n_paths
    # symmetric blocks are stored as packed lower triangles: n(n+1)/2 values each
    dense = 8 * sum(a.size for a in (rm.r_i.full, rm.l_i.full, rm.r_d, rm.l_d, rm.m0, rm.lift,
                                      rm.k, e, rm.basis.w))
    assert os.path.getsize(p) < dense - 8 * 2 * (11 * 11 - 66) + 4096


def test_cache_errors(tmp_path):
    from paper_2407_11993_b200 import matrixio
    from paper_2407_11993_b200.errors import ParseError, ValidationError
    bad = tmp_path / "bad.txt"
    bad.write_text("matrix R_I 2 2 f\n1.0 0.0\n0.0\n")
    with pytest.raises(ParseError):
        matrixio.read_cache(bad)
    bad.write_text("bogus line\n")
    with pytest.raises(ParseError):
        matrixio.read_cache(bad)
    bad.write_text("matrix R_I 1 1 f\n1.0\n")
    with pytest.raises(ParseError):
        matrixio.read_cache(bad)
    rm, _ = matrixio.read_cache(CACHE)
    with pytest.raises(ValidationError):
        matrixio.write_cache(tmp_path / "x.txt", rm, net=object())
    with pytest.raises(ParseError):
        matrixio.read_cache_binary(bad)


@pytest.mark.gpu
def test_basis_file_roundtrip_on_device(tmp_path):
    from paper_2407_11993_b200 import matrixio, modal
    from tests.conftest import golden
    g = golden("plate_small")
    basis = modal.generalized_eig(g["l_i"], g["r_i"])
    p = tmp_path / "basis.emb"
    matrixio._CHUNK = 1 << 14  # many chunks: exercise the double buffering
    matrixio.save_basis(p, basis)
    b2 = matrixio.load_basis(p)
    assert np.array_equal(b2.tau, basis.tau) and np.array_equal(b2.l_n, basis.l_n)
    assert np.array_equal(b2.r_n, basis.r_n)
    assert np.array_equal(b2.v, basis.v) and np.array_equal(b2.vt_r, basis.vt_r)
    assert b2.v_dev.is_cuda
