"""CPU-only checks of the boundary and the host logic (no device compute):
the C-ABI library loads and exports every symbol include/*.h declares; the
Python mirror keeps the reference's names, validation and error behaviour; the
drive sample table matches the reference sampler; synthetic inputs are sane."""
import os
import re

import numpy as np
import pytest

from tests.conftest import REPO

HEADER = os.path.join(REPO, "include", "eddymodes_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(em_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2407_11993_b200 import _native
    lib = _native.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # and the ctypes signature table covers the header
    assert set(syms) == set(_native.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(REPO, "paper_2407_11993_b200", "libeddymodes_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core math is present


def test_errors_mirror_reference_hierarchy():
    from paper_2407_11993_b200 import errors as E
    assert issubclass(E.NotPositiveDefinite, E.NumericalError)
    assert issubclass(E.DimensionMismatch, E.InputError)
    assert issubclass(E.ValidationError, E.InputError)
    e = E.NotPositiveDefinite(3, "stepping matrix")
    assert e.pivot == 3 and str(e) == "stepping matrix is not positive definite (pivot 3 <= 0)"


def test_transient_config_validation():
    from paper_2407_11993_b200.errors import ValidationError
    from paper_2407_11993_b200.transient import TransientConfig
    with pytest.raises(ValidationError):
        TransientConfig(theta=1.5, dt=1e-6, t_end=1e-5)
    with pytest.raises(ValidationError):
        TransientConfig(theta=0.5, dt=0.0, t_end=1e-5)
    with pytest.raises(ValidationError):
        TransientConfig(theta=0.5, dt=1e-6, t_end=1e-7)
    with pytest.raises(ValidationError):
        TransientConfig(theta=0.5, dt=1e-6, t_end=1e-5, method="td3")
    with pytest.raises(ValidationError):
        TransientConfig(theta=0.5, dt=1e-6, t_end=1e-5, capture_stride=0)
    assert TransientConfig(theta=0.5, dt=1e-6, t_end=2000e-6).n_steps == 2000


def test_symmatrix_mirrors_lower():
    from paper_2407_11993_b200.errors import DimensionMismatch
    from paper_2407_11993_b200.linalg import SymMatrix
    s = SymMatrix(np.array([[1.0, 99.0], [0.3, 2.0]]))
    assert np.array_equal(s.full, s.full.T) and s.full[0, 1] == 0.3
    with pytest.raises(DimensionMismatch):
        SymMatrix.from_full(np.array([[1.0, 2.0], [3.0, 4.0]]))


def test_drive_samples_match_reference_sampler():
    """transient.drive_samples == the reference's per-step sampler (oracle restatement)."""
    from oracle import oracle as O
    from paper_2407_11993_b200 import reduction, transient
    from paper_2407_11993_b200.network import DriveSignal, Tone
    n = 4
    rm = reduction.from_blocks(np.eye(n), np.eye(n), np.ones((n, 1)), np.ones((n, 1)),
                               np.ones((n, 2)), port_names=("p",), source_names=("a", "b"))
    drives = (DriveSignal(tones=(Tone(0.7, 2e4, 0.3), Tone(0.2, 5e4, 1.1)), ports=("p",)),
              DriveSignal(tones=(Tone(1.0, 1e4),), sources=("b",)))
    i_d, i0 = transient.drive_samples(None, rm, drives, 1e-6, 300)
    sd = O.tone_sampler([[(0.7, 2e4, 0.3), (0.2, 5e4, 1.1)]])
    s0 = O.tone_sampler([[], [(1.0, 1e4, 0.0)]])
    np.testing.assert_allclose(i_d, O.sample_table(sd, 300, 1e-6), rtol=0, atol=1e-15)
    np.testing.assert_allclose(i0, O.sample_table(s0, 300, 1e-6), rtol=0, atol=1e-15)


def test_drive_validation_errors():
    from paper_2407_11993_b200 import reduction, transient
    from paper_2407_11993_b200.errors import ValidationError
    from paper_2407_11993_b200.network import DriveSignal, Tone
    with pytest.raises(ValidationError):
        DriveSignal(tones=(Tone(1.0, 0.0),))
    with pytest.raises(ValidationError):
        DriveSignal(tones=(Tone(1.0, 5.0), Tone(2.0, 5.0)))
    rm = reduction.from_blocks(np.eye(2), np.eye(2), None, None, np.ones((2, 1)),
                               source_names=("s",))
    with pytest.raises(ValidationError):
        transient.drive_samples(None, rm, DriveSignal(tones=(Tone(1, 1e3),), sources=("zz",)),
                                1e-6, 5)


def test_synthetic_plate_is_spd_and_matches_survey_conventions():
    from paper_2407_11993_b200.synth import Plate, plate_model
    m = plate_model(6, 5, 2, n_ports=1, n_sources=1, n_obs=4)
    r, l = m["r_i"], m["l_i"]
    assert np.allclose(r, r.T) and np.allclose(l, l.T, rtol=0, atol=1e-22)
    assert np.linalg.eigvalsh(r).min() > 0 and np.linalg.eigvalsh(l).min() > 0
    assert np.allclose(np.diag(r), 6 * 1.7e-8 + 1e-3)
    p = Plate(6, 5, 2)
    assert np.isclose(l[0, 0], 1e-7 * 2 / p.h)
    assert m["c"].shape == (4, 60) and m["r_d"].shape == (60, 1)
    # notch removes voxels
    assert Plate(40, 30, 2, notch=True).n < 40 * 30 * 2


def test_oracle_is_not_imported_by_product():
    import ast
    pkg = os.path.join(REPO, "paper_2407_11993_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, (ast.Import, ast.ImportFrom)):
                    names = [a.name for a in node.names] + [getattr(node, "module", "") or ""]
                    assert not any(n.startswith("oracle") for n in names), fn


def test_no_device_means_loud_failure(monkeypatch):
    import torch
    from paper_2407_11993_b200 import _native, linalg
    from paper_2407_11993_b200.errors import DeviceError
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(DeviceError):
        linalg.cholesky(np.eye(3))
