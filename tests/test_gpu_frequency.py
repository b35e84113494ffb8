"""Frequency-domain companions on the device against the reference's
outputs (tests/golden/fd.npz from the unmodified reference) and the oracle."""
import numpy as np
import pytest

from oracle import oracle
from tests.conftest import golden

pytestmark = pytest.mark.gpu


def _rm(name):
    from paper_2407_11993_b200 import reduction
    m = golden(name)
    n_p, n_s = m["r_d"].shape[1], m["m0"].shape[1]
    return reduction.from_blocks(m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"],
                                 port_names=tuple(f"p{i}" for i in range(n_p)),
                                 source_names=tuple(f"s{i}" for i in range(n_s))), m


@pytest.mark.parametrize("name", ["plate_small", "tube_small"])
def test_solve_tone_matches_reference(name):
    from paper_2407_11993_b200 import frequency
    g = golden("fd")
    rm, _ = _rm(name)
    for k, w in enumerate(g[f"{name}_omegas"]):
        got = frequency.solve_tone(rm, float(w), g[f"{name}_i_d"], g[f"{name}_i0"])
        ref = g[f"{name}_I_{k}"]
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), (name, k)
    cur, fields = frequency.fd_solve(rm, None, float(g[f"{name}_omegas"][2]),
                                     g[f"{name}_i_d"], g[f"{name}_i0"])
    assert fields is None and np.linalg.norm(cur - g[f"{name}_I_2"]) <= 1e-10 * np.linalg.norm(cur)


def test_solve_tone_larger_plate_vs_oracle():
    from paper_2407_11993_b200 import frequency
    rm, m = _rm("plate_200")
    i_d, i0 = np.array([0.4 - 1.0j]), np.array([2.0 + 0.1j])
    for w in (0.0, 2 * np.pi * 1e4, 2 * np.pi * 3e5):
        got = frequency.solve_tone(rm, w, i_d, i0)
        ref = oracle.solve_tone(m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"], w, i_d, i0)
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), w


def test_solve_tone_errors():
    from paper_2407_11993_b200 import frequency, reduction
    from paper_2407_11993_b200.errors import (DimensionMismatch, NotPositiveDefinite,
                                              ValidationError)
    rm, _ = _rm("plate_small")
    with pytest.raises(ValidationError):
        frequency.solve_tone(rm, -1.0, np.zeros(1), np.zeros(1))
    with pytest.raises(DimensionMismatch):
        frequency.solve_tone(rm, 1.0, np.zeros(2), np.zeros(1))
    with pytest.raises(ValidationError):
        frequency.fd_solve(rm, None, 1.0, np.zeros(1), probes=np.zeros((1, 3)))
    bad = reduction.from_blocks(np.array([[1.0, 2.0], [2.0, 1.0]]), np.eye(2), np.zeros((2, 0)),
                                np.zeros((2, 0)), np.zeros((2, 0)))
    with pytest.raises(NotPositiveDefinite) as e:
        frequency.solve_tone(bad, 1.0, np.zeros(0), np.zeros(0))
    assert e.value.pivot == 1


def test_dft_phasors_match_reference():
    from paper_2407_11993_b200 import frequency
    from paper_2407_11993_b200.errors import NonintegerPeriods, NyquistViolation, ValidationError
    g = golden("fd")
    x, dt = g["dft_x"], float(g["dft_dt"])
    for f, p in zip(g["dft_freqs"], g["dft_phasors"]):
        assert abs(frequency.dft_phasor(x, dt, float(f)) - p) < 1e-13
    assert abs(frequency.dft_phasor(x[500:1500], dt, 1e4, t0=500 * dt)
               - g["dft_phasor_t0"]) < 1e-13
    # a pure sine lands on 1 + 0j (Im convention)
    t = dt * np.arange(2000)
    assert abs(frequency.dft_phasor(np.sin(2 * np.pi * 1e4 * t), dt, 1e4) - 1.0) < 1e-13
    ps = frequency.extract_phasors(t, g["ext_rec"], [1e4, 5e4], [0.0, 1.0, 2.0],
                                   window=(2e-4, 1.2e-3))
    keys = sorted(ps.entries)
    assert np.array_equal(np.array([[p, f] for (p, f) in keys]), g["ext_keys"])
    assert np.max(np.abs(np.array([ps[k] for k in keys]) - g["ext_vals"])) < 1e-13
    assert ps.frequencies == (1e4, 5e4) and ps.probe_ids == (0, 1, 2)
    with pytest.raises(NyquistViolation):
        frequency.dft_phasor(x, dt, 6e5)
    with pytest.raises(NonintegerPeriods):
        frequency.dft_phasor(x[:1999], dt, 1e4)
    with pytest.raises(ValidationError):
        frequency.extract_phasors(t, g["ext_rec"], [1e4], [0, 1, 2], window=(1.5e-3, 2.5e-3))


def test_phasors_of_device_observables():
    """Phasors straight from the device observables of a TD2 run (no host round trip of
    the N x T record) equal the host DFT of the same record."""
    from paper_2407_11993_b200 import frequency, modal, transient
    rm, m = _rm("plate_small")
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    dt, steps = 1e-6, 1000
    t = dt * np.arange(steps + 1)
    i_d = np.sin(2 * np.pi * 1e4 * t)[:, None]
    i0 = np.zeros((steps + 1, rm.n_sources))
    st = transient.Td2Stepper(rm, basis, dt, 0.5)
    st.set_observables((m["c"], None))
    from paper_2407_11993_b200 import _native as nat
    drive = nat.device_vector(np.concatenate([i_d, i0], axis=1).reshape(-1))
    q = nat.zeros(basis.n_modes)
    y_dev, _ = st.run_device(drive, steps, q)
    n_obs = m["c"].shape[0]
    # y_dev is row-major (steps, n_obs) == column-major n_obs x steps; records are its rows,
    # i.e. column-major (steps x n_obs) = torch (n_obs, steps): transpose on the device
    rec = y_dev.t().contiguous()
    ph = frequency.phasor_matrix(rec, steps, n_obs, dt, dt, [1e4, 2e4])
    y = y_dev.cpu().numpy()
    for j in range(n_obs):
        for fi, f in enumerate((1e4, 2e4)):
            assert abs(ph[j, fi] - oracle.dft_phasor(y[:, j], dt, f, t0=dt)) < 1e-12 * (
                1 + abs(ph[j, fi]))
