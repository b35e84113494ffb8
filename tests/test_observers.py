"""Probe observers and crack signatures against the unmodified reference
(tests/golden/observers.npz from make_golden.py case_observers, the reference's own tube
network): field_transfer (assembly.py:350-386) incl. its ProbeTooClose message,
run_transient with probes for td2 and td1 (transient.py:266-273, 302-305), fd_solve's
probe phasors, crack_signature / normalized (ndt.py:201-240)."""
from types import SimpleNamespace

import numpy as np
import pytest

from tests.conftest import golden, rel_l2


def _net(g):
    return SimpleNamespace(branch_starts=g["starts"], branch_ends=g["ends"],
                           wire_radius=g["wire_radius"])


def _rm(g):
    from paper_2407_11993_b200 import linalg, reduction
    n_p = int(g["n_ports"])
    return reduction.ReducedModel(
        r_i=linalg.SymMatrix(g["r_i"]), l_i=linalg.SymMatrix(g["l_i"]), r_d=g["r_d"],
        l_d=g["l_d"], m0=g["m0"], lift=g["lift"], k=g["k"],
        basis=SimpleNamespace(w=g["w"]), port_names=("drive",)[:n_p])


def test_crack_signature_matches_reference():
    from paper_2407_11993_b200.errors import IndexMismatch
    from paper_2407_11993_b200.frequency import PhasorSet
    from paper_2407_11993_b200.ndt import crack_signature
    g = golden("observers")
    angles = tuple(float(a) for a in g["cs_angles"])
    freqs = [float(f) for f in g["cs_freqs"]]
    pd, pb = PhasorSet(probe_angles=angles), PhasorSet(probe_angles=angles)
    for p in range(len(angles)):
        for j, f in enumerate(freqs):
            pd[(p, f)] = g["cs_defect"][p, j]
            pb[(p, f)] = g["cs_background"][p, j]
    sig = crack_signature(pd, pb)
    keys = [tuple(k) for k in g["cs_keys"]]
    assert sorted(sig.entries) == keys
    assert np.array_equal(np.array([sig.entries[k] for k in keys]), g["cs_sig"])
    nrm = sig.normalized()
    assert np.array_equal(np.array([nrm.entries[k] for k in keys]), g["cs_norm"])
    assert np.array_equal(np.array([sig.magnitude_by_angle(f) for f in freqs]), g["cs_mag"])
    assert sig.frequencies == tuple(freqs)
    short = PhasorSet(probe_angles=angles)
    short[(0, freqs[0])] = 1.0
    with pytest.raises(IndexMismatch):
        crack_signature(pd, short)
    other = PhasorSet(entries=dict(pb.entries), probe_angles=angles[::-1])
    with pytest.raises(IndexMismatch):
        crack_signature(pd, other)


@pytest.mark.gpu
def test_field_transfer_matches_reference():
    from paper_2407_11993_b200.errors import ProbeTooClose
    from paper_2407_11993_b200.observers import biot_savart, field_transfer
    g = golden("observers")
    t = field_transfer(_net(g), g["probes"])
    assert t.shape == g["transfer"].shape
    assert np.abs(t - g["transfer"]).max() <= 1e-13 * np.abs(g["transfer"]).max()
    with pytest.raises(ProbeTooClose) as e:
        field_transfer(_net(g), g["bad_probes"])
    assert str(e.value) == str(g["bad_msg"])
    cur = np.linspace(-1, 1, g["starts"].shape[0])
    assert rel_l2(biot_savart(_net(g), cur, g["probes"]), g["transfer"] @ cur) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["td2", "td1"])
def test_run_transient_probe_fields_match_reference(method):
    from paper_2407_11993_b200 import modal, transient
    from paper_2407_11993_b200.network import DriveSignal, Tone
    g = golden("observers")
    rm = _rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i) if method == "td2" else None
    dt = float(g["dt"])
    cfg = transient.TransientConfig(theta=1.0, dt=dt, t_end=60 * dt, method=method,
                                    capture_stride=3, probes=g["probes"])
    drive = DriveSignal(tones=(Tone(1.0, 1e3, 0.0),), ports=("drive",))
    res = transient.run_transient(rm, _net(g), drive, cfg, modal=basis)
    ref = g[f"{method}_fields"]
    assert res.probe_fields.shape == ref.shape
    assert rel_l2(res.probe_fields, ref) < 1e-8


@pytest.mark.gpu
def test_fd_solve_probe_phasors():
    from paper_2407_11993_b200 import frequency
    from paper_2407_11993_b200.observers import field_transfer
    g = golden("observers")
    rm = _rm(g)
    i_d = np.array([1.0 + 0.5j])
    cur, fields = frequency.fd_solve(rm, _net(g), 2e4, i_d, probes=g["probes"])
    branch = g["w"] @ (g["k"] @ cur + g["lift"] @ i_d)
    t = field_transfer(_net(g), g["probes"])
    ref = t @ branch.real + 1j * (t @ branch.imag)
    assert fields.shape == (12, 3) and np.abs(fields - ref).max() <= 1e-12 * np.abs(ref).max()
