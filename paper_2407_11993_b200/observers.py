"""Probe observers: the magnetic field at probe points from the
branch currents, and run_transient's probe fields built on it.

field_transfer follows the reference's assembly.field_transfer
(pkg/src/eddymodes/assembly.py:350-386): exact Biot-Savart field of every straight
branch segment at every probe, computed on the device (em_field_transfer). The network
only has to expose the segment geometry (`branch_starts`, `branch_ends`, `wire_radius`,
the reference's LoopNetwork attributes); the network generators themselves are a
geometry front end outside this path.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .errors import DimensionMismatch, ProbeTooClose


def field_transfer(net, probes: np.ndarray) -> np.ndarray:
    """(n_probes, 3, n_branches) map from branch currents to B at the probes
    (assembly.py:350-386). Raises ProbeTooClose for a probe within a branch's wire radius
    of its segment (the first such (probe, branch) pair, as the reference names it)."""
    probes = np.atleast_2d(np.asarray(probes, dtype=float))
    if probes.shape[1] != 3:
        raise DimensionMismatch("probes must be (n, 3) positions")
    a = np.ascontiguousarray(net.branch_starts, dtype=float)
    b = np.ascontiguousarray(net.branch_ends, dtype=float)
    rad = np.ascontiguousarray(net.wire_radius, dtype=float)
    nb, n_p = a.shape[0], probes.shape[0]
    if n_p == 0 or nb == 0:
        return np.zeros((n_p, 3, nb))
    t = nat.empty(n_p * 3 * nb)
    bad = ctypes.c_int64(-1)
    # the device copies must outlive the call (nat.ptr keeps no reference)
    da, db = nat.device_vector(a.reshape(-1)), nat.device_vector(b.reshape(-1))
    dr, dp = nat.device_vector(rad), nat.device_vector(probes.reshape(-1))
    rc = nat.load_library().em_field_transfer(nat.context(), nb, nat.ptr(da), nat.ptr(db),
                                              nat.ptr(dr), n_p, nat.ptr(dp), nat.ptr(t),
                                              ctypes.byref(bad))
    if bad.value >= 0:
        p, j = divmod(int(bad.value), nb)
        raise ProbeTooClose(f"probe {p} lies on branch {j} (within the wire radius)")
    nat.check(rc, "em_field_transfer")
    return t.cpu().numpy().reshape(n_p, 3, nb)


def biot_savart(net, branch_currents: np.ndarray, probes: np.ndarray) -> np.ndarray:
    """B vectors (tesla) at the probes for the given branch currents (assembly.py:389-396)."""
    currents = np.asarray(branch_currents, dtype=float)
    nb = np.asarray(net.branch_starts).shape[0]
    if currents.shape != (nb,):
        raise DimensionMismatch(f"expected {nb} branch currents, got {currents.shape}")
    return field_transfer(net, probes) @ currents


def probe_observables(net, rm, probes: np.ndarray):
    """The probe fields as observables of the internal currents (transient.py:266-273):
    C = transfer @ (W K) (3 p x N) and D = transfer @ (W lift) (3 p x n_p), rows ordered
    (probe, component); fields[cap] = (C I + D i_D(t_{k+1})).reshape(p, 3)."""
    if net is None or getattr(rm, "basis", None) is None:
        from .errors import ValidationError
        raise ValidationError("probe observers require the network geometry")
    tr = field_transfer(net, probes)                       # (p, 3, nb)
    w = np.asarray(rm.basis.w, dtype=float)
    flat = tr.reshape(-1, tr.shape[2])
    c = flat @ (w @ np.asarray(rm.k, dtype=float))
    d = flat @ (w @ np.asarray(rm.lift, dtype=float))
    return c, d
