"""Frequency-domain companions of the modal path, mirroring
`eddymodes.frequency` (E/frequency.py): the per-tone solve and DFT phasor extraction.

Phasor convention throughout: x(t) = Im{X e^(j w t)}, so a pure sin(w t) maps to
X = 1 at angle 0 (E/frequency.py:1-7).

* `solve_tone` (E/frequency.py:56-94): the reference LU-factors the real 2n embedding
  [[R, wL], [wL, -R]] per tone. Here `FdPlan` factors R and forms K = L R^-1 L once on
  the device; each tone is one Cholesky of the SPD Schur complement R + w^2 K
  (em_fd_plan_create / em_fd_solve), the same solution to round-off.
* `dft_phasor` / `extract_phasors` (E/frequency.py:114-166): the tone table
  [sin(w t), cos(w t)] is built on the device (em_tone_table) and the phasors of every
  record are one DMMA GEMM (em_dgemm).
* `azimuthal_component` (E/frequency.py:169-174) is a per-probe 3-vector projection,
  kept on the host as in the reference (O(n_t n_probes)).

Probe fields (`fd_solve(..., probes=...)`) need the filament geometry
(`assembly.field_transfer`), a front end outside this path: ValidationError.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import (DimensionMismatch, NonintegerPeriods, NotPositiveDefinite,
                     NyquistViolation, SingularSystem, ValidationError)
from .reduction import ReducedModel

#: Marker string recorded with every phasor set (E/frequency.py:29).
IM_CONVENTION = "x(t) = Im{X exp(jwt)}"


@dataclass
class PhasorSet:
    """Complex value per (probe_id, tone frequency) (E/frequency.py:32-53)."""

    entries: dict[tuple[int, float], complex] = field(default_factory=dict)
    probe_angles: tuple[float, ...] = ()
    convention: str = IM_CONVENTION

    def __setitem__(self, key, value):
        self.entries[key] = complex(value)

    def __getitem__(self, key):
        return self.entries[key]

    @property
    def frequencies(self) -> tuple[float, ...]:
        return tuple(sorted({f for (_, f) in self.entries}))

    @property
    def probe_ids(self) -> tuple[int, ...]:
        return tuple(sorted({p for (p, _) in self.entries}))


def _sym_full(m) -> np.ndarray:
    return m.full if hasattr(m, "full") else np.asarray(m, dtype=float)


class FdPlan:
    """Device factorisation shared by every tone of one reduced model:
    R = G G^T and K = L R^-1 L (potrf, trsm and a lower DMMA GEMM)."""

    def __init__(self, rm: ReducedModel):
        self.rm = rm
        self.n = n = rm.n_internal
        self._plan = None
        if n == 0:
            return
        ld = nat.device_symmetric(_sym_full(rm.l_i))
        rd = nat.device_symmetric(_sym_full(rm.r_i))
        plan = ctypes.c_void_p()
        piv = ctypes.c_int64(-1)
        rc = nat.load_library().em_fd_plan_create(nat.context(), n, nat.ptr(ld), n, nat.ptr(rd),
                                                  n, ctypes.byref(plan), ctypes.byref(piv))
        if rc == nat.EM_ERR_NOT_PD:
            raise NotPositiveDefinite(int(piv.value), "modal resistance matrix")
        nat.check(rc, "em_fd_plan_create")
        self._plan = plan

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            nat.load_library().em_fd_plan_destroy(plan)
            self._plan = None

    def solve(self, omega: float, e: np.ndarray) -> np.ndarray:
        """I with (R + j w L) I = e (complex n-vector)."""
        n = self.n
        if n == 0:
            return np.zeros(0, dtype=complex)
        c = np.ascontiguousarray(e.real, dtype=float)
        d = np.ascontiguousarray(e.imag, dtype=float)
        a, b = np.empty(n), np.empty(n)
        piv = ctypes.c_int64(-1)
        f = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        rc = nat.load_library().em_fd_solve(self._plan, float(omega), f(c), f(d), f(a), f(b),
                                            ctypes.byref(piv))
        if rc == nat.EM_ERR_NOT_PD:
            raise SingularSystem(f"tone system numerically singular at column {int(piv.value)}")
        nat.check(rc, "em_fd_solve")
        return a - 1j * b


_PLAN_CACHE: list = []  # [(rm, FdPlan)]: the last model's factorisation


def _plan_for(rm: ReducedModel) -> FdPlan:
    if _PLAN_CACHE and _PLAN_CACHE[0][0] is rm:
        return _PLAN_CACHE[0][1]
    plan = FdPlan(rm)
    _PLAN_CACHE[:] = [(rm, plan)]
    return plan


def solve_tone(rm: ReducedModel, omega: float, i_d_phasor: np.ndarray,
               i0_phasor: np.ndarray) -> np.ndarray:
    """Internal current phasors for one tone (E/frequency.py:56-94):
    (R_i + j w L_i) I = -(R_D + j w L_D) i_D - j w M0 i0."""
    if omega < 0:
        raise ValidationError("omega must be >= 0")
    n = rm.n_internal
    i_d_phasor = np.asarray(i_d_phasor, dtype=complex)
    i0_phasor = np.asarray(i0_phasor, dtype=complex)
    if i_d_phasor.shape != (rm.n_ports,):
        raise DimensionMismatch(f"expected {rm.n_ports} port phasors")
    if i0_phasor.shape != (rm.n_sources,):
        raise DimensionMismatch(f"expected {rm.n_sources} source phasors")
    if n == 0:
        return np.zeros(0, dtype=complex)
    e = np.zeros(n, dtype=complex)
    if rm.n_ports:
        e -= (rm.r_d + 1j * omega * rm.l_d) @ i_d_phasor
    if rm.n_sources:
        e -= 1j * omega * (rm.m0 @ i0_phasor)
    return _plan_for(rm).solve(omega, e)


def fd_solve(rm: ReducedModel, net, omega: float, i_d_phasor: np.ndarray,
             i0_phasor: np.ndarray | None = None, probes: np.ndarray | None = None):
    """One-tone solve returning (internal current phasors, probe field phasors or None)
    (E/frequency.py:93-111): probe fields superpose the Biot-Savart transfers
    (observers.field_transfer) of the lifted total phasor currents."""
    if probes is not None and (net is None or getattr(rm, "basis", None) is None):
        raise ValidationError("probe fields require the network geometry")
    if i0_phasor is None:
        i0_phasor = np.zeros(rm.n_sources, dtype=complex)
    currents = solve_tone(rm, omega, i_d_phasor, i0_phasor)
    fields = None
    if probes is not None:
        from .observers import field_transfer
        transfer = field_transfer(net, probes)
        coords = np.asarray(rm.k) @ currents + np.asarray(rm.lift) @ np.asarray(i_d_phasor,
                                                                               dtype=complex)
        branch = np.asarray(rm.basis.w, dtype=float) @ coords
        fields = transfer @ branch.real + 1j * (transfer @ branch.imag)
    return currents, fields


def _check_record(n: int, dt: float, f: float):
    if n < 2:
        raise ValidationError("need at least 2 samples")
    if f >= 0.5 / dt:
        raise NyquistViolation(f"{f} Hz is not below Nyquist {0.5 / dt} Hz")
    periods = n * dt * f
    if abs(periods - round(periods)) > 1e-9:
        raise NonintegerPeriods(f"window of {n} samples spans {periods} periods of {f} Hz")


def phasor_matrix(records_dev, n_t: int, n_rec: int, dt: float, t0: float, freqs) -> np.ndarray:
    """Phasors of n_rec uniformly sampled records held on the device (column-major
    n_t x n_rec, i.e. a torch (n_rec, n_t) tensor) at every tone: (n_rec, n_f) complex.
    One tone table (em_tone_table) and one DMMA GEMM."""
    freqs = np.ascontiguousarray(np.asarray(freqs, dtype=float))
    n_f = freqs.shape[0]
    for f in freqs:
        _check_record(n_t, dt, float(f))
    ctx, lib = nat.context(), nat.load_library()
    table = nat.empty(2 * n_f, n_t)  # column-major n_t x 2 n_f
    nat.check(lib.em_tone_table(ctx, n_t, float(dt), float(t0), n_f,
                                freqs.ctypes.data_as(ctypes.c_void_p), nat.ptr(table), n_t),
              "em_tone_table")
    proj = nat.empty(2 * n_f, n_rec)  # column-major n_rec x 2 n_f
    nat.check(lib.em_dgemm(ctx, 1, 0, n_rec, 2 * n_f, n_t, 2.0 / n_t, nat.ptr(records_dev), n_t,
                           nat.ptr(table), n_t, 0.0, nat.ptr(proj), n_rec), "em_dgemm")
    p = nat.host_colmajor(proj, n_rec, 2 * n_f)
    # j * (2/N) sum x e^{-jwt} = (2/N) sum x sin + j (2/N) sum x cos
    return p[:, 0::2] + 1j * p[:, 1::2]


def dft_phasor(samples: np.ndarray, dt: float, f: float, t0: float = 0.0) -> complex:
    """Single-tone phasor of a uniformly sampled record (E/frequency.py:114-138)."""
    samples = np.asarray(samples, dtype=float)
    n = samples.shape[0]
    _check_record(n, dt, f)
    rec = nat.device_vector(np.ascontiguousarray(samples))
    return complex(phasor_matrix(rec, n, 1, dt, t0, [f])[0, 0])


def extract_phasors(times: np.ndarray, fields_phi: np.ndarray, frequencies, probe_angles,
                    window: tuple[float, float] | None = None) -> PhasorSet:
    """Tone phasors of per-probe records (E/frequency.py:141-166); all probes and tones
    in one device GEMM."""
    times = np.asarray(times, dtype=float)
    fields_phi = np.asarray(fields_phi, dtype=float)
    dt = times[1] - times[0]
    if window is None:
        sel = slice(None)
    else:
        start, end = window
        first = int(np.searchsorted(times, start - 0.5 * dt))
        count = int(round((end - start) / dt))
        if first + count > times.shape[0]:
            raise ValidationError("analysis window extends past the record")
        sel = slice(first, first + count)
    tsel = times[sel]
    fsel = fields_phi[sel]
    ps = PhasorSet(probe_angles=tuple(float(a) for a in probe_angles))
    freqs = [float(f) for f in frequencies]
    if not freqs or fsel.shape[1] == 0:
        return ps
    n_t, n_rec = fsel.shape
    rec = nat.device_colmajor(fsel)  # column-major n_t x n_rec
    ph = phasor_matrix(rec, n_t, n_rec, dt, float(tsel[0]), freqs)
    for f_i, f in enumerate(freqs):
        for p in range(n_rec):
            ps[(p, f)] = ph[p, f_i]
    return ps


def azimuthal_component(fields: np.ndarray, probe_angles: np.ndarray) -> np.ndarray:
    """Project (n_times, n_probes, 3) field vectors on each probe's azimuthal unit
    vector (E/frequency.py:169-174)."""
    a = np.asarray(probe_angles, dtype=float)
    phi_hat = np.stack([-np.sin(a), np.cos(a), np.zeros_like(a)], axis=1)
    return np.einsum("tpc,pc->tp", fields, phi_hat)
