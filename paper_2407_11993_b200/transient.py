"""Theta-method time integration two ways — the reference's transient module
(pkg/src/eddymodes/transient.py:1-404) on the B200 library.

td1 (Td1Stepper): Z = L_i + dt*theta*R_i factored once on the device; every step
is a lower-triangle symv with R plus two persistent triangular-solve kernels.
td2 (Td2Stepper): the drive is projected onto the modes once (DMMA GEMM), and a
whole run is ONE blocked linear-recurrence scan over time fused with the
forcing and the observable reconstruction (em_td2_run).

The per-step `step()` methods keep the reference's host in-place semantics
(one device round trip per call); `run()` and run_transient are the batched
fast path. Observables y = C I + D i_D(t_{k+1}) (the reference's
`t_internal @ internal + t_ports @ i_d_next`, transient.py:304-305) are given
directly as matrices; the probe geometry (assembly.field_transfer) is a front
end outside this path.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import linalg
from .errors import DimensionMismatch, NotPositiveDefinite, ValidationError
from .modal import ModalBasis, drive_rhs
from .network import DriveSignal
from .reduction import ReducedModel


@dataclass(frozen=True)
class TransientConfig:
    """theta in [0, 1], step dt, final time t_end, method td1/td2 (transient.py:27-57)."""

    theta: float
    dt: float
    t_end: float
    method: str = "td1"
    probes: np.ndarray | None = None
    capture_stride: int = 1
    capture_state: bool = True

    def __post_init__(self):
        if not (0.0 <= self.theta <= 1.0):
            raise ValidationError("theta must lie in [0, 1]")
        if self.dt <= 0:
            raise ValidationError("dt must be positive")
        if self.t_end < self.dt:
            raise ValidationError("t_end must be at least one step")
        if self.method not in ("td1", "td2"):
            raise ValidationError(f"unknown method {self.method!r}")
        if self.capture_stride < 1:
            raise ValidationError("capture_stride must be >= 1")
        if self.probes is not None:
            object.__setattr__(self, "probes",
                               np.atleast_2d(np.asarray(self.probes, dtype=float)))

    @property
    def n_steps(self) -> int:
        return max(int(round(self.t_end / self.dt)), 1)


@dataclass
class SimulationResult:
    """Captured trajectory plus the setup/stepping wall-time split (transient.py:60-74).
    `observables` (n_captures, n_obs) is filled when run_transient gets observables=(C, D)."""

    times: np.ndarray
    internal_states: np.ndarray | None
    probe_fields: np.ndarray | None
    wall_time_setup: float
    wall_time_stepping: float
    n_steps: int
    method: str
    observables: np.ndarray | None = None

    @property
    def per_step_cost(self) -> float:
        return self.wall_time_stepping / self.n_steps


def _check_theta_dt(dt, theta):
    if dt <= 0:
        raise ValidationError("dt must be positive")
    if not (0.0 <= theta <= 1.0):
        raise ValidationError("theta must lie in [0, 1]")


def _drive_table(i_d_samples, i0_samples, n_p, n_s) -> np.ndarray:
    """(T+1) x (n_p + n_s) row-major sample table [i_d(t_k) | i0(t_k)]."""
    i_d = np.asarray(i_d_samples, dtype=float).reshape(-1, n_p) if n_p else None
    i0 = np.asarray(i0_samples, dtype=float).reshape(-1, n_s) if n_s else None
    rows = (i_d if i_d is not None else i0).shape[0] if (n_p or n_s) else None
    if rows is None:
        raise ValidationError("drive table needs the number of samples")
    parts = [p for p in (i_d, i0) if p is not None]
    for p in parts:
        if p.shape[0] != rows:
            raise DimensionMismatch("port and source sample tables differ in length")
    return np.ascontiguousarray(np.concatenate(parts, axis=1))


def _obs_device(observables, n: int, n_p: int):
    """(C (n_obs x n), D (n_obs x n_p) or None) -> device column-major buffers."""
    c, d = observables if isinstance(observables, tuple) else (observables, None)
    c = np.atleast_2d(np.asarray(c, dtype=float))
    if c.shape[1] != n:
        raise DimensionMismatch(f"observables need {n} columns, got {c.shape}")
    if c.shape[0] > 128:
        raise ValidationError("at most 128 observables per run")
    dd = None
    if d is not None and n_p:
        d = np.asarray(d, dtype=float).reshape(c.shape[0], n_p)
        dd = nat.device_colmajor(d)
    return c.shape[0], nat.device_colmajor(c), dd


def _drive_projection(rm: ReducedModel, basis: ModalBasis):
    """V^T [R_D | L_D | M0] on the device (transient.py:134-144), column-major n x n_d
    (torch (n_d, n)); a (1, n) zero block when there are no drive channels."""
    n, n_p, n_s = basis.n_modes, rm.n_ports, rm.n_sources
    nd = 2 * n_p + n_s
    if not nd:
        return nat.zeros(1, n)
    ctx, lib = nat.context(), nat.load_library()
    drv = np.concatenate([rm.r_d.reshape(n, n_p), rm.l_d.reshape(n, n_p),
                          rm.m0.reshape(n, n_s)], axis=1)
    ddrv = nat.device_colmajor(drv)
    proj = nat.empty(nd, n)
    nat.check(lib.em_dgemm(ctx, 1, 0, n, nd, n, 1.0, nat.ptr(basis.v_dev), n,
                           nat.ptr(ddrv), n, 0.0, nat.ptr(proj), n), "em_dgemm")
    return proj


def select_modes(basis: ModalBasis, tau_min: float | None = None, count: int | None = None
                 ) -> np.ndarray:
    """Mode indices for selective integration ("(iv) in a selective
    manner"): the modes with tau >= tau_min and/or the `count` slowest
    (tau is descending, so these are leading indices). Pass to Td2Stepper(modes=...)."""
    idx = np.arange(basis.n_modes)
    if tau_min is not None:
        idx = idx[basis.tau[idx] >= tau_min]
    if count is not None:
        idx = idx[:max(int(count), 0)]
    return idx


def _mode_selection(n: int, modes) -> np.ndarray | None:
    """None (all modes) or sorted unique int64 indices from indices / a boolean mask."""
    if modes is None:
        return None
    sel = np.asarray(modes)
    if sel.dtype == bool:
        if sel.shape != (n,):
            raise DimensionMismatch(f"mode mask needs {n} entries, got {sel.shape}")
        sel = np.flatnonzero(sel)
    sel = np.unique(sel.astype(np.int64))
    if sel.size and (sel[0] < 0 or sel[-1] >= n):
        raise ValidationError("mode index out of range")
    return None if sel.size == n else sel


class Td2Stepper:
    """Decoupled stepper (transient.py:116-166): per-mode scalar updates after
    projecting the drive onto the modes.

    modes (optional): integrate only these modes (indices or a boolean mask; see
    select_modes) — the selective integration of PAPER.md:299. The others stay at their
    state (rest for run()); observables and reconstructed currents are the truncated
    modal sums."""

    def __init__(self, rm: ReducedModel, basis: ModalBasis, dt: float, theta: float,
                 modes=None):
        _check_theta_dt(dt, theta)
        if basis.n_modes != rm.n_internal:
            raise DimensionMismatch("modal basis does not match the reduced model")
        t0 = time.perf_counter()
        self.rm = rm
        self.basis = basis
        self.dt = float(dt)
        self.theta = float(theta)
        n_full, n_p, n_s = basis.n_modes, rm.n_ports, rm.n_sources
        sel = _mode_selection(n_full, modes)
        self._sel = sel
        self._sel_dev = None if sel is None else nat.torch().from_numpy(sel).to("cuda")
        n = n_full if sel is None else int(sel.size)
        self._n_full = n_full
        self._n, self._n_p, self._n_s = n, n_p, n_s
        l_n = basis.l_n if sel is None else basis.l_n[sel]
        r_n = basis.r_n if sel is None else basis.r_n[sel]
        # host copies kept for API compatibility (transient.py:134-144)
        den = l_n + self.dt * self.theta * r_n
        self._c = np.sqrt(den)
        self._rn = r_n.copy()
        ctx = nat.context()
        lib = nat.load_library()
        proj = _drive_projection(rm, basis)
        if sel is not None:
            proj = proj.index_select(1, self._sel_dev).contiguous()
        self._proj = proj
        p_r = proj[0:n_p] if n_p else proj[0:1]
        p_l = proj[n_p:2 * n_p] if n_p else proj[0:1]
        p_m = proj[2 * n_p:] if n_s else proj[0:1]
        self._ln_dev = nat.device_vector(l_n)
        self._rn_dev = nat.device_vector(r_n)
        plan = ctypes.c_void_p()
        nat.check(lib.em_td2_plan_create(ctx, n, n_p, n_s, nat.ptr(self._ln_dev),
                                         nat.ptr(self._rn_dev), nat.ptr(p_r), nat.ptr(p_l),
                                         nat.ptr(p_m), self.dt, self.theta, ctypes.byref(plan)),
                  "em_td2_plan_create")
        self._plan = plan
        self.setup_time = time.perf_counter() - t0

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            nat.load_library().em_td2_plan_destroy(plan)
            self._plan = None

    @property
    def _p_r(self):
        return nat.host_colmajor(self._proj[0:self._n_p], self._n, self._n_p)

    @property
    def _p_m(self):
        return nat.host_colmajor(self._proj[2 * self._n_p:], self._n, self._n_s)

    def forcing(self, i_d, delta_i_d, delta_i0) -> np.ndarray:
        """-dt P_r i_D - P_ltr dI_D - P_m dI_0 (transient.py:147-155), on the device
        (zero for modes outside a selection)."""
        f = nat.empty(self._n)
        u = [np.ascontiguousarray(np.asarray(x, dtype=float)) for x in (i_d, delta_i_d, delta_i0)]
        ptrs = [x.ctypes.data_as(ctypes.c_void_p) for x in u]
        nat.check(nat.load_library().em_td2_forcing(self._plan, *ptrs, nat.ptr(f)),
                  "em_td2_forcing")
        if self._sel is None:
            return f.cpu().numpy()
        out = np.zeros(self._n_full)
        out[self._sel] = f.cpu().numpy()
        return out

    def step(self, modal_state: np.ndarray, i_d, delta_i_d, delta_i0) -> np.ndarray:
        """Advance one step in place (transient.py:157-166); with a selection only the
        selected modes move."""
        n = self._n_full
        if modal_state.shape != (n,):
            raise DimensionMismatch(f"modal state must have {n} components")
        if n == 0 or self._n == 0:
            return modal_state
        sub = modal_state if self._sel is None else modal_state[self._sel]
        q = nat.device_vector(sub)
        u = [np.ascontiguousarray(np.asarray(x, dtype=float)) for x in (i_d, delta_i_d, delta_i0)]
        ptrs = [x.ctypes.data_as(ctypes.c_void_p) for x in u]
        nat.check(nat.load_library().em_td2_step(self._plan, nat.ptr(q), *ptrs), "em_td2_step")
        if self._sel is None:
            modal_state[:] = q.cpu().numpy()
        else:
            modal_state[self._sel] = q.cpu().numpy()
        return modal_state

    def set_observables(self, observables):
        nf = self._n_full
        n_obs, cdev, ddev = _obs_device(observables, nf, self._n_p)
        ctx = nat.context()
        cv = nat.empty(nf, n_obs)  # C V column-major n_obs x n
        nat.check(nat.load_library().em_dgemm(ctx, 0, 0, n_obs, nf, nf, 1.0,
                                               nat.ptr(cdev), n_obs, nat.ptr(self.basis.v_dev),
                                               nf, 0.0, nat.ptr(cv), n_obs), "em_dgemm")
        if self._sel is not None:
            cv = cv.index_select(0, self._sel_dev).contiguous()  # the selected modes' columns
        nat.check(nat.load_library().em_td2_set_observables(
            self._plan, n_obs, nat.ptr(cv), n_obs, nat.ptr(ddev), n_obs), "em_td2_set_observables")
        self._n_obs = n_obs

    def run_device(self, drive_dev, steps: int, q_dev, capture_stride: int = 1,
                   capture_state: bool = False, want_obs: bool = True):
        """Batched device run over a device drive table ((steps+1) x (n_p+n_s)).
        Returns (Y device (n_caps, n_obs) or None, Qcap device (n_caps, N) or None)."""
        n_caps = steps // capture_stride
        y = nat.empty(n_caps, self._n_obs) if (want_obs and getattr(self, "_n_obs", 0)) else None
        qcap = nat.empty(n_caps, self._n) if capture_state else None
        nat.check(nat.load_library().em_td2_run(self._plan, steps, nat.ptr(drive_dev),
                                                 nat.ptr(q_dev), nat.ptr(y), capture_stride,
                                                 nat.ptr(qcap)), "em_td2_run")
        return y, qcap

    def run(self, i_d_samples, i0_samples, capture_stride: int = 1, capture_state: bool = True,
            observables=None, modal_state0=None):
        """Integrate over a sample table (rows t_0..t_T) from rest (or modal_state0).
        Returns (internal_states (n_caps, N) or None, observables or None, final q)."""
        table = _drive_table(i_d_samples, i0_samples, self._n_p, self._n_s) \
            if (self._n_p or self._n_s) else np.zeros((np.asarray(i_d_samples).shape[0], 0))
        steps = table.shape[0] - 1
        if observables is not None:
            self.set_observables(observables)
        drive = nat.device_vector(table.reshape(-1)) if table.size else nat.zeros(1)
        q0 = np.zeros(self._n_full) if modal_state0 is None else \
            np.asarray(modal_state0, dtype=float)
        q = nat.device_vector(q0 if self._sel is None else q0[self._sel])
        y, qcap = self.run_device(drive, steps, q, capture_stride, capture_state,
                                  observables is not None)
        states = None
        if qcap is not None:
            states = _reconstruct(self.basis, qcap, qcap.shape[0], self._sel_dev)
        q_out = q.cpu().numpy()
        if self._sel is not None:
            full = q0.copy()
            full[self._sel] = q_out
            q_out = full
        return states, (y.cpu().numpy() if y is not None else None), q_out

    def run_sweep_device(self, drive_dev, steps: int, q_dev, capture_stride: int = 1,
                         want_obs: bool = True):
        """Device sweep: every drive channel integrated alone (em_td2_run_sweep).
        q_dev: (n_c, N) torch (column-major N x n_c), in/out. Returns Y device
        (n_c, n_caps, n_obs) or None."""
        n_c = self._n_p + self._n_s
        n_caps = steps // capture_stride
        y = nat.empty(n_c, n_caps, self._n_obs) \
            if (want_obs and getattr(self, "_n_obs", 0)) else None
        nat.check(nat.load_library().em_td2_run_sweep(self._plan, steps, nat.ptr(drive_dev),
                                                       nat.ptr(q_dev), nat.ptr(y),
                                                       capture_stride), "em_td2_run_sweep")
        return y

    def run_sweep(self, i_d_samples, i0_samples, capture_stride: int = 1, observables=None,
                  modal_states0=None):
        """Batched-excitation sweep (BASELINE configs[4]): the response to each drive
        channel (ports, then sources) ALONE, all channels integrated in one call — the
        reference would run one trajectory per channel (run_transient superposes them,
        transient.py:147-155). Returns (observables (n_c, n_caps, n_obs) or None,
        final modal states (N, n_c))."""
        n_c = self._n_p + self._n_s
        if n_c == 0:
            raise ValidationError("a sweep needs at least one drive channel")
        table = _drive_table(i_d_samples, i0_samples, self._n_p, self._n_s)
        steps = table.shape[0] - 1
        if observables is not None:
            self.set_observables(observables)
        drive = nat.device_vector(table.reshape(-1))
        q0 = np.zeros((self._n, n_c)) if modal_states0 is None else \
            np.asarray(modal_states0, dtype=float).reshape(self._n, n_c)
        q = nat.device_colmajor(q0)
        y = self.run_sweep_device(drive, steps, q, capture_stride, observables is not None)
        return (y.cpu().numpy() if y is not None else None), \
            nat.host_colmajor(q, self._n, n_c)


def _reconstruct(basis: ModalBasis, qcap, n_caps: int, sel_dev=None) -> np.ndarray:
    """internal states I = V Q for captured modal states (n_caps x N host); sel_dev:
    the modes Q holds (V's columns sel)."""
    n = basis.n_modes
    if n_caps == 0:
        return np.zeros((0, n))
    v = basis.v_dev if sel_dev is None else basis.v_dev.index_select(0, sel_dev).contiguous()
    m = v.shape[0]
    ctx = nat.context()
    out = nat.empty(n_caps, n)
    nat.check(nat.load_library().em_dgemm(ctx, 0, 0, n, n_caps, m, 1.0, nat.ptr(v), n,
                                           nat.ptr(qcap), m, 0.0, nat.ptr(out), n), "em_dgemm")
    return out.cpu().numpy()


class Td1Stepper:
    """Coupled stepper (transient.py:77-113): Cholesky factor of L_i + dt theta R_i."""

    def __init__(self, rm: ReducedModel, dt: float, theta: float):
        _check_theta_dt(dt, theta)
        t0 = time.perf_counter()
        self.rm = rm
        self.dt = float(dt)
        self.theta = float(theta)
        n, n_p, n_s = rm.n_internal, rm.n_ports, rm.n_sources
        self._n, self._n_p, self._n_s = n, n_p, n_s
        self._chol = None
        self._plan = None
        if n:
            ctx = nat.context()
            lib = nat.load_library()
            ld = nat.device_symmetric(rm.l_i.full)   # SymMatrix: exactly symmetric
            rd = nat.device_symmetric(rm.r_i.full)
            dr = nat.device_colmajor(rm.r_d.reshape(n, n_p)) if n_p else nat.zeros(1)
            dl = nat.device_colmajor(rm.l_d.reshape(n, n_p)) if n_p else nat.zeros(1)
            dm = nat.device_colmajor(rm.m0.reshape(n, n_s)) if n_s else nat.zeros(1)
            plan = ctypes.c_void_p()
            piv = ctypes.c_int64(-1)
            rc = lib.em_td1_plan_create(ctx, n, n_p, n_s, nat.ptr(ld), n, nat.ptr(rd), n,
                                        nat.ptr(dr), nat.ptr(dl), nat.ptr(dm), self.dt,
                                        self.theta, ctypes.byref(plan), ctypes.byref(piv))
            if rc == nat.EM_ERR_NOT_PD:
                raise NotPositiveDefinite(int(piv.value), "stepping matrix")
            nat.check(rc, "em_td1_plan_create")
            self._plan = plan
        self.setup_time = time.perf_counter() - t0

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            nat.load_library().em_td1_plan_destroy(plan)
            self._plan = None

    @property
    def chol(self) -> linalg.LowerTriangular | None:
        """The stepping-matrix factor (transient.py:95), copied from the device."""
        if self._plan is None:
            return None
        if self._chol is None:
            out = nat.empty(self._n, self._n)
            nat.check(nat.load_library().em_td1_factor(self._plan, nat.ptr(out), self._n),
                      "em_td1_factor")
            self._chol = linalg.LowerTriangular(nat.host_colmajor(out, self._n, self._n))
        return self._chol

    def step(self, state: np.ndarray, i_d, delta_i_d, delta_i0) -> np.ndarray:
        """Advance one step in place and return the state (transient.py:102-113)."""
        n = self._n
        if state.shape != (n,):
            raise DimensionMismatch(f"state must have {n} components")
        if n == 0:
            return state
        s = nat.device_vector(state)
        u = [np.ascontiguousarray(np.asarray(x, dtype=float)) for x in (i_d, delta_i_d, delta_i0)]
        ptrs = [x.ctypes.data_as(ctypes.c_void_p) for x in u]
        nat.check(nat.load_library().em_td1_step(self._plan, nat.ptr(s), *ptrs), "em_td1_step")
        state[:] = s.cpu().numpy()
        return state

    def set_observables(self, observables):
        n_obs, cdev, ddev = _obs_device(observables, self._n, self._n_p)
        nat.check(nat.load_library().em_td1_set_observables(
            self._plan, n_obs, nat.ptr(cdev), n_obs, nat.ptr(ddev), n_obs), "em_td1_set_observables")
        self._n_obs = n_obs

    def run_device(self, drive_dev, steps: int, i_dev, capture_stride: int = 1,
                   capture_state: bool = False, want_obs: bool = True):
        n_caps = steps // capture_stride
        y = nat.empty(n_caps, self._n_obs) if (want_obs and getattr(self, "_n_obs", 0)) else None
        icap = nat.empty(n_caps, self._n) if capture_state else None
        nat.check(nat.load_library().em_td1_run(self._plan, steps, nat.ptr(drive_dev),
                                                 nat.ptr(i_dev), nat.ptr(y), capture_stride,
                                                 nat.ptr(icap)), "em_td1_run")
        return y, icap

    def run(self, i_d_samples, i0_samples, capture_stride: int = 1, capture_state: bool = True,
            observables=None, state0=None):
        table = _drive_table(i_d_samples, i0_samples, self._n_p, self._n_s) \
            if (self._n_p or self._n_s) else np.zeros((np.asarray(i_d_samples).shape[0], 0))
        steps = table.shape[0] - 1
        if observables is not None:
            self.set_observables(observables)
        drive = nat.device_vector(table.reshape(-1)) if table.size else nat.zeros(1)
        s = nat.device_vector(np.zeros(self._n) if state0 is None else state0)
        y, icap = self.run_device(drive, steps, s, capture_stride, capture_state,
                                  observables is not None)
        states = icap.cpu().numpy() if icap is not None else None
        return states, (y.cpu().numpy() if y is not None else None), s.cpu().numpy()


def prepare_td1(rm: ReducedModel, cfg: TransientConfig) -> Td1Stepper:
    return Td1Stepper(rm, cfg.dt, cfg.theta)


def step_td1(stepper: Td1Stepper, state, i_d, delta_i_d, delta_i0) -> np.ndarray:
    """Functional wrapper over Td1Stepper.step (transient.py:173-178)."""
    return stepper.step(np.asarray(state, dtype=float), np.asarray(i_d, dtype=float),
                        np.asarray(delta_i_d, dtype=float), np.asarray(delta_i0, dtype=float))


def prepare_td2(rm: ReducedModel, basis: ModalBasis, cfg: TransientConfig) -> Td2Stepper:
    return Td2Stepper(rm, basis, cfg.dt, cfg.theta)


def step_td2(stepper: Td2Stepper, modal_state, forcing) -> np.ndarray:
    """Advance modal coordinates one step with a precomputed forcing (transient.py:185-195)."""
    modal_state = np.asarray(modal_state, dtype=float)
    forcing = np.asarray(forcing, dtype=float)
    if forcing.shape != modal_state.shape:
        raise DimensionMismatch("forcing and state sizes differ")
    sel = stepper._sel
    if modal_state.shape[0] and stepper._n:
        q = nat.device_vector(modal_state if sel is None else modal_state[sel])
        f = nat.device_vector(forcing if sel is None else forcing[sel])
        nat.check(nat.load_library().em_td2_step_forcing(stepper._plan, nat.ptr(q), nat.ptr(f)),
                  "em_td2_step_forcing")
        if sel is None:
            modal_state[:] = q.cpu().numpy()
        else:
            modal_state[sel] = q.cpu().numpy()
    return modal_state


def _drive_channels(net, rm: ReducedModel, drives):
    """Port/source name order and per-channel tone lists (transient.py:198-219)."""
    # a geometry-only network (observers need just the segment geometry) names nothing
    if net is not None and hasattr(net, "electrodes"):
        port_names = [el.name for el in net.electrodes[:-1]] if net.n_electrodes else []
        source_names = [c.name for c in net.sources if c.port is None]
    else:
        port_names = list(rm.port_names) or [str(i) for i in range(rm.n_ports)]
        source_names = list(rm.source_names) or [str(i) for i in range(rm.n_sources)]
    if len(port_names) != rm.n_ports or len(source_names) != rm.n_sources:
        raise DimensionMismatch("network and reduced model disagree on ports/sources")
    port_tones: list[list] = [[] for _ in port_names]
    source_tones: list[list] = [[] for _ in source_names]
    for d in drives:
        for p in d.ports:
            if p not in port_names:
                raise ValidationError(f"drive references unknown port {p!r}")
            port_tones[port_names.index(p)].extend(d.tones)
        for s in d.sources:
            if s not in source_names:
                raise ValidationError(f"drive references unknown source {s!r}")
            source_tones[source_names.index(s)].extend(d.tones)
    return port_tones, source_tones


def _sample_channels(tone_lists, t: np.ndarray) -> np.ndarray:
    """Per-channel multisine samples at times t, (len(t), n_ch); per channel the
    tones are accumulated in order from 0.0 like np.add.at in transient.py:237-241."""
    out = np.zeros((t.shape[0], len(tone_lists)))
    for ch, tones in enumerate(tone_lists):
        for tone in tones:
            out[:, ch] += tone.amplitude * np.sin((2 * np.pi * tone.frequency) * t + tone.phase)
    return out


def drive_samples(net, rm: ReducedModel, drives, dt: float, n_steps: int):
    """The sample table run_transient steps through: t_0 = 0, t_{k+1} = (k+1) dt."""
    if isinstance(drives, DriveSignal):
        drives = (drives,)
    port_tones, source_tones = _drive_channels(net, rm, drives)
    t = np.concatenate([[0.0], np.arange(1, n_steps + 1, dtype=float) * dt])
    return _sample_channels(port_tones, t), _sample_channels(source_tones, t)


def run_transient(rm: ReducedModel, net, drives, cfg: TransientConfig,
                  modal: ModalBasis | None = None, observables=None,
                  modes=None) -> SimulationResult:
    """Integrate from rest, capture every capture_stride steps (transient.py:248-312).

    observables: optional (C, D) with C (n_obs x N) and D (n_obs x n_ports) or None;
    captured values are C I + D i_D(t_{k+1}) for each capture. modes (td2 only): the
    selective integration of PAPER.md:299 (see select_modes)."""
    if isinstance(drives, DriveSignal):
        drives = (drives,)
    if cfg.method == "td2" and modal is None:
        raise ValidationError("td2 requires a modal basis")
    probe_cd = None
    if cfg.probes is not None:
        # probe observers (transient.py:266-273): fields = transfer @ (W K I + W lift i_D)
        from .observers import probe_observables
        probe_cd = probe_observables(net, rm, cfg.probes)
        if observables is not None:
            raise ValidationError("pass either cfg.probes or observables, not both")
    n_steps = cfg.n_steps
    i_d_tab, i0_tab = drive_samples(net, rm, drives, cfg.dt, n_steps)
    n_caps = n_steps // cfg.capture_stride
    times = cfg.dt * cfg.capture_stride * np.arange(1, n_caps + 1)

    setup0 = time.perf_counter()
    if cfg.method == "td1":
        stepper = Td1Stepper(rm, cfg.dt, cfg.theta)
    else:
        stepper = Td2Stepper(rm, modal, cfg.dt, cfg.theta, modes=modes)
    nat.synchronize()
    setup_time = time.perf_counter() - setup0

    if rm.n_internal == 0:
        states = np.zeros((n_caps, 0)) if cfg.capture_state else None
        return SimulationResult(times, states, None, setup_time, 0.0, n_steps, cfg.method)
    step0 = time.perf_counter()
    fields = None
    if probe_cd is None:
        states, obs, _ = stepper.run(i_d_tab, i0_tab, cfg.capture_stride, cfg.capture_state,
                                     observables)
    else:
        # at most 128 observables per scan: 42 probes (3 components each) per run
        c, d = probe_cd
        parts, states, obs = [], None, None
        for r0 in range(0, c.shape[0], 126):
            st, y, _ = stepper.run(i_d_tab, i0_tab, cfg.capture_stride,
                                   cfg.capture_state and r0 == 0,
                                   (c[r0:r0 + 126], d[r0:r0 + 126] if d.shape[1] else None))
            states = st if r0 == 0 else states
            parts.append(y)
        fields = np.concatenate(parts, axis=1).reshape(n_caps, -1, 3)
    nat.synchronize()
    stepping_time = time.perf_counter() - step0
    return SimulationResult(times=times, internal_states=states, probe_fields=fields,
                            wall_time_setup=setup_time, wall_time_stepping=stepping_time,
                            n_steps=n_steps, method=cfg.method, observables=obs)


def exact_first_order(l_n: np.ndarray, r_n: np.ndarray, y0: np.ndarray,
                      e0: np.ndarray, slope: np.ndarray, h: float) -> np.ndarray:
    """Closed-form step of l y' + r y = e0 + slope t (transient.py:352-360), per
    component (a small host formula, as in the reference)."""
    tau = l_n / r_n
    yp0 = (e0 - slope * tau) / r_n
    yph = (e0 + slope * h - slope * tau) / r_n
    return yph + (y0 - yp0) * np.exp(-h / tau)


def exact_modal_reference(basis: ModalBasis, rm: ReducedModel, i_d_samples, i0_samples,
                          times, modal_state0=None) -> np.ndarray:
    """Exact per-interval integration of every mode for piecewise-linear drives
    (transient.py:315-349), on the device: per mode q^{k+1} = a q^k + c1 e0 + c2 s with
    a = exp(-h r/l) is the same linear recurrence as the theta-method, so it runs as one
    blocked scan (em_td2_plan_create_exact + em_td2_run). The scan needs one factor a
    per mode, i.e. uniformly spaced sample times (ValidationError otherwise).
    Returns modal coordinates at every sample time, shape (len(times), n_modes)."""
    times = np.asarray(times, dtype=float)
    n_t = times.shape[0]
    n, n_p, n_s = basis.n_modes, rm.n_ports, rm.n_sources
    i_d_samples = np.asarray(i_d_samples, dtype=float).reshape(n_t, n_p)
    i0_samples = np.asarray(i0_samples, dtype=float).reshape(n_t, n_s)
    q0 = np.zeros(n) if modal_state0 is None else np.asarray(modal_state0, float).copy()
    if q0.shape != (n,):
        raise DimensionMismatch(f"modal state must have {n} components")
    out = np.zeros((n_t, n))
    if n_t == 0:
        return out
    out[0] = q0
    if n_t == 1 or n == 0:
        return out
    steps = n_t - 1
    h = (times[-1] - times[0]) / steps
    if not h > 0 or np.max(np.abs(np.diff(times) - h)) > 1e-9 * h:
        raise ValidationError("exact_modal_reference on the device needs uniformly spaced, "
                              "increasing sample times")
    ctx, lib = nat.context(), nat.load_library()
    proj = _drive_projection(rm, basis)
    p_r = proj[0:n_p] if n_p else proj[0:1]
    p_l = proj[n_p:2 * n_p] if n_p else proj[0:1]
    p_m = proj[2 * n_p:] if n_s else proj[0:1]
    ln, rn = nat.device_vector(basis.l_n), nat.device_vector(basis.r_n)
    plan = ctypes.c_void_p()
    nat.check(lib.em_td2_plan_create_exact(ctx, n, n_p, n_s, nat.ptr(ln), nat.ptr(rn),
                                           nat.ptr(p_r), nat.ptr(p_l), nat.ptr(p_m), h,
                                           ctypes.byref(plan)), "em_td2_plan_create_exact")
    try:
        table = _drive_table(i_d_samples, i0_samples, n_p, n_s) if (n_p or n_s) \
            else np.zeros((n_t, 0))
        drive = nat.device_vector(table.reshape(-1)) if table.size else nat.zeros(1)
        q = nat.device_vector(q0)
        qcap = nat.empty(steps, n)
        nat.check(lib.em_td2_run(plan, steps, nat.ptr(drive), nat.ptr(q), None, 1,
                                 nat.ptr(qcap)), "em_td2_run")
        out[1:] = qcap.cpu().numpy()
    finally:
        lib.em_td2_plan_destroy(plan)
    return out


# --- CSV export (transient.py:363-404) -----------------------------------------------

def write_timeseries_csv(path, result: SimulationResult, header_lines: tuple[str, ...] = ()):
    if result.probe_fields is None:
        raise ValidationError("result holds no probe fields")
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(f"# {line}\n")
        fh.write("t,probe_id,Bx,By,Bz\n")
        for it, t in enumerate(result.times):
            for p in range(result.probe_fields.shape[1]):
                bx, by, bz = (float(v) for v in result.probe_fields[it, p])
                fh.write(f"{float(t)!r},{p},{bx!r},{by!r},{bz!r}\n")


def write_states_csv(path, result: SimulationResult, header_lines: tuple[str, ...] = ()):
    if result.internal_states is None:
        raise ValidationError("result holds no internal states")
    n = result.internal_states.shape[1]
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(f"# {line}\n")
        fh.write("t," + ",".join(f"i{j}" for j in range(n)) + "\n")
        for it, t in enumerate(result.times):
            row = ",".join(repr(float(v)) for v in result.internal_states[it])
            fh.write(f"{float(t)!r},{row}\n")


def write_timing_csv(path, results: list[SimulationResult], header_lines: tuple[str, ...] = ()):
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(f"# {line}\n")
        fh.write("method,setup_s,stepping_s,steps,per_step_s\n")
        for r in results:
            fh.write(f"{r.method},{r.wall_time_setup!r},{r.wall_time_stepping!r},"
                     f"{r.n_steps},{r.per_step_cost!r}\n")


class ImplicitTd2:
    """The modal transient without forming the eigenvectors ("implicit V"):
    em_sygv_implicit applies V^T = U^T Q^T G^-1 to the drive columns [R_D | L_D | M0]
    and the observable rows C^T only, so the eigensolve skips the 4 N^3 flops that form
    V (the Q2 and Q1 back-transforms). The scan is the same em_td2 plan as Td2Stepper's,
    with l_n = tau, r_n = 1 (V^T L V = diag(tau), V^T R V = I). Observables (C, D) are
    fixed at construction; run() returns them exactly as Td2Stepper.run does. V, the
    modal states' signs and the reconstructed currents are not available on this path.
    """

    def __init__(self, rm: ReducedModel, observables, dt: float, theta: float):
        _check_theta_dt(dt, theta)
        t0 = time.perf_counter()
        self.rm, self.dt, self.theta = rm, float(dt), float(theta)
        n, n_p, n_s = rm.n_internal, rm.n_ports, rm.n_sources
        self._n, self._n_p, self._n_s = n, n_p, n_s
        c, d = observables if isinstance(observables, tuple) else (observables, None)
        c = np.atleast_2d(np.asarray(c, dtype=float))
        if c.shape[1] != n:
            raise DimensionMismatch(f"observables need {n} columns, got {c.shape}")
        n_obs = c.shape[0]
        if n_obs > 128:
            raise ValidationError("at most 128 observables per run")
        nd = 2 * n_p + n_s
        cols = [rm.r_d.reshape(n, n_p), rm.l_d.reshape(n, n_p), rm.m0.reshape(n, n_s), c.T]
        y = nat.device_colmajor(np.concatenate(cols, axis=1))      # (nd + n_obs, n)
        lm, rmat = rm.l_i.full, rm.r_i.full
        dl, dr = nat.device_symmetric(lm), nat.device_symmetric(rmat)
        tau = nat.empty(n)
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        rc = nat.load_library().em_sygv_implicit(
            nat.context(), n, nat.ptr(dl), n, nat.ptr(dr), n, nat.ptr(tau), nat.ptr(y), n,
            nd + n_obs, None, None, 1, ctypes.byref(piv), ctypes.byref(which))
        if rc == nat.EM_ERR_NOT_PD:
            from .errors import NotPositiveDefinite
            what = "modal resistance matrix" if which.value == 0 else "modal inductance matrix"
            raise NotPositiveDefinite(int(piv.value), what)
        nat.check(rc, "em_sygv_implicit")
        del dl, dr
        self.tau = tau.cpu().numpy()
        self._ln = tau
        self._rn = nat.torch().ones(n, dtype=nat.torch().float64, device="cuda")
        proj = y[:max(nd, 1)] if nd else nat.zeros(1, n)
        self._proj = proj
        p_r = proj[0:n_p] if n_p else proj[0:1]
        p_l = proj[n_p:2 * n_p] if n_p else proj[0:1]
        p_m = proj[2 * n_p:nd] if n_s else proj[0:1]
        plan = ctypes.c_void_p()
        nat.check(nat.load_library().em_td2_plan_create(
            nat.context(), n, n_p, n_s, nat.ptr(self._ln), nat.ptr(self._rn), nat.ptr(p_r),
            nat.ptr(p_l), nat.ptr(p_m), self.dt, self.theta, ctypes.byref(plan)),
            "em_td2_plan_create")
        self._plan = plan
        cv = y[nd:nd + n_obs].t().contiguous()                     # C V column-major n_obs x n
        self._cv = cv
        dd = None
        if d is not None and n_p:
            dd = nat.device_colmajor(np.asarray(d, dtype=float).reshape(n_obs, n_p))
        self._dd = dd
        nat.check(nat.load_library().em_td2_set_observables(
            plan, n_obs, nat.ptr(cv), n_obs, nat.ptr(dd), n_obs), "em_td2_set_observables")
        self._n_obs = n_obs
        self.setup_time = time.perf_counter() - t0

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            nat.load_library().em_td2_plan_destroy(plan)
            self._plan = None

    def run(self, i_d_samples, i0_samples, capture_stride: int = 1):
        """Observables (n_caps, n_obs) over a sample table (rows t_0..t_T) from rest."""
        table = _drive_table(i_d_samples, i0_samples, self._n_p, self._n_s) \
            if (self._n_p or self._n_s) else np.zeros((np.asarray(i_d_samples).shape[0], 0))
        steps = table.shape[0] - 1
        drive = nat.device_vector(table.reshape(-1)) if table.size else nat.zeros(1)
        q = nat.zeros(self._n)
        y = nat.empty(steps // capture_stride, self._n_obs)
        nat.check(nat.load_library().em_td2_run(self._plan, steps, nat.ptr(drive), nat.ptr(q),
                                                 nat.ptr(y), capture_stride, None), "em_td2_run")
        return y.cpu().numpy()
