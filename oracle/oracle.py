"""CPU ORACLE — test infrastructure only, never the product path.

A restatement of the reference's hot path (package `eddymodes`,
/root/reference/pkg/src/eddymodes) used to check the CUDA implementation:

* the compiled numerics (_kernels.py:18-222) are restated in plain C
  (oracle/eddy_oracle.c, loaded here through ctypes) in the same operation
  order, so they reproduce the reference's numba kernels bit for bit;
* the Python layers around them (linalg.py, modal.py, transient.py) are
  restated below with numpy, each function citing the file:line it follows.

Pinning: tests/test_oracle.py checks this oracle against the golden fixtures
in tests/golden/, which were produced by running the unmodified reference
(tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libeddy_oracle.so")

JACOBI_TOL = 1e-14          # linalg.py:18-21
JACOBI_MAX_SWEEPS = 50


class OracleNotPositiveDefinite(Exception):
    def __init__(self, pivot: int, what: str):
        self.pivot = pivot
        self.what = what
        super().__init__(f"{what} is not positive definite (pivot {pivot} <= 0)")


class OracleNoConvergence(Exception):
    pass


def build() -> str:
    """Compile eddy_oracle.c with strict IEEE semantics (no contraction)."""
    os.makedirs(os.path.dirname(_SO), exist_ok=True)
    src = os.path.join(_HERE, "eddy_oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        _lib.orc_cholesky.argtypes = [d, d, i64]
        _lib.orc_cholesky.restype = i64
        _lib.orc_tri_solve_vec.argtypes = [d, d, d, d, i64]
        _lib.orc_tri_lower_solve_mat.argtypes = [d, d, i64, i64]
        _lib.orc_tri_lower_t_solve_mat.argtypes = [d, d, i64, i64]
        _lib.orc_jacobi.argtypes = [d, d, i64, i64, ctypes.c_double]
        _lib.orc_jacobi.restype = i64
        _lib.orc_jacobi_rotations.argtypes = [d, d, i64, i64]
        _lib.orc_jacobi_rotations.restype = i64
        _lib.orc_td1_step.argtypes = [d, d, d, ctypes.c_double, d, d, d, d, i64]
        _lib.orc_td2_step.argtypes = [d, d, d, ctypes.c_double, d, i64]
        _lib.orc_td2_run.argtypes = [d, d, d, ctypes.c_double, d, d, d, i64, i64, i64, d, i64,
                                     d, i64, i64, d, d]
        _lib.orc_lu_factor.argtypes = [d, ctypes.c_void_p, i64]
        _lib.orc_lu_factor.restype = i64
        _lib.orc_lu_solve.argtypes = [d, ctypes.c_void_p, d, i64]
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous and a.dtype == np.float64
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# --- linalg.py ----------------------------------------------------------------

def sym_mirror(a) -> np.ndarray:
    """linalg.py:34-41 SymMatrix: lower triangle mirrored (exactly symmetric)."""
    a = np.asarray(a, dtype=float)
    lower = np.tril(a)
    return lower + np.tril(lower, -1).T


def cholesky(a, what: str = "matrix") -> np.ndarray:
    """linalg.py:92-104 -> _kernels.py:18-36."""
    a = np.ascontiguousarray(a, dtype=float)
    c = np.zeros_like(a)
    piv = lib().orc_cholesky(_p(a), _p(c), a.shape[0])
    if piv >= 0:
        raise OracleNotPositiveDefinite(int(piv), what)
    return c


def solve_cholesky(c: np.ndarray, b: np.ndarray) -> np.ndarray:
    """linalg.py:107-116 -> _kernels.py:39-53."""
    c = np.ascontiguousarray(c, dtype=float)
    b = np.ascontiguousarray(b, dtype=float)
    y = np.empty_like(b)
    x = np.empty_like(b)
    lib().orc_tri_solve_vec(_p(c), _p(b), _p(y), _p(x), c.shape[0])
    return x


def sym_eig(a) -> tuple[np.ndarray, np.ndarray]:
    """linalg.py:119-134: Jacobi, then descending order with stable ties."""
    a = np.ascontiguousarray(a, dtype=float).copy()
    n = a.shape[0]
    v = np.eye(n)
    sweeps = lib().orc_jacobi(_p(a), _p(v), n, JACOBI_MAX_SWEEPS, JACOBI_TOL)
    if sweeps < 0:
        raise OracleNoConvergence("Jacobi did not converge")
    lam = np.diag(a).copy()
    order = np.argsort(-lam, kind="stable")
    return lam[order], np.ascontiguousarray(v[:, order])


# --- modal.py -----------------------------------------------------------------

@dataclass
class Basis:
    v: np.ndarray
    tau: np.ndarray
    l_n: np.ndarray
    r_n: np.ndarray
    vt_r: np.ndarray


def _finish_basis(v: np.ndarray, tau: np.ndarray, lm: np.ndarray, rm: np.ndarray) -> Basis:
    """modal.py:74-81: sign fix (largest |entry| positive), l_n, r_n, vt_r."""
    n = v.shape[0]
    idx = np.argmax(np.abs(v), axis=0)
    signs = np.sign(v[idx, np.arange(n)])
    signs[signs == 0] = 1.0
    v = v * signs[None, :]
    l_n = np.einsum("ij,ij->j", v, lm @ v)
    r_n = np.einsum("ij,ij->j", v, rm @ v)
    return Basis(v=v, tau=tau.copy(), l_n=l_n, r_n=r_n, vt_r=v.T @ rm)


def generalized_eig(l_i, r_i) -> Basis:
    """modal.py:46-81 with the reference's Jacobi eigensolver (O(sweeps N^3))."""
    lm = np.asarray(l_i, dtype=float)
    rm = np.asarray(r_i, dtype=float)
    n = lm.shape[0]
    g = cholesky(rm, what="modal resistance matrix")
    b = np.ascontiguousarray(lm.copy())
    lib().orc_tri_lower_solve_mat(_p(g), _p(b), n, n)
    bt = np.ascontiguousarray(b.T)
    lib().orc_tri_lower_solve_mat(_p(g), _p(bt), n, n)
    b = 0.5 * (bt + bt.T)
    cholesky(lm, what="modal inductance matrix")
    tau, u = sym_eig(b)
    v = np.ascontiguousarray(u)
    lib().orc_tri_lower_t_solve_mat(_p(g), _p(v), n, n)
    return _finish_basis(v, tau, lm, rm)


def generalized_eig_lapack(l_i, r_i) -> Basis:
    """Restatement of modal.py:46-81 for N where Jacobi is infeasible: LAPACK
    dsygvd (potrf + sygst + syevd + trsm: the same Cholesky reduction), then
    the reference's descending order, sign fix and l_n/r_n/vt_r (modal.py:74-81).
    Labelled a restatement wherever it is used."""
    import scipy.linalg as sl
    lm = np.asarray(l_i, dtype=float)
    rm = np.asarray(r_i, dtype=float)
    w, v = sl.eigh(lm, rm, driver="gvd", lower=True)
    order = np.argsort(-w, kind="stable")
    return _finish_basis(np.ascontiguousarray(v[:, order]), w[order], lm, rm)


def drive_rhs(r_d, l_d, m0, i_d, delta_i_d, delta_i0, dt, theta) -> np.ndarray:
    """modal.py:121-131."""
    n = r_d.shape[0]
    rhs = np.zeros(n)
    if r_d.shape[1]:
        rhs -= dt * (r_d @ i_d)
        rhs -= (l_d + dt * theta * r_d) @ delta_i_d
    if m0.shape[1]:
        rhs -= m0 @ delta_i0
    return rhs


# --- transient.py ---------------------------------------------------------------

def tone_sampler(tones_per_channel):
    """transient.py:221-243: per-channel sums of amp*sin(omega t + phase) via np.add.at."""
    amps, omegas, phases, owner = [], [], [], []
    for ch, tones in enumerate(tones_per_channel):
        for (amp, freq, ph) in tones:
            amps.append(amp)
            omegas.append(2 * np.pi * freq)
            phases.append(ph)
            owner.append(ch)
    n_ch = len(tones_per_channel)
    amps, omegas, phases = np.array(amps), np.array(omegas), np.array(phases)
    owner = np.array(owner, dtype=np.int64)

    def sample(t):
        out = np.zeros(n_ch)
        if amps.size:
            np.add.at(out, owner, amps * np.sin(omegas * t + phases))
        return out
    return sample


def sample_table(sample, steps: int, dt: float) -> np.ndarray:
    """Samples at t_k = k*dt exactly as run_transient evaluates them (transient.py:290-296)."""
    rows = [sample(0.0)] + [sample((k + 1) * dt) for k in range(steps)]
    return np.array(rows).reshape(steps + 1, -1)


class Td1:
    """transient.py:77-113 (Td1Stepper) over the C kernels."""

    def __init__(self, l_i, r_i, r_d, l_d, m0, dt, theta):
        self.r = np.ascontiguousarray(r_i, dtype=float)
        self.r_d, self.l_d, self.m0 = r_d, l_d, m0
        self.dt, self.theta = float(dt), float(theta)
        z = np.asarray(l_i) + self.dt * self.theta * self.r
        self.chol = cholesky(z, what="stepping matrix")
        n = self.r.shape[0]
        self._b, self._y, self._x = np.empty(n), np.empty(n), np.empty(n)

    def step(self, state, i_d, d_id, d_i0):
        extra = np.ascontiguousarray(drive_rhs(self.r_d, self.l_d, self.m0, i_d, d_id, d_i0,
                                               self.dt, self.theta))
        lib().orc_td1_step(_p(self.chol), _p(self.r), _p(state), self.dt, _p(extra),
                           _p(self._b), _p(self._y), _p(self._x), state.shape[0])
        return state


class Td2:
    """transient.py:116-166 (Td2Stepper) over the C kernels."""

    def __init__(self, basis: Basis, r_d, l_d, m0, dt, theta):
        self.basis = basis
        self.dt, self.theta = float(dt), float(theta)
        den = basis.l_n + self.dt * self.theta * basis.r_n
        self._c = np.sqrt(den)
        self._rn = basis.r_n.copy()
        n = basis.tau.shape[0]
        vt = basis.v.T
        self.n_p, self.n_s = r_d.shape[1], m0.shape[1]
        self._p_r = vt @ r_d if self.n_p else np.zeros((n, 0))
        self._p_l = vt @ l_d if self.n_p else np.zeros((n, 0))
        self._p_m = vt @ m0 if self.n_s else np.zeros((n, 0))
        self._p_ltr = self._p_l + self.dt * self.theta * self._p_r

    def forcing(self, i_d, d_id, d_i0):
        f = np.zeros(self.basis.tau.shape[0])
        if self.n_p:
            f -= self.dt * (self._p_r @ i_d)
            f -= self._p_ltr @ d_id
        if self.n_s:
            f -= self._p_m @ d_i0
        return f

    def step(self, q, i_d, d_id, d_i0):
        f = np.ascontiguousarray(self.forcing(i_d, d_id, d_i0))
        lib().orc_td2_step(_p(q), _p(self._rn), _p(self._c), self.dt, _p(f), q.shape[0])
        return q


def td2_run_table(l_n, r_n, p_r, p_l, p_m, dt, theta, tab, steps, cv=None, stride=1, q0=None):
    """run_transient's td2 loop (transient.py:293-306) in C (orc_td2_run) for a modal
    model given directly by l_n, r_n and the drive projections P = V^T [R_D | L_D | M0]
    (n x n_p, n x n_p, n x n_s), as Td2Stepper.__init__ forms them (transient.py:122-145).
    Returns (q after the last step, observables (steps // stride, n_obs) = (C V) q or None)."""
    n = l_n.shape[0]
    den = l_n + float(dt) * float(theta) * r_n
    c = np.ascontiguousarray(np.sqrt(den))
    rn = np.ascontiguousarray(r_n, dtype=float)
    n_p, n_s = p_r.shape[1], p_m.shape[1]
    pr = np.ascontiguousarray(p_r, dtype=float).reshape(n, n_p)
    pltr = np.ascontiguousarray(p_l + float(dt) * float(theta) * p_r, dtype=float).reshape(n, n_p)
    pm = np.ascontiguousarray(p_m, dtype=float).reshape(n, n_s)
    tab = np.ascontiguousarray(tab, dtype=float)
    q = np.zeros(n) if q0 is None else np.ascontiguousarray(q0, dtype=float).copy()
    n_caps = steps // stride
    obs = None
    if cv is not None:
        cv = np.ascontiguousarray(cv, dtype=float)
        obs = np.zeros((n_caps, cv.shape[0]))
    f = np.empty(n)
    z = np.zeros(1)
    lib().orc_td2_run(_p(q), _p(rn), _p(c), float(dt), _p(pr) if n_p else _p(z),
                      _p(pltr) if n_p else _p(z), _p(pm) if n_s else _p(z), n, n_p, n_s,
                      _p(tab), int(steps), _p(cv) if cv is not None else _p(z),
                      cv.shape[0] if cv is not None else 0, int(stride),
                      _p(obs) if obs is not None else None, _p(f))
    return q, obs


def run(stepper, n: int, i_d_tab: np.ndarray, i0_tab: np.ndarray, modal: Basis | None,
        c_obs: np.ndarray | None = None, capture_stride: int = 1, capture_state: bool = True,
        max_steps: int | None = None):
    """transient.py:248-312 (run_transient) driven by a sample table (rows t_0..t_T).

    Returns (states (n_caps, N) or None, observables (n_caps, n_obs) or None).
    td2 reconstructs internal = V q at every capture (transient.py:301)."""
    steps = i_d_tab.shape[0] - 1 if max_steps is None else max_steps
    n_caps = steps // capture_stride
    states = np.zeros((n_caps, n)) if capture_state else None
    obs = np.zeros((n_caps, c_obs.shape[0])) if c_obs is not None else None
    state = np.zeros(n)
    cap = 0
    for k in range(steps):
        stepper.step(state, i_d_tab[k], i_d_tab[k + 1] - i_d_tab[k], i0_tab[k + 1] - i0_tab[k])
        if (k + 1) % capture_stride == 0:
            internal = modal.v @ state if modal is not None else state
            if states is not None:
                states[cap] = internal
            if obs is not None:
                obs[cap] = c_obs @ internal
            cap += 1
    return states, obs


def exact_first_order(l_n, r_n, y0, e0, slope, h):
    """transient.py:352-360."""
    tau = l_n / r_n
    yp0 = (e0 - slope * tau) / r_n
    yph = (e0 + slope * h - slope * tau) / r_n
    return yph + (y0 - yp0) * np.exp(-h / tau)


def exact_modal_reference(basis: Basis, r_d, l_d, m0, i_d_samples, i0_samples, times):
    """transient.py:315-349: exact per-interval integration for piecewise-linear drives."""
    n_t = times.shape[0]
    n = basis.tau.shape[0]
    vt = basis.v.T
    p_r = vt @ r_d if r_d.shape[1] else np.zeros((n, 0))
    p_l = vt @ l_d if l_d.shape[1] else np.zeros((n, 0))
    p_m = vt @ m0 if m0.shape[1] else np.zeros((n, 0))
    out = np.zeros((n_t, n))
    state = np.zeros(n)
    for k in range(n_t - 1):
        h = times[k + 1] - times[k]
        di_d = (i_d_samples[k + 1] - i_d_samples[k]) / h
        di_0 = (i0_samples[k + 1] - i0_samples[k]) / h
        e0 = -(p_r @ i_d_samples[k]) - (p_l @ di_d) - (p_m @ di_0)
        s = -(p_r @ di_d)
        state = exact_first_order(basis.l_n, basis.r_n, state, e0, s, h)
        out[k + 1] = state
    return out


# --- frequency domain (E/frequency.py) -------------------------------------------------

def lu_factor(a: np.ndarray):
    """linalg.py:137-147 + _kernels.py:144-170 (pivoted LU); SingularSystem on a zero pivot."""
    a = np.ascontiguousarray(a, dtype=float).copy()
    piv = np.zeros(a.shape[0], dtype=np.int64)
    col = lib().orc_lu_factor(_p(a), piv.ctypes.data_as(ctypes.c_void_p), a.shape[0])
    if col >= 0:
        raise RuntimeError(f"zero pivot in column {col}")
    return a, piv


def lu_solve(lu_piv, b: np.ndarray) -> np.ndarray:
    """linalg.py:150-156 + _kernels.py:173-193."""
    lu, piv = lu_piv
    x = np.ascontiguousarray(b, dtype=float).copy()
    lib().orc_lu_solve(_p(lu), piv.ctypes.data_as(ctypes.c_void_p), _p(x), lu.shape[0])
    return x


def solve_tone(r_i, l_i, r_d, l_d, m0, omega, i_d_phasor, i0_phasor) -> np.ndarray:
    """frequency.py:56-94: (R + j w L) I = -(R_D + j w L_D) i_D - j w M0 i0 through the
    real 2n embedding [[R, wL], [wL, -R]] and the pivoted LU."""
    r, l = sym_mirror(r_i), sym_mirror(l_i)
    n = r.shape[0]
    e = np.zeros(n, dtype=complex)
    if r_d.shape[1]:
        e -= (r_d + 1j * omega * l_d) @ np.asarray(i_d_phasor, dtype=complex)
    if m0.shape[1]:
        e -= 1j * omega * (m0 @ np.asarray(i0_phasor, dtype=complex))
    big = np.zeros((2 * n, 2 * n))
    big[:n, :n] = r
    big[:n, n:] = omega * l
    big[n:, :n] = omega * l
    big[n:, n:] = -r
    x = lu_solve(lu_factor(big), np.concatenate([e.real, e.imag]))
    return x[:n] - 1j * x[n:]


def dft_phasor(samples, dt, f, t0=0.0) -> complex:
    """frequency.py:114-138 (Im convention: sin(w t) -> 1 + 0j)."""
    samples = np.asarray(samples, dtype=float)
    n = samples.shape[0]
    t = t0 + dt * np.arange(n)
    w = 2 * np.pi * f
    return 1j * ((2.0 / n) * np.sum(samples * np.exp(-1j * w * t)))
