"""Generalized symmetric-definite eigendecomposition and the modal coordinate
transform — the reference's modal module (pkg/src/eddymodes/modal.py:1-142)
on the B200 library.

generalized_eig runs entirely on the device (em_sygv): blocked DMMA Cholesky of
R, the two-sided reduction exactly as the reference forms it, the Cholesky
certificate of L, Householder tridiagonalisation + divide and conquer (instead
of cyclic Jacobi), back-transform V = G^-T U, descending order, sign fix and
l_n / r_n / V^T R. The N x N results stay device-resident; ModalBasis.v and
.vt_r materialise host copies on first access (the reference holds them
eagerly as numpy arrays).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import linalg
from .errors import DimensionMismatch, NotPositiveDefinite
from .reduction import ReducedModel


class ModalBasis:
    """Generalized eigenpairs of L_i v = tau R_i v (modal.py:22-43).

    v: (n, n) R-orthonormal eigenvector columns, sign-fixed (largest-magnitude
    entry positive); tau: time constants, descending; l_n, r_n: per-mode
    inductance / resistance; vt_r: V^T R_i.
    """

    __slots__ = ("_v", "_vt_r", "tau", "l_n", "r_n", "_v_dev", "_vtr_dev", "_r_dev", "_frozen")

    def __init__(self, v=None, tau=None, l_n=None, r_n=None, vt_r=None, *, v_dev=None,
                 vtr_dev=None, r_dev=None):
        object.__setattr__(self, "_v", None if v is None else np.asarray(v, dtype=float))
        object.__setattr__(self, "_vt_r", None if vt_r is None else np.asarray(vt_r, dtype=float))
        object.__setattr__(self, "tau", np.asarray(tau, dtype=float))
        object.__setattr__(self, "l_n", np.asarray(l_n, dtype=float))
        object.__setattr__(self, "r_n", np.asarray(r_n, dtype=float))
        object.__setattr__(self, "_v_dev", v_dev)
        object.__setattr__(self, "_vtr_dev", vtr_dev)
        # device R_i kept for a deferred V^T R (large n: not formed during the eigensolve)
        object.__setattr__(self, "_r_dev", r_dev)
        object.__setattr__(self, "_frozen", True)

    def __setattr__(self, key, value):
        raise AttributeError("ModalBasis is immutable")

    @property
    def n_modes(self) -> int:
        return self.tau.shape[0]

    @property
    def v(self) -> np.ndarray:
        if self._v is None:
            n = self.n_modes
            object.__setattr__(self, "_v", nat.host_colmajor(self._v_dev, n, n))
        return self._v

    @property
    def vt_r(self) -> np.ndarray:
        if self._vt_r is None:
            n = self.n_modes
            # the device buffer is R V column-major == V^T R row-major
            object.__setattr__(self, "_vt_r",
                               np.ascontiguousarray(self.vtr_dev.reshape(n, n).cpu().numpy()))
        return self._vt_r

    # device views -------------------------------------------------------------
    @property
    def v_dev(self):
        """Column-major V on the device (torch tensor shaped (n, n))."""
        if self._v_dev is None:
            object.__setattr__(self, "_v_dev", nat.device_colmajor(self._v))
        return self._v_dev

    @property
    def vtr_dev(self):
        """R V column-major on the device (== V^T R row-major)."""
        if self._vtr_dev is None and self._r_dev is not None:
            n = self.n_modes
            rv = nat.empty(n, n)
            nat.check(nat.load_library().em_sym_mm(nat.context(), n, n, nat.ptr(self._r_dev), n,
                                                   nat.ptr(self.v_dev), n, nat.ptr(rv), n),
                      "em_sym_mm")
            object.__setattr__(self, "_vtr_dev", rv)
            object.__setattr__(self, "_r_dev", None)
        if self._vtr_dev is None:
            object.__setattr__(self, "_vtr_dev", nat.device_vector(
                np.ascontiguousarray(self._vt_r).reshape(-1)).reshape(self.n_modes,
                                                                      self.n_modes))
        return self._vtr_dev


def _host_square(a) -> np.ndarray:
    return a.full if isinstance(a, linalg.SymMatrix) else np.asarray(a, dtype=float)


def generalized_eig(l_i, r_i, *, vt_r: str = "auto") -> ModalBasis:
    """Solve L_i V = tau R_i V for an SPD pair (modal.py:46-81).

    vt_r: "eager" forms V^T R_i inside the eigensolve (as the reference does),
    "lazy" defers it to the first access of ModalBasis.vt_r / vtr_dev (one fewer
    N x N buffer at the eigensolve's memory peak), "auto" is eager while the device
    has room for it.

    Raises NotPositiveDefinite("modal resistance matrix" / "modal inductance
    matrix") with the failing pivot, in the reference's order."""
    t = nat.torch()
    own = False  # R uploaded here: usable as the factor workspace (EM_SYGV_R_WORKSPACE)
    l_host = None  # L left on the host for em_sygv_lh
    if isinstance(l_i, t.Tensor) and isinstance(r_i, t.Tensor):
        # device-resident symmetric inputs (row-major bytes == column-major)
        ld = l_i.to(dtype=t.float64).contiguous()
        rd = r_i.to(dtype=t.float64).contiguous()
        if ld.shape != rd.shape:
            raise DimensionMismatch("L_i and R_i must have the same shape")
        n = ld.shape[0]
    else:
        lm, rm = _host_square(l_i), _host_square(r_i)
        if lm.shape != rm.shape:
            raise DimensionMismatch("L_i and R_i must have the same shape")
        n = lm.shape[0]
        if n == 0:
            z = np.zeros(0)
            zz = np.zeros((0, 0))
            return ModalBasis(v=zz, tau=z, l_n=z, r_n=z, vt_r=zz)
        # SymMatrix is exactly symmetric: upload its bytes as they are. R goes first; an
        # exactly symmetric L is uploaded by the library on a copy engine while R is
        # factored (em_sygv_lh)
        rd = nat.device_symmetric(rm) if isinstance(r_i, linalg.SymMatrix) else \
            nat.device_colmajor(rm)
        if isinstance(l_i, linalg.SymMatrix):
            l_host = np.ascontiguousarray(lm, dtype=np.float64)
            ld = nat.empty(n, n)
        else:
            ld = nat.device_colmajor(lm)
        own = True
    ctx = nat.context()
    if vt_r not in ("auto", "eager", "lazy"):
        raise ValueError("vt_r must be 'auto', 'eager' or 'lazy'")
    if vt_r == "auto":
        free = t.cuda.mem_get_info()[0]
        # V, V^T R and the eigensolver's own G, B, two D&C matrices + slack
        vt_r = "eager" if 7.5 * 8.0 * n * n < free else "lazy"
    tau, ln, rn = nat.empty(n), nat.empty(n), nat.empty(n)
    v = nat.empty(n, n)
    vtr = nat.empty(n, n) if vt_r == "eager" else None
    piv = ctypes.c_int64(-1)
    which = ctypes.c_int(-1)
    lib = nat.load_library()
    common = (nat.ptr(rd), n, nat.ptr(tau), nat.ptr(v), n, nat.ptr(ln), nat.ptr(rn),
              None if vtr is None else nat.ptr(vtr), n, 1 if own else 0, ctypes.byref(piv),
              ctypes.byref(which))
    if l_host is not None:
        rc = lib.em_sygv_lh(ctx, n, l_host.ctypes.data, nat.ptr(ld), n, *common)
    else:
        rc = lib.em_sygv_ex(ctx, n, nat.ptr(ld), n, *common)
    if rc == nat.EM_ERR_NOT_PD:
        what = "modal resistance matrix" if which.value == 0 else "modal inductance matrix"
        raise NotPositiveDefinite(int(piv.value), what)
    nat.check(rc, "em_sygv")
    return ModalBasis(tau=tau.cpu().numpy(), l_n=ln.cpu().numpy(), r_n=rn.cpu().numpy(),
                      v_dev=v, vtr_dev=vtr, r_dev=rd if vtr is None else None)


def _gemv(a_dev, trans: int, n: int, x: np.ndarray) -> np.ndarray:
    ctx = nat.context()
    xd = nat.device_vector(x)
    yd = nat.empty(n)
    nat.check(nat.load_library().em_dgemm(ctx, trans, 0, n, 1, n, 1.0, nat.ptr(a_dev), n,
                                           nat.ptr(xd), n, 0.0, nat.ptr(yd), n), "em_dgemm")
    return yd.cpu().numpy()


def to_modal(basis: ModalBasis, i_internal: np.ndarray) -> np.ndarray:
    """Modal coordinates V^T R_i I (modal.py:84-90)."""
    i_internal = np.asarray(i_internal, dtype=float)
    if i_internal.shape != (basis.n_modes,):
        raise DimensionMismatch(f"expected {basis.n_modes} components, got {i_internal.shape}")
    # vtr_dev holds R V column-major; (R V)^T I = V^T R I
    return _gemv(basis.vtr_dev, 1, basis.n_modes, i_internal)


def from_modal(basis: ModalBasis, modal: np.ndarray) -> np.ndarray:
    """Internal current vector V m (modal.py:93-98)."""
    modal = np.asarray(modal, dtype=float)
    if modal.shape != (basis.n_modes,):
        raise DimensionMismatch(f"expected {basis.n_modes} components, got {modal.shape}")
    return _gemv(basis.v_dev, 0, basis.n_modes, modal)


def drive_rhs(rm: ReducedModel, i_d: np.ndarray, delta_i_d: np.ndarray,
              delta_i0: np.ndarray, dt: float, theta: float) -> np.ndarray:
    """Drive part of the coupled theta-step right-hand side (modal.py:121-131):
    -dt R_D i_D - (L_D + dt theta R_D) delta_i_D - M0 delta_i0. O(N n_d) host
    arithmetic, exactly as the reference; the batched device paths form the
    same expression on the GPU."""
    rhs = np.zeros(rm.n_internal)
    if rm.n_ports:
        rhs -= dt * (rm.r_d @ i_d)
        rhs -= (rm.l_d + dt * theta * rm.r_d) @ delta_i_d
    if rm.n_sources:
        rhs -= rm.m0 @ delta_i0
    return rhs


def modal_forcing(basis: ModalBasis, rm: ReducedModel, i_d: np.ndarray,
                  delta_i_d: np.ndarray, delta_i0: np.ndarray,
                  dt: float, theta: float) -> np.ndarray:
    """V^T applied to the drive part of the coupled right-hand side (modal.py:101-118)."""
    i_d = np.asarray(i_d, dtype=float)
    delta_i_d = np.asarray(delta_i_d, dtype=float)
    delta_i0 = np.asarray(delta_i0, dtype=float)
    if i_d.shape != (rm.n_ports,) or delta_i_d.shape != (rm.n_ports,):
        raise DimensionMismatch(f"expected {rm.n_ports} port currents")
    if delta_i0.shape != (rm.n_sources,):
        raise DimensionMismatch(f"expected {rm.n_sources} source increments")
    rhs = drive_rhs(rm, i_d, delta_i_d, delta_i0, dt, theta)
    return _gemv(basis.v_dev, 1, basis.n_modes, rhs)


def write_modal_csv(path, basis: ModalBasis, header_lines: tuple[str, ...] = ()):
    """Mode table export: n, tau_s, L_n_H, R_n_ohm (modal.py:134-142)."""
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(f"# {line}\n")
        fh.write("n,tau_s,L_n_H,R_n_ohm\n")
        for i in range(basis.n_modes):
            fh.write(f"{i},{float(basis.tau[i])!r},{float(basis.l_n[i])!r},"
                     f"{float(basis.r_n[i])!r}\n")


def implicit_eig(l_i, r_i, y, *, r_band: int | None = None, l_workspace: bool = False):
    """tau (descending) and V^T Y for the pencil L_i V = tau R_i V without forming V
    (em_sygv_implicit / em_sygv_implicit_band; SURVEY.md §7 "implicit V"). Y is (n, k).
    r_band: pass R_i as LAPACK lower band storage of that bandwidth (host (bw+1, n) array or
    a dense R_i that is banded). l_workspace: L_i's device copy is reduced in place.

    V's per-mode signs are the eigensolver's (the reference's sign fix needs V), so each row
    of V^T Y is determined up to sign; products of two rows, (V^T Y)^T (V^T Y) = Y^T R^-1 Y
    and (V^T Y)^T diag(tau) (V^T Y) = Y^T R^-1 L R^-1 Y are not."""
    lm, rm = _host_square(l_i), _host_square(r_i)
    n = lm.shape[0]
    y = np.asarray(y, dtype=float).reshape(n, -1)
    k = y.shape[1]
    ld = nat.device_symmetric(lm)
    dy = nat.device_colmajor(y)
    tau = nat.empty(max(n, 1))
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    flags = nat.EM_SYGV_L_WORKSPACE if l_workspace else 0
    lib = nat.load_library()
    if r_band is not None:
        bw = int(r_band)
        rb = np.zeros((n, bw + 1))  # column j of band storage = R[j:j+bw+1, j]
        for q in range(bw + 1):
            rb[:n - q, q] = np.diagonal(rm, -q)
        drb = nat.device_colmajor(rb.T)  # column-major (bw+1) x n
        rc = lib.em_sygv_implicit_band(nat.context(), n, nat.ptr(ld), n, nat.ptr(drb), bw + 1,
                                       bw, nat.ptr(tau), nat.ptr(dy), n, k, None, None, flags,
                                       ctypes.byref(piv), ctypes.byref(which))
    else:
        dr = nat.device_symmetric(rm)
        rc = lib.em_sygv_implicit(nat.context(), n, nat.ptr(ld), n, nat.ptr(dr), n,
                                  nat.ptr(tau), nat.ptr(dy), n, k, None, None, flags,
                                  ctypes.byref(piv), ctypes.byref(which))
    if rc == nat.EM_ERR_NOT_PD:
        what = "modal resistance matrix" if which.value == 0 else "modal inductance matrix"
        raise NotPositiveDefinite(int(piv.value), what)
    nat.check(rc, "em_sygv_implicit")
    return tau.cpu().numpy()[:n], nat.host_colmajor(dy, n, k)
