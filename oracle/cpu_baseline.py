"""CPU ORACLE timing leg — test/benchmark infrastructure only.

Times the reference algorithm on this host's cores and extrapolates the full
end-to-end time of a configuration from bounded samples. The work timed is
exactly what modal.generalized_eig + run_transient do
(pkg/src/eddymodes/modal.py:46-81, transient.py:248-312), through the bit-exact C
restatement of the reference's numba kernels (oracle/eddy_oracle.c) and numpy/BLAS
for its GEMMs:

  eigensolve stages, each timed on seeded synthetic plates of the config's construction
  at three sample orders and fitted by t = a n^3 (the fit's worst relative residual and
  the free-exponent fit are reported):
    cholesky(R)  cholesky(L)            _kernels.py:18-36
    sygst: 2 x tri_lower_solve_mat      _kernels.py:56-66
    cyclic Jacobi                       _kernels.py:82-141: sweeps x n(n-1)/2 rotations; the
                                        sweep count to convergence is measured by full runs
                                        on small plates and fitted s0 + s1 ln n; the cost of
                                        one rotation (row and column-strided updates of A and
                                        V) is timed on n x n matrices of three orders beyond
                                        the caches and fitted a n
    back-transform tri_lower_t_solve    _kernels.py:69-79
    l_n, r_n, V^T R (numpy GEMMs)       modal.py:79-81
  stepping, per step (transient.py:293-306):
    Td2Stepper.forcing + td2_step_kernel  timed for >= 100 steps at the FULL N
    from_modal V @ q (every capture)      dense GEMV, timed at three orders and fitted by
                                          t = a n^2; the benchmark's cpu_baseline leg also
                                          times it at the full N on the device's own V
                                          (reported beside the fit)

Every extrapolated figure is labelled `extrapolated`. Used only by bench.py (the
cpu_baseline leg and --impl reference), never by the product path.
"""
from __future__ import annotations

import os
import platform
import time

import numpy as np

from . import oracle as O

CUBIC_SIZES = (384, 512, 768)      # voxel plates (k x 8 x 2) of these orders
SWEEP_SIZES = (128, 192, 256)      # full Jacobi runs (sweep counts)
ROTATION_SIZES = (4096, 6144, 8192)
GEMV_SIZES = (2048, 4096, 8192)


def _timeit(fn, reps=1):
    fn()  # first call outside the timing (page faults, BLAS thread start)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _fit(sizes, times, power):
    """t = a n^power by least squares in relative terms; worst relative residual and the
    free-exponent (log-log) fit for reference."""
    x = np.asarray(sizes, dtype=float) ** power
    t = np.asarray(times, dtype=float)
    a = float(np.sum(t / x) / len(x))
    resid = float(np.max(np.abs(t / (a * x) - 1.0)))
    p_free = float(np.polyfit(np.log(sizes), np.log(np.maximum(t, 1e-12)), 1)[0])
    return a, resid, p_free


_CACHE: dict = {}


def _plate_pair(n_s: int, seed: int):
    """Mirrored (L, R) of the seeded k x 8 x 2 plate of order n_s (cached per process:
    the samples are repeated once per benchmark step)."""
    key = ("plate", n_s, seed)
    if key not in _CACHE:
        from paper_2407_11993_b200.synth import plate_model
        m = plate_model(n_s // 16, 8, 2, n_ports=1, n_sources=1, n_obs=4, seed=seed)
        _CACHE[key] = (O.sym_mirror(m["l_i"]), O.sym_mirror(m["r_i"]))
    return _CACHE[key]


def _dense_pair(n: int, seed: int):
    """A dense symmetric n x n matrix and an n x n identity (cached; rotation timing only)."""
    key = ("dense", n, seed)
    if key not in _CACHE:
        a = np.random.default_rng(seed + n).standard_normal((n, n))
        a += a.T
        _CACHE[key] = (a, np.eye(n))
    return _CACHE[key]


def jacobi_samples(sweep_sizes=SWEEP_SIZES, rot_sizes=ROTATION_SIZES, rotations: int = 64,
                   seed: int = 20240807) -> dict:
    """Sweep counts of full Jacobi runs on reduced plate matrices, and the per-rotation
    time on dense n x n matrices (orc_jacobi_rotations: the reference's rotation loop)."""
    lib = O.lib()
    sweeps = []
    for n_s in sweep_sizes:
        lm, rm = _plate_pair(n_s, seed)
        n = lm.shape[0]
        g = O.cholesky(rm)
        b = np.ascontiguousarray(lm.copy())
        lib.orc_tri_lower_solve_mat(O._p(g), O._p(b), n, n)
        bt = np.ascontiguousarray(b.T)
        lib.orc_tri_lower_solve_mat(O._p(g), O._p(bt), n, n)
        a = np.ascontiguousarray(0.5 * (bt + bt.T))
        v = np.eye(n)
        sweeps.append(int(lib.orc_jacobi(O._p(a), O._p(v), n, O.JACOBI_MAX_SWEEPS,
                                         O.JACOBI_TOL)))
    t_rot = []
    for n in rot_sizes:
        a, v = _dense_pair(n, seed)
        lib.orc_jacobi_rotations(O._p(a), O._p(v), n, 4)
        t0 = time.perf_counter()
        done = lib.orc_jacobi_rotations(O._p(a), O._p(v), n, rotations)
        t_rot.append((time.perf_counter() - t0) / max(int(done), 1))
    return {"sweep_sizes": list(sweep_sizes), "sweeps": sweeps, "rot_sizes": list(rot_sizes),
            "rotation_s": t_rot}


def eigensolve_samples(sizes=CUBIC_SIZES, seed: int = 20240807) -> dict:
    """Per-stage times of the reference eigensolve (all but Jacobi) on plates of the
    given orders."""
    lib = O.lib()
    rows = {k: [] for k in ("cholesky_R", "sygst", "cholesky_L", "back_transform", "gemms")}
    for n_s in sizes:
        lm, rm = _plate_pair(n_s, seed)
        n = lm.shape[0]
        c = np.zeros_like(rm)
        rows["cholesky_R"].append(_timeit(lambda: lib.orc_cholesky(O._p(rm), O._p(c), n)))
        g = O.cholesky(rm)

        def sygst():
            b = np.ascontiguousarray(lm.copy())
            lib.orc_tri_lower_solve_mat(O._p(g), O._p(b), n, n)
            bt = np.ascontiguousarray(b.T)
            lib.orc_tri_lower_solve_mat(O._p(g), O._p(bt), n, n)
            return 0.5 * (bt + bt.T)
        rows["sygst"].append(_timeit(sygst))
        b = sygst()
        rows["cholesky_L"].append(_timeit(lambda: lib.orc_cholesky(O._p(lm), O._p(c), n)))
        u = np.ascontiguousarray(np.linalg.qr(b)[0])  # an orthonormal n x n stand-in for U
        rows["back_transform"].append(
            _timeit(lambda: lib.orc_tri_lower_t_solve_mat(O._p(g), O._p(u.copy()), n, n)))
        rows["gemms"].append(_timeit(lambda: (lm @ u, rm @ u, u.T @ rm)))
    return {"sizes": list(sizes), "times_s": rows}


def gemv_samples(sizes=GEMV_SIZES, reps: int = 5) -> dict:
    """from_modal's V @ q (modal.py:93-98) on dense n x n operands."""
    times = []
    for n in sizes:
        v, _ = _dense_pair(n, 1)
        q = np.random.default_rng(n).standard_normal(n)
        times.append(_timeit(lambda: v @ q, reps))
    return {"sizes": list(sizes), "times_s": times}


def stepping_sample(n: int, n_p: int, n_s: int, dt: float, steps: int = 100) -> float:
    """Seconds per step of Td2Stepper.forcing + td2_step_kernel at order n
    (transient.py:147-166, _kernels.py:213-222), from the reference's own loop."""
    rng = np.random.default_rng(2)
    tau = np.exp(rng.uniform(np.log(0.05), np.log(60.0), size=n))
    basis = O.Basis(v=None, tau=tau, l_n=tau.copy(), r_n=np.ones(n), vt_r=None)
    st = O.Td2.__new__(O.Td2)
    st.basis, st.dt, st.theta = basis, float(dt), 0.5
    st._c = np.sqrt(basis.l_n + st.dt * st.theta * basis.r_n)
    st._rn = basis.r_n.copy()
    st.n_p, st.n_s = n_p, n_s
    st._p_r = rng.standard_normal((n, n_p))
    st._p_l = rng.standard_normal((n, n_p))
    st._p_m = rng.standard_normal((n, n_s))
    st._p_ltr = st._p_l + st.dt * st.theta * st._p_r
    q = np.zeros(n)
    u_d, u_s = np.ones(n_p), np.ones(n_s)
    return _timeit(lambda: st.step(q, u_d, u_d, u_s), steps)


def estimate(n: int, n_p: int, n_s: int, steps: int, n_runs: int, dt: float,
             v_full: np.ndarray | None = None, cubic_sizes=CUBIC_SIZES,
             gemv_sizes=GEMV_SIZES, step_samples: int = 100) -> dict:
    """Extrapolated reference end-to-end time of one eigensolve + n_runs transients of
    `steps` steps (n_runs: theta values x sweep channels) at order n."""
    eig = eigensolve_samples(cubic_sizes)
    comp, fits = {}, {}
    for k, ts in eig["times_s"].items():
        a, resid, p = _fit(eig["sizes"], ts, 3)
        comp[f"{k}_s"] = a * float(n) ** 3
        fits[k] = {"a": a, "max_rel_residual": resid, "free_exponent": p}
    jac = jacobi_samples()
    s1, s0 = np.polyfit(np.log(jac["sweep_sizes"]), jac["sweeps"], 1)
    sweeps_n = float(min(max(s0 + s1 * np.log(n), max(jac["sweeps"])), O.JACOBI_MAX_SWEEPS))
    a1, r1, p1 = _fit(jac["rot_sizes"], jac["rotation_s"], 1)
    comp["jacobi_s"] = sweeps_n * n * (n - 1) / 2 * a1 * n
    fits["jacobi_rotation"] = {"a": a1, "max_rel_residual": r1, "free_exponent": p1}
    fits["jacobi_sweeps"] = {"measured": dict(zip(jac["sweep_sizes"], jac["sweeps"])),
                             "fit": [float(s0), float(s1)], "at_N": sweeps_n}
    gv = gemv_samples(gemv_sizes)
    a2, r2, p2 = _fit(gv["sizes"], gv["times_s"], 2)
    t_gemv = a2 * float(n) ** 2
    fits["from_modal_gemv"] = {"a": a2, "max_rel_residual": r2, "free_exponent": p2}
    t_kernel = stepping_sample(n, n_p, n_s, dt, step_samples)
    gemv_full = None
    if v_full is not None:
        q = np.random.default_rng(3).standard_normal(v_full.shape[1])
        gemv_full = _timeit(lambda: v_full @ q, 10)
    per_step = t_kernel + (gemv_full if gemv_full is not None else t_gemv)
    comp["stepping_s"] = n_runs * steps * per_step
    total = sum(comp.values())
    cores = len(os.sched_getaffinity(0))
    return {
        "total_s": total,
        "components": comp,
        "fits": fits,
        "per_step_ms": per_step * 1e3,
        "step_kernel_ms": t_kernel * 1e3,
        "from_modal_gemv_ms_fit": t_gemv * 1e3,
        "from_modal_gemv_ms_full_n": gemv_full * 1e3 if gemv_full is not None else None,
        "cores": cores,
        "cpu_model": cpu_model(),
        "extrapolated": True,
        "sample": (f"reference kernels (C restatement of _kernels.py, single-threaded) + numpy "
                   f"BLAS on {cores} host threads ({cpu_model()}): every eigensolve stage timed "
                   f"on seeded plates of order {list(cubic_sizes)} and extrapolated by a n^3 "
                   f"to N={n}; Jacobi = fitted sweeps ({sweeps_n:.1f} at N) x N(N-1)/2 x the "
                   f"rotation time fitted at {list(ROTATION_SIZES)}; Td2Stepper step kernel timed over {step_samples} steps at N={n}; "
                   f"from_modal V@q timed at {list(gemv_sizes)} (a n^2)"
                   + (f" and at N={n} on the solved V" if gemv_full is not None else "")
                   + f"; x {steps} steps x {n_runs} runs; extrapolated"),
    }
