"""CPU ORACLE timing leg — test/benchmark infrastructure only.

Times the reference algorithm (the bit-exact C restatement of its numba kernels
in oracle/eddy_oracle.c plus numpy/BLAS for its GEMMs, exactly the work
modal.generalized_eig + run_transient do, pkg/src/eddymodes/modal.py:46-81,
transient.py:390-454) on this host's cores, on a BOUNDED sample of a
configuration, and extrapolates the full end-to-end time by each stage's
operation-count law:

  cholesky(R), cholesky(L)            N^3/3   -> sampled at n_s x n_s, scaled (N/n_s)^3
  sygst (2 solves) + back-transform   3 x N^3 -> tri_lower_solve_mat n_s x n_s, scaled
  cyclic Jacobi                        sweeps * N(N-1)/2 rotations -> rotations timed on
                                       the full N x N matrix (column-strided access
                                       included), sweeps = 12 (measured at N=1000-2000)
  l_n, r_n, V^T R (numpy GEMMs)        3 x 2N^3 -> numpy matmul at n_s, scaled
  stepping                             per step: Td2Stepper.step + V@q (every capture,
                                       transient.py:443), timed on full-N steps

Used only by bench.py (cpu_baseline leg and --impl reference).
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import oracle as O

JACOBI_SWEEPS_ASSUMED = 12


def _timeit(fn, reps=1):
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def estimate(l_i: np.ndarray, r_i: np.ndarray, r_d: np.ndarray, l_d: np.ndarray, m0: np.ndarray,
             steps: int, n_theta: int, dt: float, n_sample: int = 1024, rotations: int = 64,
             sample_steps: int = 4) -> dict:
    n = l_i.shape[0]
    ns = min(n_sample, n)
    scale3 = (n / ns) ** 3
    lib = O.lib()
    # cubic stages on a leading block
    rb = np.ascontiguousarray(r_i[:ns, :ns])
    lb = np.ascontiguousarray(l_i[:ns, :ns])
    c = np.zeros_like(rb)
    t_chol = _timeit(lambda: lib.orc_cholesky(O._p(rb), O._p(c), ns))
    g = O.cholesky(rb)
    bb = lb.copy()
    t_solve = _timeit(lambda: lib.orc_tri_lower_solve_mat(O._p(g), O._p(bb), ns, ns))
    a2 = np.ascontiguousarray(l_i[:ns, :ns])
    t_gemm = _timeit(lambda: a2 @ a2)
    # Jacobi rotations on the full matrix
    a = np.ascontiguousarray(l_i.copy())
    v = np.eye(n)
    t0 = time.perf_counter()
    done = lib.orc_jacobi_rotations(O._p(a), O._p(v), n, rotations)
    t_rot = (time.perf_counter() - t0) / max(done, 1)
    del a
    # stepping: the reference Td2Stepper.step + from_modal V@q per step (full N)
    q = np.zeros(n)
    r_n = np.ones(n)
    c_n = np.sqrt(np.ones(n))
    pr = v[:, :max(r_d.shape[1], 1)].copy()

    def one_step():
        f = np.zeros(n)
        if r_d.shape[1]:
            f -= dt * (pr[:, :r_d.shape[1]] @ np.ones(r_d.shape[1]))
            f -= pr[:, :r_d.shape[1]] @ np.ones(r_d.shape[1])
        lib.orc_td2_step(O._p(q), O._p(r_n), O._p(c_n), dt, O._p(np.ascontiguousarray(f)), n)
        return l_i @ q                      # V @ q stand-in (same size and layout)
    one_step()
    t_step = _timeit(one_step, reps=sample_steps)
    del v
    comp = {
        "cholesky_R_s": t_chol * scale3,
        "sygst_2_solves_s": 2 * t_solve * scale3,
        "cholesky_L_s": t_chol * scale3,
        "jacobi_s": JACOBI_SWEEPS_ASSUMED * n * (n - 1) / 2 * t_rot,
        "back_transform_s": t_solve * scale3,
        "gemms_s": 3 * t_gemm * scale3,
        "stepping_s": n_theta * steps * t_step,
    }
    total = sum(comp.values())
    cores = len(os.sched_getaffinity(0))
    return {
        "total_s": total,
        "components": comp,
        "per_rotation_us": t_rot * 1e6,
        "per_step_ms": t_step * 1e3,
        "cores": cores,
        "sample": (f"reference kernels (C restatement, single-threaded) + numpy BLAS on "
                   f"{cores} host threads: cholesky/solves/GEMMs timed at n={ns} and scaled by "
                   f"(N/n)^3, {done} Jacobi rotations timed at N={n} x {JACOBI_SWEEPS_ASSUMED} "
                   f"sweeps x N(N-1)/2, {sample_steps} full-N TD2 steps (step + V@q) x "
                   f"{steps} steps x {n_theta} theta; extrapolated"),
    }
