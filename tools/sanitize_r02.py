"""Small workload for compute-sanitizer (measurement tool, not product): the one-stage
eigensolve (sytrd PDL column chain + CUDA graph), the two-stage eigensolve (cooperative
panel QR, flag-chained bulge chasing, register-resident Q2 with its mbarrier ring), the
TD1 solves (sentinel-polled persistent kernels) and a TD2 run, at N ~ 1000.

    compute-sanitizer --tool memcheck python tools/sanitize_r02.py
    compute-sanitizer --tool racecheck python tools/sanitize_r02.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_11993_b200 import _native as nat  # noqa: E402
from paper_2407_11993_b200 import modal, reduction, transient  # noqa: E402
from paper_2407_11993_b200.synth import plate_model  # noqa: E402


def main():
    m = plate_model(32, 16, 2, n_ports=1, n_sources=1, n_obs=8)  # N = 1024, b = 32
    rm = reduction.from_blocks(m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"],
                               port_names=("p0",), source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)           # one-stage
    nat.set_two_stage_min(0)
    basis2 = modal.generalized_eig(rm.l_i, rm.r_i)          # two-stage
    nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    dt, steps = 1e-6, 100
    i_d, i0 = (np.minimum(dt * np.arange(steps + 1) / 5e-6, 1.0)[:, None],
               np.sin(2 * np.pi * 1e4 * dt * np.arange(steps + 1))[:, None])
    obs = (m["c"], None)
    _, y2, _ = transient.Td2Stepper(rm, basis, dt, 0.5).run(i_d, i0, capture_state=False,
                                                              observables=obs)
    _, y1, _ = transient.Td1Stepper(rm, dt, 0.5).run(i_d[:21], i0[:21], capture_state=False,
                                                      observables=obs)
    nat.synchronize()
    err = np.abs(basis.tau - basis2.tau).max() / basis.tau.max()
    print(f"sanitize workload done: N={rm.n_internal} tau(1-stage vs 2-stage) {err:.1e} "
          f"td1 vs td2 {np.abs(y1 - y2[:20]).max() / np.abs(y2[:20]).max():.1e}")


if __name__ == "__main__":
    main()
