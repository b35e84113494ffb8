"""Repetition checks for the kernels that synchronise across CTAs (compute-sanitizer is
closed on this pool: see profiles/r02/compute_sanitizer_closed.txt). A race between CTAs
shows up as run-to-run differences, so each is run repeatedly on the same inputs and
must reproduce its output BIT FOR BIT: the two-stage eigensolve (cooperative panel QR,
flag-chained bulge chasing, the register-resident Q2 with its mbarrier ring and staging
copies — the staging race of round 2 was caught exactly this way, tools/dbg_q2.py), the
one-stage eigensolve (PDL column chain), the TD1 solves (sentinel-polled persistent
kernels) and the TD2 scan."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _syev(a, reps):
    import torch
    from paper_2407_11993_b200 import _native as nat
    n = a.shape[0]
    lib, ctx = nat.load_library(), nat.context()
    out = []
    for _ in range(reps):
        ad = nat.device_vector(a.reshape(-1))
        w = torch.empty(n, device="cuda", dtype=torch.float64)
        u = torch.empty(n * n, device="cuda", dtype=torch.float64)
        nat.check(lib.em_syev(ctx, n, nat.ptr(ad), n, nat.ptr(w), nat.ptr(u), n), "em_syev")
        out.append((w.cpu().numpy(), u.cpu().numpy()))
    return out


@pytest.mark.parametrize("two_stage,n", [(True, 5000), (True, 9800), (False, 3000)])
def test_eigensolve_bitwise_repeatable(two_stage, n):
    from paper_2407_11993_b200 import _native as nat
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    a = b + b.T
    if two_stage:
        nat.set_two_stage_min(0)
    try:
        runs = _syev(a, 4)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    for w, u in runs[1:]:
        assert np.array_equal(w, runs[0][0]) and np.array_equal(u, runs[0][1])


def test_td1_and_td2_bitwise_repeatable():
    from paper_2407_11993_b200 import modal, reduction, transient
    from paper_2407_11993_b200.synth import drive_table, plate_model
    m = plate_model(40, 24, 2, n_ports=1, n_sources=1, n_obs=8)  # N = 1920: 30 TD1 blocks
    rm = reduction.from_blocks(m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"],
                               port_names=("p0",), source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    i_d, i0 = drive_table("tone50k", 300, 2e-7, 1, 1)
    obs = (m["c"], None)
    y1 = [transient.Td1Stepper(rm, 2e-7, 0.5).run(i_d, i0, capture_state=False,
                                                  observables=obs)[1] for _ in range(4)]
    y2 = [transient.Td2Stepper(rm, basis, 2e-7, 0.5).run(i_d, i0, capture_state=False,
                                                         observables=obs)[1] for _ in range(4)]
    for y in y1[1:]:
        assert np.array_equal(y, y1[0])
    for y in y2[1:]:
        assert np.array_equal(y, y2[0])
    assert np.abs(y1[0] - y2[0]).max() <= 1e-8 * np.abs(y2[0]).max()
