"""Device time stepping vs the reference trajectories (golden fixtures from the
unmodified reference run_transient) — north-star tolerance 1e-8 relative L2
for observables and current densities — plus the SPEC acceptance properties the
reference suite never tested (TD1 == TD2, theta convergence)."""
import os

import numpy as np
import pytest

from oracle import oracle
from tests.conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-8  # north_star: observable waveforms and current densities, relative L2


def _plate_rm(g):
    from paper_2407_11993_b200 import reduction
    return reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], g["m0"],
                                 port_names=("p0",), source_names=("s0",))


def _plate_drives():
    from paper_2407_11993_b200.network import DriveSignal, Tone
    return (DriveSignal(tones=(Tone(1.0, 1e4, 0.0),), sources=("s0",)),
            DriveSignal(tones=(Tone(0.7, 2e4, 0.3), Tone(0.2, 5e4, 1.1)), ports=("p0",)))


@pytest.mark.parametrize("name", ["plate_small", "plate_200"])
@pytest.mark.parametrize("method", ["td2", "td1"])
def test_run_transient_matches_reference(name, method):
    from paper_2407_11993_b200 import modal, transient
    g = golden(name)
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i) if method == "td2" else None
    steps, dt, ke = int(g["steps"]), float(g["dt"]), int(g["keep_every"])
    for th in g["thetas"]:
        th = float(th)
        cfg = transient.TransientConfig(theta=th, dt=dt, t_end=steps * dt, method=method)
        res = transient.run_transient(rm, None, _plate_drives(), cfg, modal=basis,
                                      observables=(g["c"], None))
        assert res.n_steps == steps and res.internal_states.shape == (steps, rm.n_internal)
        ref_obs = g[f"{method}_obs_theta{th}"]
        assert rel_l2(res.observables, ref_obs) < TOL
        assert rel_l2(res.internal_states[ke - 1::ke], g[f"{method}_states_theta{th}"]) < TOL
        np.testing.assert_allclose(res.times, dt * np.arange(1, steps + 1))


@pytest.mark.parametrize("name", ["tube_small", "tube_ref"])
def test_tube_trajectories_match_reference(name):
    """Degenerate tube spectrum: V differs by rotations inside clusters, the
    trajectory I = V q must not."""
    from paper_2407_11993_b200 import modal, reduction, transient
    from paper_2407_11993_b200.network import DriveSignal, Tone
    g = golden(name)
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], None, port_names=("p",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    dt = float(g["dt"])
    drive = DriveSignal(tones=(Tone(1.0, 1e3, 0.0),), ports=("p",))
    for method in ("td2", "td1"):
        cfg = transient.TransientConfig(theta=1.0, dt=dt, t_end=200 * dt, method=method)
        res = transient.run_transient(rm, None, drive, cfg,
                                      modal=basis if method == "td2" else None)
        assert rel_l2(res.internal_states, g[f"{method}_states"]) < TOL


def test_capture_stride_and_state_flags():
    from paper_2407_11993_b200 import modal, transient
    g = golden("plate_small")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    dt = float(g["dt"])
    full = g["td2_obs_theta0.5"]
    for stride in (1, 7, 64, 300):
        cfg = transient.TransientConfig(theta=0.5, dt=dt, t_end=300 * dt, method="td2",
                                        capture_stride=stride, capture_state=False)
        res = transient.run_transient(rm, None, _plate_drives(), cfg, modal=basis,
                                      observables=(g["c"], None))
        assert res.internal_states is None
        assert res.observables.shape == (300 // stride, g["c"].shape[0])
        assert rel_l2(res.observables, full[stride - 1::stride][:300 // stride]) < TOL


def test_step_api_matches_oracle_per_step():
    """Td2Stepper.step / Td1Stepper.step / step_td2 keep the reference's
    in-place single-step semantics."""
    from oracle import oracle as O
    from paper_2407_11993_b200 import modal, transient
    g = golden("plate_small")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    ref = O.generalized_eig(rm.l_i.full, rm.r_i.full)
    dt, th = 1e-6, 0.5
    s2 = transient.Td2Stepper(rm, basis, dt, th)
    s1 = transient.Td1Stepper(rm, dt, th)
    o1 = O.Td1(rm.l_i.full, rm.r_i.full, g["r_d"], g["l_d"], g["m0"], dt, th)
    q = np.zeros(rm.n_internal)
    i1 = np.zeros(rm.n_internal)
    i1_ref = np.zeros(rm.n_internal)
    rng = np.random.default_rng(5)
    for _ in range(20):
        u = rng.standard_normal(3)
        out = s2.step(q, u[:1], u[1:2], u[2:])
        assert out is q
        s1.step(i1, u[:1], u[1:2], u[2:])
        o1.step(i1_ref, u[:1], u[1:2], u[2:])
    assert rel_l2(basis.v @ q, i1_ref) < 1e-10
    assert rel_l2(i1, i1_ref) < 1e-10
    from paper_2407_11993_b200.modal import drive_rhs
    f = s2.forcing(np.ones(1), np.ones(1), np.ones(1))
    f_ref = basis.v.T @ drive_rhs(rm, np.ones(1), np.ones(1), np.ones(1), dt, th)
    assert rel_l2(f, f_ref) < 1e-10
    o2 = O.Td2(ref, g["r_d"], g["l_d"], g["m0"], dt, th)
    q2 = q.copy()
    transient.step_td2(s2, q2, f)
    q3 = q.copy()
    s2.step(q3, np.ones(1), np.ones(1), np.ones(1))
    assert rel_l2(q2, q3) < 1e-14
    c = s1.chol.c
    z = rm.l_i.full + dt * th * rm.r_i.full
    assert np.linalg.norm(c @ c.T - z) <= 1e-12 * np.linalg.norm(z)
    assert o2 is not None


def test_td1_equals_td2_long_horizon():
    """SPEC acceptance #1: TD1 == TD2 to < 1e-8 over 10^4 steps."""
    from paper_2407_11993_b200 import modal, transient
    g = golden("plate_200")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), 1e-6, 10000)
    c = g["c"]
    _, y2, _ = transient.Td2Stepper(rm, basis, 1e-6, 0.5).run(i_d, i0, capture_state=False,
                                                               observables=(c, None))
    _, y1, _ = transient.Td1Stepper(rm, 1e-6, 0.5).run(i_d, i0, capture_state=False,
                                                        observables=(c, None))
    assert rel_l2(y2, y1) < 1e-8


def test_theta_convergence_orders():
    """SPEC acceptance #3: dt halving error ratios ~2 (theta=1) and
    ~4 (theta=0.5) against the exact modal integrator, moderate dt/tau."""
    from paper_2407_11993_b200 import modal, reduction, transient
    g = golden("plate_small")
    # scale R so dt/tau is moderate (the exact oracle's cancellation floor)
    rm = reduction.from_blocks(g["r_i"] * 2e3, g["l_i"], g["r_d"] * 2e3, g["l_d"], g["m0"],
                               port_names=("p0",), source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    t_end = 4e-4

    def final_state(theta, dt):
        n = int(round(t_end / dt))
        i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), dt, n)
        _, _, q = transient.Td2Stepper(rm, basis, dt, theta).run(i_d, i0, capture_state=False)
        return q

    n_ref = 4000
    i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), t_end / n_ref, n_ref)
    # the independent host restatement of exact_modal_reference (oracle/oracle.py)
    exact = oracle.exact_modal_reference(basis, rm.r_d, rm.l_d, rm.m0, i_d, i0,
                                         t_end / n_ref * np.arange(n_ref + 1))[-1]
    for theta, order in ((1.0, 2.0), (0.5, 4.0)):
        errs = [np.linalg.norm(final_state(theta, t_end / k) - exact) for k in (50, 100, 200)]
        r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
        assert abs(r1 - order) < 0.35 * order and abs(r2 - order) < 0.35 * order, (theta, errs)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c1.npz")), reason="c1 golden absent")
def test_c1_full_config_matches_reference():
    """Config C1 (N=2000, 2000 steps): observables and current densities vs the
    reference run (Jacobi eigensolve + Td2Stepper / Td1Stepper)."""
    from paper_2407_11993_b200 import modal, reduction, transient
    from paper_2407_11993_b200.network import DriveSignal, Tone
    from paper_2407_11993_b200.synth import plate_model
    g = golden("c1")
    m = plate_model(40, 25, 2, n_ports=0, n_sources=1, n_obs=16)
    rm = reduction.from_blocks(m["r_i"], m["l_i"], None, None, m["m0"], source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    drive = DriveSignal(tones=(Tone(1.0, 1e4, 0.0),), sources=("s0",))
    for method in ("td2", "td1"):
        cfg = transient.TransientConfig(theta=0.5, dt=1e-6, t_end=2000e-6, method=method)
        res = transient.run_transient(rm, None, drive, cfg,
                                      modal=basis if method == "td2" else None,
                                      observables=(m["c"], None))
        assert rel_l2(res.observables, g[f"{method}_obs"]) < TOL
        assert rel_l2(res.internal_states[499::500], g[f"{method}_states"]) < TOL


def test_mode_sharded_stepping_on_device():
    """parallel.ShardedTd2: the per-rank device scans over disjoint mode ranges sum to
    the unsharded observables (ranks emulated in one process; the NCCL all-reduce is
    the only step not exercised here — it is covered by the gloo tests)."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal, transient
    from paper_2407_11993_b200.parallel import ShardedTd2, shard_ranges
    g = golden("plate_200")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    steps, dt = int(g["steps"]), float(g["dt"])
    i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), dt, steps)
    table = nat.device_vector(np.concatenate([i_d, i0], axis=1).reshape(-1))
    y = None
    for lo, hi in shard_ranges(rm.n_internal, 3):
        sh = ShardedTd2(rm, basis, dt, 0.5, g["c"], block=128, mode_range=(lo, hi))
        part = sh.run(table, steps).cpu().numpy()
        y = part if y is None else y + part
    assert rel_l2(y, g["td2_obs_theta0.5"]) < TOL


def test_exact_modal_integrator_on_device_matches_oracle():
    """exact_modal_reference (transient.py:315-360) on the device (the
    exponential integrator as the blocked scan) against the host restatement, over a
    ramp + tone drive, moderate dt/tau; with an initial state; non-uniform times rejected."""
    from paper_2407_11993_b200 import modal, reduction, transient
    from paper_2407_11993_b200.errors import ValidationError
    g = golden("plate_small")
    rm = reduction.from_blocks(g["r_i"] * 2e3, g["l_i"], g["r_d"] * 2e3, g["l_d"], g["m0"],
                               port_names=("p0",), source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    n_t, dt = 1501, 2e-7
    times = dt * np.arange(n_t)
    i_d = np.minimum(times / 5e-5, 1.0)[:, None]
    i0 = np.sin(2 * np.pi * 2e4 * times)[:, None]
    got = transient.exact_modal_reference(basis, rm, i_d, i0, times)
    ref = oracle.exact_modal_reference(basis, rm.r_d, rm.l_d, rm.m0, i_d, i0, times)
    assert got.shape == ref.shape == (n_t, basis.n_modes)
    assert rel_l2(got, ref) < 1e-9
    q0 = np.linspace(-1.0, 1.0, basis.n_modes) * 1e-3
    got0 = transient.exact_modal_reference(basis, rm, i_d, i0, times, modal_state0=q0)
    # linearity: the initial state decays independently of the drive
    decay = transient.exact_modal_reference(basis, rm, 0 * i_d, 0 * i0, times, modal_state0=q0)
    assert rel_l2(got0, got + decay) < 1e-12
    tau = basis.l_n / basis.r_n
    assert np.allclose(decay[-1], q0 * np.exp(-times[-1] / tau), rtol=1e-10, atol=1e-300)
    with pytest.raises(ValidationError):
        transient.exact_modal_reference(basis, rm, i_d[:3], i0[:3], np.array([0.0, 1e-7, 3e-7]))


@pytest.mark.parametrize("theta", [0.5, 1.0])
def test_excitation_sweep_matches_oracle_per_channel(theta):
    """Batched-excitation sweep (BASELINE configs[4], em_td2_run_sweep): each drive
    channel integrated alone as its own right-hand side. Every channel's observables
    (with the port's direct term D) against the oracle run with only that channel
    driven; the channels sum to the superposed trajectory of the UNMODIFIED reference
    (golden td2_obs, transient.py:147-155 superposes them); final per-channel states."""
    from paper_2407_11993_b200 import modal, reduction, transient
    g = golden("plate_small")
    rng = np.random.default_rng(7)
    n = g["r_i"].shape[0]
    m0 = np.concatenate([g["m0"], rng.standard_normal((n, 3)) / np.sqrt(n)], axis=1)
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], m0,
                               port_names=("p0",), source_names=("s0", "s1", "s2", "s3"))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    ref = oracle.generalized_eig(g["l_i"], g["r_i"])
    steps, dt = int(g["steps"]), float(g["dt"])
    t = dt * np.arange(steps + 1)
    i_d = np.minimum(t / 5e-6, 1.0)[:, None]
    f = np.array([1e4, 3e4, 7e4, 1.3e5])
    i0 = np.sin(2 * np.pi * f[None, :] * t[:, None] + np.arange(4)[None, :])
    c = g["c"]
    d = rng.standard_normal((c.shape[0], 1))
    st = transient.Td2Stepper(rm, basis, dt, theta)
    y, q = st.run_sweep(i_d, i0, observables=(c, d))
    assert y.shape == (5, steps, c.shape[0]) and q.shape == (n, 5)
    o = oracle.Td2(ref, rm.r_d, rm.l_d, rm.m0, dt, theta)
    for ch in range(5):
        i_d_c, i0_c = np.zeros_like(i_d), np.zeros_like(i0)
        if ch == 0:
            i_d_c[:] = i_d
        else:
            i0_c[:, ch - 1] = i0[:, ch - 1]
        states, _ = oracle.run(o, n, i_d_c, i0_c, ref)
        y_ref = states @ c.T + (i_d_c[1:] @ d.T if ch == 0 else 0.0)
        assert rel_l2(y[ch], y_ref) < TOL, ch
        # final state of the channel as currents I = V q (the oracle captures V q)
        assert rel_l2(basis.v @ q[:, ch], states[-1]) < TOL, ch
    # superposition of the first two channels = the reference's own superposed run
    rm1 = _plate_rm(g)
    st1 = transient.Td2Stepper(rm1, modal.generalized_eig(rm1.l_i, rm1.r_i), dt, theta)
    i_d1, i01 = transient.drive_samples(None, rm1, _plate_drives(), dt, steps)
    y1, _ = st1.run_sweep(i_d1, i01, observables=(c, None))
    assert rel_l2(y1.sum(axis=0), g[f"td2_obs_theta{theta}"]) < TOL


def test_mode_sharded_sweep_on_device():
    """parallel.ShardedTd2.run_sweep (C5: the sweep with modes sharded across GPUs): the
    per-rank sweeps over disjoint mode ranges, run block by block with the carried
    per-channel states, sum to the unsharded sweep (ranks emulated in one process)."""
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import modal, transient
    from paper_2407_11993_b200.parallel import ShardedTd2, shard_ranges
    g = golden("plate_200")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    steps, dt = int(g["steps"]), float(g["dt"])
    i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), dt, steps)
    table = nat.device_vector(np.concatenate([i_d, i0], axis=1).reshape(-1))
    ref, _ = transient.Td2Stepper(rm, basis, dt, 0.5).run_sweep(i_d, i0, observables=(g["c"], None))
    y = None
    for lo, hi in shard_ranges(rm.n_internal, 3):
        sh = ShardedTd2(rm, basis, dt, 0.5, g["c"], block=96, mode_range=(lo, hi))
        part = sh.run_sweep(table, steps).cpu().numpy()
        y = part if y is None else y + part
    assert y.shape == ref.shape
    assert rel_l2(y, ref) < 1e-12
    assert rel_l2(y.sum(axis=0), g["td2_obs_theta0.5"]) < TOL


@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_c2_full_size_td1_equals_td2(theta):
    """BASELINE configs[1] at its full size (N = 16,384 plate, electrode ramp, dt = 5e-7,
    32 observables), where no CPU oracle finishes: the two independent device paths —
    banded-R eigensolve + modal scan vs the Cholesky theta-method (dense factor of
    L + dt theta R, triangular solves) — must agree to the north-star 1e-8 relative L2
    over the first 500 steps, and every current density (captured states) too."""
    import ctypes
    import torch
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200.synth import device_plate_model, drive_table
    m = device_plate_model(64, 64, 4, n_ports=1, n_sources=0, n_obs=32)
    n = m["l_i"].shape[0]
    steps, dt = 500, 5e-7
    i_d, _ = drive_table("ramp5us", steps, dt, 1, 0)
    lib, ctx = nat.load_library(), nat.context()
    tau, ln, rn, V = nat.empty(n), nat.empty(n), nat.empty(n), nat.empty(n, n)
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    nat.check(lib.em_sygv_ex(ctx, n, nat.ptr(m["l_i"]), n, nat.ptr(m["r_i"]), n, nat.ptr(tau),
                             nat.ptr(V), n, nat.ptr(ln), nat.ptr(rn), None, n, 1,
                             ctypes.byref(piv), ctypes.byref(which)), "em_sygv_ex")
    drv = torch.cat([m["r_d"], m["l_d"]], dim=0).contiguous()      # (2, n): [R_D | L_D]
    P = nat.empty(2, n)
    nat.check(lib.em_dgemm(ctx, 1, 0, n, 2, n, 1.0, nat.ptr(V), n, nat.ptr(drv), n, 0.0,
                           nat.ptr(P), n))
    c_dev = nat.device_colmajor(m["c"])
    CV = nat.empty(n, 32)
    nat.check(lib.em_dgemm(ctx, 0, 0, 32, n, n, 1.0, nat.ptr(c_dev), 32, nat.ptr(V), n, 0.0,
                           nat.ptr(CV), 32))
    table = nat.device_vector(np.ascontiguousarray(i_d).reshape(-1))
    plan = ctypes.c_void_p()
    nat.check(lib.em_td2_plan_create(ctx, n, 1, 0, nat.ptr(ln), nat.ptr(rn), nat.ptr(P[0:1]),
                                     nat.ptr(P[1:2]), nat.ptr(P[0:1]), dt, theta,
                                     ctypes.byref(plan)))
    nat.check(lib.em_td2_set_observables(plan, 32, nat.ptr(CV), 32, None, 0))
    q = nat.zeros(n)
    y2 = nat.empty(steps, 32)
    qcap = nat.empty(steps, n)
    nat.check(lib.em_td2_run(plan, steps, nat.ptr(table), nat.ptr(q), nat.ptr(y2), 1,
                             nat.ptr(qcap)))
    lib.em_td2_plan_destroy(plan)
    icap2 = (qcap @ V).cpu().numpy()   # currents I = V q per step (V column-major)
    plan1 = ctypes.c_void_p()
    nat.check(lib.em_td1_plan_create(ctx, n, 1, 0, nat.ptr(m["l_i"]), n, nat.ptr(m["r_i"]), n,
                                     nat.ptr(m["r_d"]), nat.ptr(m["l_d"]), None, dt, theta,
                                     ctypes.byref(plan1), ctypes.byref(piv)))
    nat.check(lib.em_td1_set_observables(plan1, 32, nat.ptr(c_dev), 32, None, 0))
    cur = nat.zeros(n)
    y1 = nat.empty(steps, 32)
    icap1 = nat.empty(steps, n)
    nat.check(lib.em_td1_run(plan1, steps, nat.ptr(table), nat.ptr(cur), nat.ptr(y1), 1,
                             nat.ptr(icap1)))
    lib.em_td1_plan_destroy(plan1)
    assert rel_l2(y2.cpu().numpy(), y1.cpu().numpy()) < 1e-8
    assert rel_l2(icap2, icap1.cpu().numpy()) < 1e-8


def test_selective_mode_integration():
    """SURVEY 8(f)4 / PAPER.md:299 "(iv) in a selective manner": a subset of modes
    integrated alone. All modes = the full run (same arithmetic); a subset = the oracle's
    run restricted to those modes; the truncation error falls as slow modes are added."""
    from paper_2407_11993_b200 import modal, transient
    g = golden("plate_200")
    rm = _plate_rm(g)
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    dt, steps = float(g["dt"]), int(g["steps"])
    i_d, i0 = transient.drive_samples(None, rm, _plate_drives(), dt, steps)
    obs = (g["c"], None)
    full = transient.Td2Stepper(rm, basis, dt, 0.5)
    s_full, y_full, q_full = full.run(i_d, i0, observables=obs)
    every = transient.Td2Stepper(rm, basis, dt, 0.5, modes=np.ones(200, dtype=bool))
    _, y_all, _ = every.run(i_d, i0, capture_state=False, observables=obs)
    np.testing.assert_array_equal(y_all, y_full)
    sel = transient.select_modes(basis, count=40)
    assert np.array_equal(sel, np.arange(40))
    part = transient.Td2Stepper(rm, basis, dt, 0.5, modes=sel)
    s_sel, y_sel, q_sel = part.run(i_d, i0, observables=obs)
    # the truncated modal sum, by the oracle's loop over the same modes
    from oracle import oracle as O
    vt = basis.v.T
    tab = np.concatenate([i_d, i0], axis=1)
    _, y_ref = O.td2_run_table(basis.l_n[sel], basis.r_n[sel], (vt @ g["r_d"])[sel],
                               (vt @ g["l_d"])[sel], (vt @ g["m0"])[sel], dt, 0.5, tab, steps,
                               cv=(g["c"] @ basis.v)[:, sel])
    assert rel_l2(y_sel, y_ref) < 1e-12
    assert np.array_equal(q_sel[40:], np.zeros(160)) and rel_l2(q_sel[:40], q_full[:40]) < 1e-12
    # the last capture (replay pass) against the carried final state: two arithmetic paths
    assert rel_l2(s_sel[-1], basis.v[:, :40] @ q_sel[:40]) < 1e-8
    # linearity: a selection and its complement superpose to the full run
    rest = np.setdiff1d(np.arange(200), sel)
    _, y_rest, _ = transient.Td2Stepper(rm, basis, dt, 0.5, modes=rest).run(
        i_d, i0, capture_state=False, observables=obs)
    assert rel_l2(y_sel + y_rest, y_full) < 1e-12
    # by time constant, and the per-step API moves only the selected modes
    slow = transient.select_modes(basis, tau_min=float(basis.tau[9]))
    assert np.array_equal(slow, np.arange(10))
    st = transient.Td2Stepper(rm, basis, dt, 0.5, modes=slow)
    q = np.zeros(200)
    st.step(q, np.ones(1), np.ones(1), np.ones(1))
    assert np.any(q[:10]) and not np.any(q[10:])
