"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists); the resulting
.npz files are committed and are all the GPU box ever sees:

    python tests/golden/make_golden.py kat plate_small plate_200 tubes fd reduction observers  # seconds
    python tests/golden/make_golden.py c1                                # ~30 min (Jacobi at N=2000)
    python tests/golden/make_golden.py c2                                # ~10 min (dsygvd at N=16384)

The reference is copied to a writable temp dir first because its numba
kernels use cache=True and would write into the (read-only) source tree.
Inputs for the plates come from paper_2407_11993_b200.synth (seeded) and
are stored alongside the outputs so the fixtures pin both.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("EDDYMODES_REF", "/root/reference/pkg/src")
TMP = "/tmp/eddymodes_ref_copy"


def import_reference():
    if not os.path.isdir(os.path.join(TMP, "eddymodes")):
        shutil.copytree(os.path.join(REF_SRC, "eddymodes"), os.path.join(TMP, "eddymodes"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(TMP, "_numba_cache"))
    sys.path.insert(0, TMP)
    import eddymodes  # noqa: F401
    return eddymodes


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def save(name: str, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


def case_kat(em):
    from eddymodes.linalg import cholesky, sym_eig
    from eddymodes.errors import NotPositiveDefinite
    rng = np.random.default_rng(20240807)
    out = {}
    for n in (1, 2, 5, 17, 40):
        b = rng.standard_normal((n, n))
        a = b.T @ b + n * np.eye(n)
        out[f"chol_a_{n}"] = a
        out[f"chol_c_{n}"] = cholesky(a).c
    try:
        cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    except NotPositiveDefinite as exc:
        out["chol_indef_pivot"] = np.array(exc.pivot)
    for name, a in (("diag", np.diag([3.0, 1.0, 2.0])),
                    ("two", np.array([[2.0, 1.0], [1.0, 2.0]]))):
        lam, u = sym_eig(a)
        out[f"eig_a_{name}"], out[f"eig_lam_{name}"], out[f"eig_u_{name}"] = a, lam, u
    a = rng.standard_normal((12, 12))
    a = (a + a.T) / 2
    lam, u = sym_eig(a)
    out["eig_a_seeded"], out["eig_lam_seeded"], out["eig_u_seeded"] = a, lam, u
    save("kat_linalg", **out)


def _reduced(em, r, l, r_d, l_d, m0, port_names=(), source_names=()):
    from eddymodes.linalg import SymMatrix
    from eddymodes.reduction import ReducedModel
    n = r.shape[0]
    return ReducedModel(r_i=SymMatrix(r), l_i=SymMatrix(l), r_d=r_d, l_d=l_d, m0=m0,
                        lift=np.zeros((n, r_d.shape[1])), k=np.eye(n),
                        port_names=tuple(port_names), source_names=tuple(source_names))


def _run_pair(em, rm, basis, drives, theta, dt, steps, c_obs, keep_every):
    from eddymodes.transient import TransientConfig, run_transient
    res = {}
    for method in ("td2", "td1"):
        cfg = TransientConfig(theta=theta, dt=dt, t_end=steps * dt, method=method,
                              capture_stride=1, capture_state=True)
        t0 = time.perf_counter()
        sim = run_transient(rm, None, drives, cfg, modal=basis if method == "td2" else None)
        print(f"  {method} theta={theta}: {time.perf_counter() - t0:.2f}s")
        res[f"{method}_obs"] = sim.internal_states @ c_obs.T
        res[f"{method}_states"] = sim.internal_states[keep_every - 1::keep_every]
    return res


def case_plate(em, name, grid, n_ports, n_sources, n_obs, steps, dt, thetas, keep_every):
    from eddymodes.modal import generalized_eig
    from eddymodes.network import DriveSignal, Tone
    sys.path.insert(0, REPO)
    from paper_2407_11993_b200.synth import plate_model
    m = plate_model(*grid, n_ports=n_ports, n_sources=n_sources, n_obs=n_obs)
    ports = tuple(f"p{i}" for i in range(n_ports))
    sources = tuple(f"s{i}" for i in range(n_sources))
    rm = _reduced(em, m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"], ports, sources)
    t0 = time.perf_counter()
    basis = generalized_eig(rm.l_i, rm.r_i)
    t_eig = time.perf_counter() - t0
    print(f"{name}: N={rm.n_internal} eig {t_eig:.2f}s")
    drives = []
    if n_sources:
        drives.append(DriveSignal(tones=(Tone(1.0, 1e4, 0.0),), sources=sources))
    if n_ports:
        drives.append(DriveSignal(tones=(Tone(0.7, 2e4, 0.3), Tone(0.2, 5e4, 1.1)), ports=ports))
    out = dict(r_i=rm.r_i.full, l_i=rm.l_i.full, r_d=m["r_d"], l_d=m["l_d"], m0=m["m0"],
               c=m["c"], grid=np.array(grid), dt=np.array(dt), steps=np.array(steps),
               thetas=np.array(thetas), keep_every=np.array(keep_every),
               tau=basis.tau, l_n=basis.l_n, r_n=basis.r_n, v=basis.v,
               t_eig_ref=np.array(t_eig))
    for th in thetas:
        res = _run_pair(em, rm, basis, tuple(drives), th, dt, steps, m["c"], keep_every)
        for k, v in res.items():
            out[f"{k}_theta{th}"] = v
    save(name, **out)


def case_tubes(em):
    from eddymodes.assembly import (assemble_branch_matrices, build_current_basis,
                                    electrode_incidence)
    from eddymodes.modal import generalized_eig
    from eddymodes.network import DriveSignal, Tone, generate_tube_grid
    from eddymodes.reduction import project_model
    from eddymodes.transient import TransientConfig, run_transient
    for name, (na, nc) in (("tube_small", (4, 8)), ("tube_ref", (12, 24))):
        net = generate_tube_grid(84e-3, 0.3, 3e-3, na, nc, 1.09e-6)
        bm = assemble_branch_matrices(net)
        basis_c = build_current_basis(net)
        e = electrode_incidence(net, basis_c)
        port_names = tuple(el.name for el in net.electrodes[:-1])
        rm = project_model(bm, basis_c, e, port_names=port_names)
        mb = generalized_eig(rm.l_i, rm.r_i)
        out = dict(r_i=rm.r_i.full, l_i=rm.l_i.full, r_d=rm.r_d, l_d=rm.l_d, m0=rm.m0,
                   tau=mb.tau, l_n=mb.l_n, r_n=mb.r_n, v=mb.v, vt_r=mb.vt_r)
        drive = DriveSignal(tones=(Tone(1.0, 1e3, 0.0),), ports=port_names[:1])
        dt = 1 / 30000
        for method in ("td2", "td1"):
            cfg = TransientConfig(theta=1.0, dt=dt, t_end=200 * dt, method=method)
            sim = run_transient(rm, None, drive, cfg, modal=mb if method == "td2" else None)
            out[f"{method}_states"] = sim.internal_states
        out["dt"] = np.array(dt)
        out["n_ports"] = np.array(rm.n_ports)
        print(f"{name}: N={rm.n_internal} ports={rm.n_ports}")
        save(name, **out)


def case_c1(em):
    from eddymodes.modal import generalized_eig
    from eddymodes.network import DriveSignal, Tone
    sys.path.insert(0, REPO)
    from paper_2407_11993_b200.synth import plate_model
    m = plate_model(40, 25, 2, n_ports=0, n_sources=1, n_obs=16)
    rm = _reduced(em, m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"], (), ("s0",))
    t0 = time.perf_counter()
    basis = generalized_eig(rm.l_i, rm.r_i)
    t_eig = time.perf_counter() - t0
    print(f"C1 eig {t_eig:.1f}s")
    drive = DriveSignal(tones=(Tone(1.0, 1e4, 0.0),), sources=("s0",))
    res = _run_pair(em, rm, basis, (drive,), 0.5, 1e-6, 2000, m["c"], 500)
    save("c1", tau=basis.tau, l_n=basis.l_n, r_n=basis.r_n, v_lead=basis.v[:, :4].copy(),
         t_eig_ref=np.array(t_eig), input_sha_r=np.array(sha(rm.r_i.full)),
         input_sha_l=np.array(sha(rm.l_i.full)), input_sha_c=np.array(sha(m["c"])),
         input_sha_m0=np.array(sha(m["m0"])), **res)


def case_c2(em):
    """C2 (BASELINE configs[1]: N = 16,384, one port with a 5 us ramp, theta = 1 and 0.5,
    dt = 5e-7, 10,000 steps, 32 observables). The reference's Jacobi is infeasible at this
    N (~10 days), so the basis is the LAPACK dsygvd restatement of modal.py:46-81 (potrf +
    sygst + syevd + trsm, then the reference's descending order, sign fix and l_n / r_n,
    modal.py:74-80), which tests/test_oracle.py pins to the reference's Jacobi on every
    smaller fixture. The stepping is the UNMODIFIED reference Td2Stepper
    (transient.py:116-166 -> _kernels.td2_step_kernel) over that basis, driven by the
    ramp sample table (run_transient's drive convention, transient.py:293-299);
    observables y^k = (C V) q^k."""
    import scipy.linalg as sl
    from eddymodes.modal import ModalBasis
    from eddymodes.transient import Td2Stepper
    sys.path.insert(0, REPO)
    from paper_2407_11993_b200.synth import drive_table, plate_model
    m = plate_model(64, 64, 4, n_ports=1, n_sources=0, n_obs=32)
    rm = _reduced(em, m["r_i"], m["l_i"], m["r_d"], m["l_d"], m["m0"], ("p0",), ())
    lm, rmat = rm.l_i.full, rm.r_i.full
    n = lm.shape[0]
    t0 = time.perf_counter()
    w, v = sl.eigh(lm, rmat, driver="gvd", lower=True)
    order = np.argsort(-w, kind="stable")
    w, v = w[order], np.ascontiguousarray(v[:, order])
    idx = np.argmax(np.abs(v), axis=0)
    signs = np.sign(v[idx, np.arange(n)])
    signs[signs == 0] = 1.0
    v *= signs[None, :]
    l_n = np.einsum("ij,ij->j", v, lm @ v)
    r_n = np.einsum("ij,ij->j", v, rmat @ v)
    print(f"C2 dsygvd + l_n/r_n {time.perf_counter() - t0:.1f}s")
    basis = ModalBasis(v=v, tau=w, l_n=l_n, r_n=r_n, vt_r=np.zeros((0, 0)))
    steps, dt, keep = 10000, 5e-7, 5
    i_d, i0 = drive_table("ramp5us", steps, dt, 1, 0)
    cv = m["c"] @ v
    out = dict(tau=w, l_n=l_n, r_n=r_n, v_lead=v[:, :4].copy(), keep_every=np.array(keep),
               dt=np.array(dt), steps=np.array(steps), thetas=np.array([1.0, 0.5]),
               input_sha_r=np.array(sha(rmat)), input_sha_l=np.array(sha(lm)),
               input_sha_c=np.array(sha(m["c"])), input_sha_ld=np.array(sha(m["l_d"])),
               input_sha_rd=np.array(sha(m["r_d"])))
    for th in (1.0, 0.5):
        st = Td2Stepper(rm, basis, dt, th)
        q = np.zeros(n)
        y = np.empty((steps // keep, cv.shape[0]))
        t0 = time.perf_counter()
        for k in range(steps):
            st.step(q, i_d[k], i_d[k + 1] - i_d[k], i0[k + 1] - i0[k])
            if (k + 1) % keep == 0:
                y[(k + 1) // keep - 1] = cv @ q
        print(f"  td2 theta={th}: {time.perf_counter() - t0:.1f}s")
        out[f"td2_obs_theta{th}"] = y
        out[f"q_final_theta{th}"] = q.copy()
    save("c2", **out)


def case_reduction(em):
    """The reference's external-model reduction (reduction.py:60-99 integer kernel,
    21-57 lift, 143-183 project_external) on seeded integer incidence matrices: exact
    integer K (pinned bitwise) and the projected model."""
    from eddymodes.reduction import integer_kernel, lift_matrix, project_external
    rng = np.random.default_rng(20240807)
    out = {}
    for t in range(12):
        r = int(rng.integers(1, 5))
        c = int(rng.integers(r + 1, 30))
        e = rng.integers(-3, 4, size=(r, c))
        if t % 3 == 0:
            e[:, int(rng.integers(0, c))] = 0
        if t % 4 == 1 and r > 1:
            e[-1] = 2 * e[0] - e[1 % r]  # dependent row: a rank-deficient E
        out[f"ik_e_{t}"] = e
        out[f"ik_k_{t}"] = integer_kernel(e)
    n_x = 48
    a = rng.standard_normal((n_x, n_x))
    r_x = a @ a.T / n_x + np.eye(n_x)
    b = rng.standard_normal((n_x, n_x))
    l_x = b @ b.T / n_x + 0.5 * np.eye(n_x)
    e = np.zeros((2, n_x), dtype=np.int64)
    e[0, :5] = [1, -1, 2, 0, 1]
    e[1, 3:9] = [1, 1, 0, -2, 1, 1]
    rm = project_external(r_x, l_x, e, port_names=("a", "b"))
    out.update(px_r_x=r_x, px_l_x=l_x, px_e=e, px_r_i=rm.r_i.full, px_l_i=rm.l_i.full,
               px_r_d=rm.r_d, px_l_d=rm.l_d, px_lift=rm.lift, px_k=rm.k,
               lift_e=e, lift_m=lift_matrix(e))
    save("reduction", **out)


def case_observers(em):
    """Probe observers: the reference's field_transfer (assembly.py:350-386)
    on its own tube network, run_transient with probes (transient.py:266-273, 302-305,
    td2 and td1) and crack_signature (ndt.py:229-240)."""
    from eddymodes.assembly import (assemble_branch_matrices, build_current_basis,
                                    electrode_incidence, field_transfer)
    from eddymodes.errors import ProbeTooClose
    from eddymodes.frequency import PhasorSet
    from eddymodes.modal import generalized_eig
    from eddymodes.ndt import crack_signature
    from eddymodes.network import DriveSignal, Tone, generate_tube_grid
    from eddymodes.reduction import project_model
    from eddymodes.transient import TransientConfig, run_transient
    net = generate_tube_grid(84e-3, 0.3, 3e-3, 4, 8, 1.09e-6)
    bm = assemble_branch_matrices(net)
    basis_c = build_current_basis(net)
    e = electrode_incidence(net, basis_c)
    port_names = tuple(el.name for el in net.electrodes[:-1])
    rm = project_model(bm, basis_c, e, port_names=port_names)
    rng = np.random.default_rng(20240807)
    ang = rng.uniform(0, 2 * np.pi, 12)
    probes = np.stack([0.095 * np.cos(ang), 0.095 * np.sin(ang), rng.uniform(0.0, 0.3, 12)], 1)
    out = dict(starts=net.branch_starts, ends=net.branch_ends, wire_radius=net.wire_radius,
               probes=probes, transfer=field_transfer(net, probes), w=basis_c.w, k=rm.k,
               lift=rm.lift, r_i=rm.r_i.full, l_i=rm.l_i.full, r_d=rm.r_d, l_d=rm.l_d,
               m0=rm.m0, n_ports=np.array(rm.n_ports))
    # a probe on a branch: ProbeTooClose names the first (probe, branch) pair
    bad = np.concatenate([probes[:3], 0.5 * (net.branch_starts[5:6] + net.branch_ends[5:6]),
                          probes[3:4]])
    try:
        field_transfer(net, bad)
        raise SystemExit("expected ProbeTooClose")
    except ProbeTooClose as exc:
        out["bad_probes"] = bad
        out["bad_msg"] = np.array(str(exc))
    mb = generalized_eig(rm.l_i, rm.r_i)
    drive = DriveSignal(tones=(Tone(1.0, 1e3, 0.0),), ports=port_names[:1])
    dt = 1 / 30000
    for method in ("td2", "td1"):
        cfg = TransientConfig(theta=1.0, dt=dt, t_end=60 * dt, method=method, capture_stride=3,
                              probes=probes)
        sim = run_transient(rm, net, drive, cfg, modal=mb if method == "td2" else None)
        out[f"{method}_fields"] = sim.probe_fields
    out["dt"] = np.array(dt)
    angles = tuple(float(a) for a in np.linspace(0, 2 * np.pi, 6, endpoint=False))
    freqs = (1e3, 5e3, 2e4)
    pd, pb = PhasorSet(probe_angles=angles), PhasorSet(probe_angles=angles)
    for pi in range(6):
        for f in freqs:
            pd[(pi, f)] = complex(rng.standard_normal(), rng.standard_normal())
            pb[(pi, f)] = complex(rng.standard_normal(), rng.standard_normal())
    sig = crack_signature(pd, pb)
    nrm = sig.normalized()
    keys = sorted(sig.entries)
    out.update(cs_angles=np.array(angles), cs_freqs=np.array(freqs),
               cs_defect=np.array([[pd[(p, f)] for f in freqs] for p in range(6)]),
               cs_background=np.array([[pb[(p, f)] for f in freqs] for p in range(6)]),
               cs_keys=np.array(keys), cs_sig=np.array([sig.entries[k] for k in keys]),
               cs_norm=np.array([nrm.entries[k] for k in keys]),
               cs_mag=np.array([sig.magnitude_by_angle(f) for f in freqs]))
    save("observers", **out)


def case_fd(em):
    """Frequency domain: the reference solve_tone on the plate_small
    and tube_small models at several tones, dft_phasor / extract_phasors KATs."""
    from eddymodes.frequency import dft_phasor, extract_phasors, solve_tone
    from eddymodes.errors import NonintegerPeriods, NyquistViolation
    out = {}
    for name in ("plate_small", "tube_small"):
        g = np.load(os.path.join(HERE, f"{name}.npz"))
        n_p = g["r_d"].shape[1]
        n_s = g["m0"].shape[1]
        rm = _reduced(em, g["r_i"], g["l_i"], g["r_d"], g["l_d"], g["m0"],
                      tuple(f"p{i}" for i in range(n_p)), tuple(f"s{i}" for i in range(n_s)))
        i_d = (np.arange(n_p) + 1.0) * (1.0 + 0.5j)
        i0 = (np.arange(n_s) + 1.0) * (0.3 - 0.2j)
        omegas = np.array([0.0, 2e3, 2 * np.pi * 5e4, 3e6])
        out[f"{name}_omegas"] = omegas
        out[f"{name}_i_d"] = i_d
        out[f"{name}_i0"] = i0
        for k, w in enumerate(omegas):
            out[f"{name}_I_{k}"] = solve_tone(rm, float(w), i_d, i0)
    dt, n = 1e-6, 2000
    t = dt * np.arange(n)
    x = (0.7 * np.sin(2 * np.pi * 1e4 * t + 0.3) + 0.2 * np.cos(2 * np.pi * 2.5e4 * t)
         + 0.05 * np.sin(2 * np.pi * 1e5 * t - 1.0))
    out["dft_x"] = x
    out["dft_dt"] = np.array(dt)
    out["dft_freqs"] = np.array([1e4, 2.5e4, 1e5, 5e4])
    out["dft_phasors"] = np.array([dft_phasor(x, dt, f) for f in out["dft_freqs"]])
    out["dft_phasor_t0"] = np.array(dft_phasor(x[500:1500], dt, 1e4, t0=500 * dt))
    rec = np.stack([x, 2 * x[::-1], np.cos(2 * np.pi * 1e4 * t)], axis=1)
    ps = extract_phasors(t, rec, [1e4, 5e4], [0.0, 1.0, 2.0], window=(2e-4, 1.2e-3))
    out["ext_rec"] = rec
    out["ext_keys"] = np.array([[p, f] for (p, f) in sorted(ps.entries)])
    out["ext_vals"] = np.array([ps.entries[k] for k in sorted(ps.entries)])
    for bad, exc in (((x, dt, 6e5), NyquistViolation), ((x[:1999], dt, 1e4), NonintegerPeriods)):
        try:
            dft_phasor(*bad)
            raise SystemExit("expected an error")
        except exc:
            pass
    save("fd", **out)


def case_cache(em):
    """The reference's text cache (E/matrixio.py) for the tube_small model, with an
    integer E and a current basis (the reference's own tube network)."""
    from eddymodes.assembly import (assemble_branch_matrices, build_current_basis,
                                    electrode_incidence)
    from eddymodes.matrixio import write_cache
    from eddymodes.network import generate_tube_grid
    from eddymodes.reduction import project_model
    net = generate_tube_grid(84e-3, 0.3, 3e-3, 3, 5, 1.09e-6)
    bm = assemble_branch_matrices(net)
    basis_c = build_current_basis(net)
    e = electrode_incidence(net, basis_c)
    port_names = tuple(el.name for el in net.electrodes[:-1])
    rm = project_model(bm, basis_c, e, port_names=port_names)
    path = os.path.join(HERE, "cache_tube.txt")
    write_cache(path, rm, None, e=e.e, header_lines=("golden: reference write_cache",))
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB) N={rm.n_internal}")


def main(argv):
    em = import_reference()
    for case in argv or ["kat", "plate_small", "plate_200", "tubes"]:
        if case == "kat":
            case_kat(em)
        elif case == "plate_small":
            case_plate(em, "plate_small", (6, 8, 2), 1, 1, 8, 300, 1e-6, (0.5, 1.0), 10)
        elif case == "plate_200":
            case_plate(em, "plate_200", (10, 10, 2), 1, 1, 16, 1000, 1e-6, (0.5,), 100)
        elif case == "tubes":
            case_tubes(em)
        elif case == "c1":
            case_c1(em)
        elif case == "c2":
            case_c2(em)
        elif case == "reduction":
            case_reduction(em)
        elif case == "observers":
            case_observers(em)
        elif case == "fd":
            case_fd(em)
        elif case == "cache":
            case_cache(em)
        else:
            raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1:])
