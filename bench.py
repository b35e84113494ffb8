#!/usr/bin/env python
"""Headline benchmark: end-to-end modal transient (generalized eigensolve +
theta-method stepping) in mode-steps/s — BASELINE.json `metric` on configs[1]
(C2: N = 16,384 plate 64x64x4, one electrode port with a 5 us current ramp,
theta = 1 and 0.5, dt = 5e-7 s, 10,000 steps, 32 observables, FP64).

One benchmark STEP = one pass of the hot path over the workload:
  generalized eigensolve (em_sygv: tau, V, l_n, r_n, V^T R)
  + for each theta: drive projection, TD2 plan, 10k-step fused scan with the
    32 observables reconstructed every step.
mode-steps per step = N * T * n_theta.

value: inputs (L, R, drive table, C) resident in HBM, outputs left on device.
e2e:   the same through the public Python API with HOST buffers (pinned), H2D of
       L, R, couplings, drive table and C and D2H of every observable inside the
       timed region.

python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C1|C2]
Multi-GPU (torchrun): the path does not shard in this round -> independent
replicas, one per GPU (scaling "weak"), value = sum of all ranks' mode-steps / max time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(grid=(40, 25, 2), thetas=(0.5,), dt=1e-6, steps=2000, n_obs=16, n_ports=0,
               n_sources=1, drive="tone10k"),
    "C2": dict(grid=(64, 64, 4), thetas=(1.0, 0.5), dt=5e-7, steps=10000, n_obs=32, n_ports=1,
               n_sources=0, drive="ramp5us"),
    # configs[2]: N = 50,000 (L = 20 GB): 7 N^2 at the eigensolve peak on one B200, so the
    # basis is formed without V^T R (not used by the transient; ModalBasis defers it)
    "C3": dict(grid=(125, 100, 4), thetas=(0.5,), dt=2e-7, steps=100000, n_obs=64, n_ports=1,
               n_sources=1, drive="tone50k", vtr=False),
    # configs[4]: N = 60,000, 64 independent source waveforms as 64 right-hand sides
    # (the excitation sweep, em_td2_run_sweep); eigensolve at 6 N^2 (R as its own factor
    # workspace, no V^T R) on one B200
    "C5": dict(grid=(150, 100, 4), thetas=(0.5,), dt=2e-7, steps=100000, n_obs=64, n_ports=0,
               n_sources=64, drive="batched", vtr=False, sweep=True),
    # configs[3]: the north-star Target plate, N = 120,000 minus a seeded 2 mm notch
    # (L = 115 GB). On one B200 only as the implicit-V solve (L reduced in place, R in band
    # storage) and the in-place Cholesky comparator: run_c4
    "C4": dict(grid=(200, 150, 4), thetas=(0.5,), dt=1e-7, steps=100000, n_obs=128, n_ports=1,
               n_sources=0, drive="trapezoid", notch=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if r[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- workload
def build_inputs(cfg):
    from paper_2407_11993_b200 import synth
    from paper_2407_11993_b200 import _native as nat
    nx, ny, nz = cfg["grid"]
    m = synth.device_plate_model(nx, ny, nz, n_ports=cfg["n_ports"], n_sources=cfg["n_sources"],
                                 n_obs=cfg["n_obs"])
    i_d, i0 = synth.drive_table(cfg["drive"], cfg["steps"], cfg["dt"], cfg["n_ports"],
                                cfg["n_sources"], plate=m["plate"])
    table = np.ascontiguousarray(np.concatenate([i_d, i0], axis=1))
    m["i_d"], m["i0"], m["table"] = i_d, i0, table
    m["table_dev"] = nat.device_vector(table.reshape(-1)) if table.size else nat.zeros(1)
    m["c_dev"] = nat.device_colmajor(m["c"])
    n = m["plate"].n
    m["m0_dev"] = nat.device_colmajor(m["m0"]) if cfg["n_sources"] else None
    return m


class DeviceStep:
    """The hot path on device-resident inputs, straight through the C ABI."""

    def __init__(self, m, cfg, form_v=True):
        from paper_2407_11993_b200 import _native as nat
        self.nat = nat
        self.m = m
        self.cfg = cfg
        n = m["plate"].n
        self.n = n
        n_p, n_s = cfg["n_ports"], cfg["n_sources"]
        self.n_p, self.n_s = n_p, n_s
        self.nd = 2 * n_p + n_s
        self.tau, self.ln, self.rn = nat.empty(n), nat.empty(n), nat.empty(n)
        self.V = nat.empty(n, n) if form_v else None
        self.VtR = nat.empty(n, n) if form_v and cfg.get("vtr", True) else None
        cols = []
        if n_p:
            cols += [m["r_d"], m["l_d"]]
        if n_s:
            cols += [m["m0_dev"]]
        t = nat.torch()
        self.drv = t.cat(cols, dim=0).contiguous() if cols else nat.zeros(1, n)
        self.P = nat.empty(max(self.nd, 1), n) if form_v else None
        self.CV = nat.empty(n, cfg["n_obs"]) if form_v else None
        self.n_rhs = (n_p + n_s) if cfg.get("sweep") else 1
        self.Y = [nat.empty(self.n_rhs, cfg["steps"], cfg["n_obs"]) for _ in cfg["thetas"]]
        self.q = nat.empty(self.n_rhs, n)

    def __call__(self):
        import ctypes
        nat, lib, ctx = self.nat, self.nat.load_library(), self.nat.context()
        n, cfg = self.n, self.cfg
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        # R (stencil) doubles as the factor workspace and is restored from its CSR copy
        nat.check(lib.em_sygv_ex(ctx, n, nat.ptr(self.m["l_i"]), n, nat.ptr(self.m["r_i"]), n,
                                 nat.ptr(self.tau), nat.ptr(self.V), n, nat.ptr(self.ln),
                                 nat.ptr(self.rn),
                                 nat.ptr(self.VtR) if self.VtR is not None else None, n, 1,
                                 ctypes.byref(piv), ctypes.byref(which)), "em_sygv_ex")
        if self.nd:
            nat.check(lib.em_dgemm(ctx, 1, 0, n, self.nd, n, 1.0, nat.ptr(self.V), n,
                                   nat.ptr(self.drv), n, 0.0, nat.ptr(self.P), n), "em_dgemm")
        n_obs = cfg["n_obs"]
        nat.check(lib.em_dgemm(ctx, 0, 0, n_obs, n, n, 1.0, nat.ptr(self.m["c_dev"]), n_obs,
                               nat.ptr(self.V), n, 0.0, nat.ptr(self.CV), n_obs), "em_dgemm")
        n_p, n_s = self.n_p, self.n_s
        p_r = self.P[0:1] if not n_p else self.P[0:n_p]
        p_l = self.P[0:1] if not n_p else self.P[n_p:2 * n_p]
        p_m = self.P[0:1] if not n_s else self.P[2 * n_p:]
        for k, th in enumerate(cfg["thetas"]):
            plan = ctypes.c_void_p()
            nat.check(lib.em_td2_plan_create(ctx, n, n_p, n_s, nat.ptr(self.ln), nat.ptr(self.rn),
                                             nat.ptr(p_r), nat.ptr(p_l), nat.ptr(p_m), cfg["dt"],
                                             th, ctypes.byref(plan)), "em_td2_plan_create")
            nat.check(lib.em_td2_set_observables(plan, n_obs, nat.ptr(self.CV), n_obs, None, 0),
                      "em_td2_set_observables")
            self.q.zero_()
            if cfg.get("sweep"):
                nat.check(lib.em_td2_run_sweep(plan, cfg["steps"], nat.ptr(self.m["table_dev"]),
                                               nat.ptr(self.q), nat.ptr(self.Y[k]), 1),
                          "em_td2_run_sweep")
            else:
                nat.check(lib.em_td2_run(plan, cfg["steps"], nat.ptr(self.m["table_dev"]),
                                         nat.ptr(self.q), nat.ptr(self.Y[k]), 1, None),
                          "em_td2_run")
            lib.em_td2_plan_destroy(plan)


class ImplicitDeviceStep(DeviceStep):
    """The same step without forming V (em_sygv_implicit, SURVEY.md §7 "implicit V"):
    V^T is applied to the drive columns and the observable rows only, the scan runs on
    l_n = tau, r_n = 1. Reported beside the headline (which forms V like the reference)."""

    def __init__(self, m, cfg):
        super().__init__(m, cfg, form_v=False)
        t = self.nat.torch()
        n_obs = cfg["n_obs"]
        # C^T as n_obs columns: c_dev is C column-major (n_obs x n) -> transpose
        ct = self.m["c_dev"].reshape(self.n, n_obs).t().contiguous()
        self.y0 = t.cat([self.drv[:self.nd], ct], dim=0).contiguous()
        self.Yp = t.empty_like(self.y0)
        self.one = t.ones(self.n, dtype=t.float64, device="cuda")

    def __call__(self):
        import ctypes
        nat, lib, ctx = self.nat, self.nat.load_library(), self.nat.context()
        n, cfg, nd = self.n, self.cfg, self.nd
        n_obs = cfg["n_obs"]
        self.Yp.copy_(self.y0)
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        nat.check(lib.em_sygv_implicit(ctx, n, nat.ptr(self.m["l_i"]), n, nat.ptr(self.m["r_i"]),
                                       n, nat.ptr(self.tau), nat.ptr(self.Yp), n, nd + n_obs,
                                       None, None, 1, ctypes.byref(piv), ctypes.byref(which)),
                  "em_sygv_implicit")
        cv = self.Yp[nd:].t().contiguous()
        n_p, n_s = self.n_p, self.n_s
        P = self.Yp
        p_r = P[0:1] if not n_p else P[0:n_p]
        p_l = P[0:1] if not n_p else P[n_p:2 * n_p]
        p_m = P[0:1] if not n_s else P[2 * n_p:nd]
        for k, th in enumerate(cfg["thetas"]):
            plan = ctypes.c_void_p()
            nat.check(lib.em_td2_plan_create(ctx, n, n_p, n_s, nat.ptr(self.tau), nat.ptr(self.one),
                                             nat.ptr(p_r), nat.ptr(p_l), nat.ptr(p_m), cfg["dt"],
                                             th, ctypes.byref(plan)), "em_td2_plan_create")
            nat.check(lib.em_td2_set_observables(plan, n_obs, nat.ptr(cv), n_obs, None, 0),
                      "em_td2_set_observables")
            self.q.zero_()
            if cfg.get("sweep"):
                nat.check(lib.em_td2_run_sweep(plan, cfg["steps"], nat.ptr(self.m["table_dev"]),
                                               nat.ptr(self.q), nat.ptr(self.Y[k]), 1),
                          "em_td2_run_sweep")
            else:
                nat.check(lib.em_td2_run(plan, cfg["steps"], nat.ptr(self.m["table_dev"]),
                                         nat.ptr(self.q), nat.ptr(self.Y[k]), 1, None),
                          "em_td2_run")
            lib.em_td2_plan_destroy(plan)


class ShardedDeviceStep:
    """N > 1: this rank's share of the hot path on device-resident inputs. The eigensolve
    is column-sharded (em_sygv_range: every rank reduces the pencil to tridiagonal form,
    then back-transforms only its own modes' eigenvectors), the stepping integrates only
    those modes and the partial observables are all-reduced (NCCL) once per time block of
    `block` steps on a side stream, overlapped with the next block's scan."""

    def __init__(self, m, cfg, dist, rank, world, block=2048):
        from paper_2407_11993_b200 import _native as nat
        from paper_2407_11993_b200.parallel import shard_ranges
        t = nat.torch()
        self.nat, self.m, self.cfg, self.dist = nat, m, cfg, dist
        n = m["plate"].n
        self.n = n
        self.lo, self.hi = shard_ranges(n, world)[rank]
        ml = self.hi - self.lo
        self.ml = ml
        n_p, n_s = cfg["n_ports"], cfg["n_sources"]
        self.n_p, self.n_s, self.nd = n_p, n_s, 2 * n_p + n_s
        self.block = block
        self.tau = nat.empty(n)
        self.ln, self.rn = nat.empty(max(ml, 1)), nat.empty(max(ml, 1))
        self.V = nat.empty(max(ml, 1), n)
        cols = []
        if n_p:
            cols += [m["r_d"], m["l_d"]]
        if n_s:
            cols += [m["m0_dev"]]
        self.drv = t.cat(cols, dim=0).contiguous() if cols else nat.zeros(1, n)
        self.P = nat.empty(max(self.nd, 1), max(ml, 1))
        self.CV = nat.empty(max(ml, 1), cfg["n_obs"])
        self.sweep = bool(cfg.get("sweep"))
        self.n_rhs = (n_p + n_s) if self.sweep else 1
        self.Y = [nat.empty(self.n_rhs, cfg["steps"], cfg["n_obs"]) for _ in cfg["thetas"]]
        self.q = nat.empty(self.n_rhs, max(ml, 1))
        self.comm = t.cuda.Stream()

    def __call__(self):
        import ctypes
        nat, lib, ctx = self.nat, self.nat.load_library(), self.nat.context()
        t = nat.torch()
        n, ml, cfg = self.n, self.ml, self.cfg
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        nat.check(lib.em_sygv_range(ctx, n, nat.ptr(self.m["l_i"]), n, nat.ptr(self.m["r_i"]), n,
                                    self.lo, self.hi, nat.ptr(self.tau), nat.ptr(self.V), n,
                                    nat.ptr(self.ln), nat.ptr(self.rn), None, n, 1,
                                    ctypes.byref(piv), ctypes.byref(which)), "em_sygv_range")
        n_obs = cfg["n_obs"]
        if self.nd:
            nat.check(lib.em_dgemm(ctx, 1, 0, ml, self.nd, n, 1.0, nat.ptr(self.V), n,
                                   nat.ptr(self.drv), n, 0.0, nat.ptr(self.P), ml), "em_dgemm")
        nat.check(lib.em_dgemm(ctx, 0, 0, n_obs, ml, n, 1.0, nat.ptr(self.m["c_dev"]), n_obs,
                               nat.ptr(self.V), n, 0.0, nat.ptr(self.CV), n_obs), "em_dgemm")
        n_p, n_s = self.n_p, self.n_s
        p_r = self.P[0:1] if not n_p else self.P[0:n_p]
        p_l = self.P[0:1] if not n_p else self.P[n_p:2 * n_p]
        p_m = self.P[0:1] if not n_s else self.P[2 * n_p:]
        n_c = n_p + n_s
        T = cfg["steps"]
        main = t.cuda.current_stream()
        for k, th in enumerate(cfg["thetas"]):
            plan = ctypes.c_void_p()
            nat.check(lib.em_td2_plan_create(ctx, ml, n_p, n_s, nat.ptr(self.ln), nat.ptr(self.rn),
                                             nat.ptr(p_r), nat.ptr(p_l), nat.ptr(p_m), cfg["dt"],
                                             th, ctypes.byref(plan)), "em_td2_plan_create")
            nat.check(lib.em_td2_set_observables(plan, n_obs, nat.ptr(self.CV), n_obs, None, 0),
                      "em_td2_set_observables")
            self.q.zero_()
            pending = []
            for k0 in range(0, T, self.block):
                k1 = min(T, k0 + self.block)
                yb = self.Y[k][:, k0:k1] if not self.sweep else t.empty(
                    self.n_rhs, k1 - k0, n_obs, dtype=t.float64, device="cuda")
                drive = self.m["table_dev"][k0 * n_c:]
                if self.sweep:
                    nat.check(lib.em_td2_run_sweep(plan, k1 - k0, nat.ptr(drive),
                                                   nat.ptr(self.q), nat.ptr(yb), 1),
                              "em_td2_run_sweep")
                else:
                    yb = self.Y[k][0, k0:k1]
                    nat.check(lib.em_td2_run(plan, k1 - k0, nat.ptr(drive), nat.ptr(self.q),
                                             nat.ptr(yb), 1, None), "em_td2_run")
                ev = t.cuda.Event()
                ev.record(main)
                with t.cuda.stream(self.comm):
                    self.comm.wait_event(ev)
                    pending.append((self.dist.all_reduce(yb, async_op=True), yb, k0, k1))
            for h, yb, k0, k1 in pending:
                h.wait()
            main.wait_stream(self.comm)
            if self.sweep:
                for _, yb, k0, k1 in pending:
                    self.Y[k][:, k0:k1] = yb
            lib.em_td2_plan_destroy(plan)


class E2EStep:
    """The same work through the public API (reference call shapes) with host buffers."""

    def __init__(self, m, cfg):
        from paper_2407_11993_b200 import _native as nat
        from paper_2407_11993_b200 import linalg, reduction
        t = nat.torch()
        n = m["plate"].n
        self.cfg = cfg
        # host copies of the inputs in pinned memory, wrapped as the reference's types
        self.pinned = []

        def pinned_sym(dev):
            h = t.empty(dev.shape, dtype=t.float64, pin_memory=True)
            h.copy_(dev)
            self.pinned.append(h)
            s = linalg.SymMatrix(np.zeros((1, 1)))
            object.__setattr__(s, "a", h.numpy())      # exactly symmetric already
            return s

        l_i, r_i = pinned_sym(m["l_i"]), pinned_sym(m["r_i"])
        r_d = m["r_d"].cpu().numpy().T.copy() if cfg["n_ports"] else None
        l_d = m["l_d"].cpu().numpy().T.copy() if cfg["n_ports"] else None
        self.rm = reduction.ReducedModel(
            r_i=r_i, l_i=l_i,
            r_d=r_d if r_d is not None else np.zeros((n, 0)),
            l_d=l_d if l_d is not None else np.zeros((n, 0)),
            m0=m["m0"], lift=np.zeros((n, cfg["n_ports"])), k=_LazyEye(n),
            port_names=tuple(f"p{i}" for i in range(cfg["n_ports"])),
            source_names=tuple(f"s{i}" for i in range(cfg["n_sources"])))
        self.i_d, self.i0, self.c = m["i_d"], m["i0"], m["c"]
        n_obs = cfg["n_obs"]
        self.h2d = 8 * (2 * n * n + n * (2 * cfg["n_ports"] + cfg["n_sources"]) +
                        len(cfg["thetas"]) * (self.i_d.size + self.i0.size + n_obs * n))
        n_rhs = (cfg["n_ports"] + cfg["n_sources"]) if cfg.get("sweep") else 1
        self.d2h = 8 * (3 * n + len(cfg["thetas"]) * cfg["steps"] * n_obs * n_rhs)
        self.out = None

    def __call__(self):
        from paper_2407_11993_b200 import modal, transient
        cfg = self.cfg
        basis = modal.generalized_eig(self.rm.l_i, self.rm.r_i)
        ys = []
        for th in cfg["thetas"]:
            st = transient.Td2Stepper(self.rm, basis, cfg["dt"], th)
            if cfg.get("sweep"):
                y, _ = st.run_sweep(self.i_d, self.i0, observables=(self.c, None))
            else:
                _, y, _ = st.run(self.i_d, self.i0, capture_state=False,
                                 observables=(self.c, None))
            ys.append(y)
            del st
        self.out = (basis.tau, ys)


class E2EShardedStep(E2EStep):
    """N > 1 e2e: the public multi-GPU API (parallel.sharded_generalized_eig +
    ShardedTd2.run / run_sweep) on host (pinned) inputs, one rank's share."""

    def __init__(self, m, cfg, dist):
        super().__init__(m, cfg)
        self.dist = dist

    def __call__(self):
        from paper_2407_11993_b200 import _native as nat
        from paper_2407_11993_b200 import parallel, transient
        cfg = self.cfg
        sb = parallel.sharded_generalized_eig(self.rm.l_i, self.rm.r_i, self.dist)
        table = transient._drive_table(self.i_d, self.i0, cfg["n_ports"], cfg["n_sources"])
        drive = nat.device_vector(table.reshape(-1))
        ys = []
        for th in cfg["thetas"]:
            st = parallel.ShardedTd2(self.rm, sb, cfg["dt"], th, self.c, dist=self.dist)
            y = st.run_sweep(drive, cfg["steps"]) if cfg.get("sweep") else \
                st.run(drive, cfg["steps"])
            ys.append(y.cpu().numpy())
            del st
        self.out = (sb.tau, ys)


class _LazyEye:
    """K = I selector stand-in: only .shape is used on this path (n_internal)."""

    def __init__(self, n):
        self.shape = (n, n)


# --------------------------------------------------------------------------- roofline
# algorithmic FP64 flop counts of the eigensolve stages at order n; the
# two-stage pieces: sy2sb 4/3 n^3 (two-sided update), Q2 and Q1 back-transforms 2 n^3 each
# (applying ~n^2/2 reflector entries to n columns, 4 flop per entry and column)
def stage_flops(name, n, k=None):
    """k: implicit V (the back-transforms act on k skinny columns, not n)."""
    m = n if k is None else k
    return {"potrf_R": n ** 3 / 3, "potrf_L": n ** 3 / 3, "sygst": 2.0 * n ** 3,
            "ormtr": 2.0 * n * n * m, "trsm_back": 1.0 * n * n * m, "sy2sb": 4.0 / 3.0 * n ** 3,
            "q2_apply": 2.0 * n * n * m, "q1_apply": 2.0 * n * n * m}.get(name)


def roofline(stages: dict, n: int, peaks: dict, k=None) -> dict:
    """The dominant eigensolve stage (by time, per step) against the FP64 tensor peak, or
    the one-stage sytrd against HBM."""
    fp64 = peaks.get("fp64_tflops", 37.1)
    hbm = peaks.get("hbm_gbs", 6550.4)
    cands = {k: v for k, v in stages.items()
             if stage_flops(k, n) is not None or k == "sytrd"}
    if k is not None:  # implicit V on a banded R: sygst is 6 n^2 b, not a dense product
        cands.pop("sygst", None)
    if "q2_apply" in stages:  # two-stage: sytrd / ormtr are the sums of their pieces
        cands.pop("sytrd", None)
        cands.pop("ormtr", None)
    if not cands:
        return None
    name, (ms, cnt) = max(cands.items(), key=lambda kv: kv[1][0])
    if name == "sytrd":
        # lower-triangle symv over the trailing matrix per column: 8 * sum m^2/2 bytes
        byts = 8.0 * sum((n - c - 1) ** 2 / 2.0 for c in range(n))
        ach = byts / (ms * 1e-3) / 1e9
        return dict(stage=name, bound="hbm", achieved=ach, peak=hbm, unit="GB/s",
                    frac=ach / hbm, traffic=None, ms_per_step=ms, launches_per_step=cnt)
    ach = stage_flops(name, n, k) / (ms * 1e-3) / 1e12
    return dict(stage=name, bound="tensor", achieved=ach, peak=fp64, unit="TFLOP/s",
                frac=ach / fp64, traffic=None, ms_per_step=ms, launches_per_step=cnt,
                algorithmic_flop=stage_flops(name, n, k))


def symv_roofline(m, n, peaks, reps=20):
    """Roofline of the dominant kernel: the lower-triangle symv over the trailing matrix
    (one per tridiagonalisation column, the HBM-bound part of the sytrd stage), timed
    live with CUDA events on the launching stream at the full size n: algorithmic bytes
    8 n (n+1)/2 per launch (tile kernel + its partial-sum reduction)."""
    import torch
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    a = m["l_i"]
    x = torch.randn(n, device="cuda", dtype=torch.float64)
    y = torch.empty_like(x)
    call = lambda: nat.check(lib.em_symv_lower(ctx, n, 1.0, nat.ptr(a), n, nat.ptr(x), 0.0,
                                               nat.ptr(y)), "em_symv_lower")
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    byts = 8.0 * n * (n + 1) / 2
    hbm = peaks.get("hbm_gbs", 6550.4)
    ach = byts / t / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r01_ncu_symv_tma.json")
    if os.path.exists(prof) and n == 16384:
        p = json.load(open(prof))
        traffic = p["dram__bytes_read_GB"] * 1e9 + p["dram__bytes_write_MB"] * 1e6
    return dict(kernel="symv_tma_kernel + symv_tma_reduce_kernel (em_symv_lower)", bound="hbm",
                achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm, traffic=traffic,
                algorithmic_bytes=byts, per_launch_ms=t * 1e3, launches_timed=reps,
                peak_source="MEASURED_PEAKS.json hbm_gbs (copy, measured)",
                traffic_source="profiles/r01_ncu_symv_tma.json (ncu --set full, one launch)")


def load_peaks():
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peaks.update(json.load(open(p)))
    # FP64 DMMA issue peak measured on this pool's B200 (profiles/r01_fp64_peaks.jsonl)
    peaks.setdefault("fp64_tflops", 37.1)
    return peaks


# --------------------------------------------------------------------------- arms
def workload_config(args, cfg, n, world):
    """The `config` object of the JSON line (identical for both arms)."""
    T = cfg["steps"]
    n_rhs = (cfg["n_ports"] + cfg["n_sources"]) if cfg.get("sweep") else 1
    return {"workload": f"{args.config}: N={n} plate {cfg['grid']}, eigensolve + "
                        f"{T} TD2 steps x theta {list(cfg['thetas'])}"
                        + (f" x {n_rhs} right-hand sides (excitation sweep)" if n_rhs > 1 else "")
                        + f", {cfg['n_obs']} observables",
            "n_rhs": n_rhs, "N": n, "T": T, "thetas": list(cfg["thetas"]),
            "n_obs": cfg["n_obs"], "mode_steps_per_step": n * T * len(cfg["thetas"]) * n_rhs,
            "l2": f"inputs larger than L2 (L, R {8 * n * n / 1e9:.1f} GB each)",
            "parallelism": parallelism(args, world)}


def parallelism(args, world):
    return "single GPU" if world == 1 else (
        f"modes sharded x{world}: band reduction distributed when the library communicator "
        f"is attached (64-column blocks round-robin, panel broadcasts + all-reduced partial "
        f"products over NCCL; see the communicator line on stderr), bulge chasing + "
        f"tridiagonal solve replicated, eigenvector "
        f"back-transforms, drive/observable projections and stepping column-sharded, one "
        f"all-reduce of partial observables per 2048-step block")


def run_ours(args, cfg, rank, world, local_rank):
    import torch
    # EM_BENCH_SAME_DEVICE=1: every rank on cuda:0 (functional test of the N > 1 path on one
    # GPU, with EM_BENCH_BACKEND=gloo); never for a reported number
    dev = 0 if os.environ.get("EM_BENCH_SAME_DEVICE") else local_rank
    torch.cuda.set_device(dev)
    from paper_2407_11993_b200 import _native as nat
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("EM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    nat.context()
    if world > 1:
        # the library's own communicator: NCCL on the context stream (callbacks through
        # torch.distributed when the ranks share a device under gloo)
        from paper_2407_11993_b200 import parallel
        try:
            parallel.attach_communicator(dist)
        except Exception as exc:  # noqa: BLE001 (the run continues with a replicated reduction)
            # every rank must take the same path: agree on the outcome
            ok = torch.zeros(1, device="cuda")
            print(f"[rank {rank}] library communicator unavailable ({exc}); band reduction "
                  f"replicated", file=sys.stderr)
        else:
            ok = torch.ones(1, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if float(ok.item()) == 0.0:
            parallel.detach_communicator()
    if args.two_stage is not None:
        nat.set_two_stage_min(args.two_stage)
    if os.environ.get("EM_SYTRD_DBG"):  # A/B switch for the tridiagonalisation code paths
        nat.check(nat.load_library().em_config(nat.context(), 98, int(os.environ["EM_SYTRD_DBG"])))
    for kv in filter(None, os.environ.get("EM_CONFIG", "").split(",")):  # A/B: "key=value,..."
        key, val = kv.split("=")
        nat.check(nat.load_library().em_config(nat.context(), int(key), int(val)))
    m = build_inputs(cfg)
    n = m["plate"].n
    T, nth = cfg["steps"], len(cfg["thetas"])
    n_rhs = (cfg["n_ports"] + cfg["n_sources"]) if cfg.get("sweep") else 1
    units = n * T * nth * n_rhs
    step = ShardedDeviceStep(m, cfg, dist, rank, world) if world > 1 else DeviceStep(m, cfg)
    for _ in range(args.warmup):
        step()
    nat.synchronize()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    nat.profile(True)  # coarse stage events on the launching stream
    l0 = nat.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        barrier()
    launches = nat.launches() - l0
    elapsed = ev0.elapsed_time(ev1) / 1e3
    stages = nat.stage_times()
    nat.profile(False)
    t_max = elapsed
    if dist:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = units * args.steps / t_max  # the whole job (N > 1 shards one workload)
    if args.profile_fine:
        nat.profile(2)
        step()
        fine = nat.stage_times()
        nat.profile(0)
        log(json.dumps({"fine_stage_ms": {k: [round(v[0], 3), v[1]] for k, v in fine.items()}}))
    v_host = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the solved V on the host: the CPU leg times the reference's per-step V @ q on it
        v_host = step.V.cpu().numpy()
    del step  # its V (and V^T R) buffers: the e2e arm allocates its own
    torch.cuda.empty_cache()

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        es = E2EShardedStep(m, cfg, dist) if world > 1 else E2EStep(m, cfg)
        # the e2e arm uploads its own L, R from the pinned host copies: drop the
        # device-resident ones meanwhile (C3: 7 N^2 of 9 available at the eigensolve peak)
        m["l_i"] = m["r_i"] = None
        torch.cuda.empty_cache()
        # no e2e warm-up pass: the device arm's warm-up steps already loaded every kernel
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            es()
        torch.cuda.synchronize()
        barrier()
        te = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": units * args.e2e_steps / te, "unit": "mode-steps/s",
               "h2d_bytes_per_step": es.h2d, "d2h_bytes_per_step": es.d2h,
               "ms_per_step": te / args.e2e_steps * 1e3, "steps": args.e2e_steps,
               "timer": "host wall clock around the public-API calls (includes H2D/D2H)"}
        m["l_i"] = es.pinned[0].to("cuda", non_blocking=False)
        m["r_i"] = es.pinned[1].to("cuda", non_blocking=False)
        del es

    # ---- the implicit-V variant of the same step (not the headline: the reference forms V)
    implicit = None
    if world == 1 and not args.no_implicit:
        ist = ImplicitDeviceStep(m, cfg)
        ist()  # warm-up (its transposed back-transform kernels)
        torch.cuda.synchronize()
        i0e, i1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0e.record()
        for _ in range(args.implicit_steps):
            ist()
        i1e.record()
        torch.cuda.synchronize()
        ti = i0e.elapsed_time(i1e) / 1e3 / args.implicit_steps
        implicit = {"value": units / ti, "unit": "mode-steps/s", "ms_per_step": ti * 1e3,
                    "steps": args.implicit_steps, "warmup": 1,
                    "note": "em_sygv_implicit: V^T applied to the drive columns and observable "
                            "rows only (no V formed, no Q1/Q2 back-transform of the n x n "
                            "eigenvectors); same eigenvalues and observables as the headline "
                            "(tests/test_gpu_parity_configs.py)"}
        del ist
        torch.cuda.empty_cache()

    peaks = load_peaks()
    n_steps_timed = args.steps
    st_avg = {k: (v[0] / n_steps_timed, v[1] / n_steps_timed) for k, v in stages.items()}
    # roofline of the dominant kernel: the largest eigensolve stage of the step (stage
    # times are CUDA events on the launching stream, averaged per step)
    rl = roofline(st_avg, n, peaks) or {}
    q2prof = os.path.join(ROOT, "profiles", "r02", "ncu_q2r.json")
    if rl.get("stage") == "q2_apply":
        rl["kernel"] = ("q2r_kernel (+ q2r_pack_kernel, q2_tfactor_kernel): register-resident "
                        "stage-2 back-transform, one launch per 64-sweep group")
        rl["peak_source"] = "DMMA issue peak measured on this pool (profiles/r01_fp64_peaks.jsonl)"
        # the stage is one q2r_kernel launch per 64-sweep group (the stage timer counts 1)
        rl["launches_per_step"] = float((n - 1 + 63) // 64)
        if os.path.exists(q2prof):
            pq = json.load(open(q2prof))
            # measured at n = 16,384 (one group of 101 blocks), not at this workload's n
            rl["traffic_ncu"] = {"n": pq.get("n"), "dram_bytes_per_launch": pq.get("dram_bytes"),
                                 "algorithmic_bytes_per_launch": pq.get("algorithmic_bytes"),
                                 "dmma_pipe_active_pct": pq.get("dmma_pipe_active_pct"),
                                 "source": "profiles/r02/ncu_q2r.json (ncu --set full, one "
                                           "launch of tools/q2_probe.py 16384)"}
        q2c3 = os.path.join(ROOT, "profiles", "r02", "ncu_q2r_c3.json")
        if n == 50000 and os.path.exists(q2c3):
            # one launch of THIS workload under ncu --set full (the middle sweep group):
            # DRAM bytes of that launch beside its algorithmic bytes (its Z rows once in,
            # once out); the stage's other 781 launches differ only in their row count
            pc = json.load(open(q2c3))
            rl["traffic"] = pc.get("dram_bytes")
            rl["traffic_launch"] = {k: pc.get(k) for k in (
                "launch_index", "group", "blocks", "duration_ms", "algorithmic_bytes",
                "useful_flop", "useful_TFps", "dmma_pipe_active_pct", "source_report")}
    if "sytrd" in st_avg and "q2_apply" not in st_avg:
        # one-stage tridiagonalisation (below the two-stage threshold): its symv is the
        # HBM-bound kernel, timed live at the full order
        rl["symv"] = symv_roofline(m, n, peaks)
    # the modal stepping (north-star (b)): the fused replay is DMMA-bound on the observable
    # reconstruction, 2 n_obs flop per mode-step (nothing N x T reaches HBM)
    if "td2_replay" in stages:
        ms_rep = stages["td2_replay"][0] / n_steps_timed
        fl = 2.0 * cfg["n_obs"] * units
        rl["stepping_roofline"] = {
            "kernel": "td2_replay (fused forcing + recurrence + DMMA reconstruction)",
            "bound": "tensor", "unit": "TFLOP/s",
            "achieved": fl / (ms_rep * 1e-3) / 1e12 if ms_rep > 0 else None,
            "peak": peaks.get("fp64_tflops", 37.1),
            "frac": (fl / (ms_rep * 1e-3) / 1e12) / peaks.get("fp64_tflops", 37.1)
            if ms_rep > 0 else None,
            "algorithmic_flop_per_step": fl, "ms_per_step": ms_rep,
            "peak_source": "DMMA issue peak measured on this pool (profiles/r01_fp64_peaks.jsonl)",
            "mode_steps_per_s": units / ((stages["td2_replay"][0] + stages.get("td2_local", (0, 0))[0]
                                          + stages.get("td2_carry", (0, 0))[0]) / n_steps_timed
                                         * 1e-3)}

    # the whole eigensolve against the FP64 tensor peak (north-star target: >= 0.6), on
    # SURVEY 8(d)'s operation counts: (17/3) N^3 for the dense one-stage LAPACK sequence,
    # and with R's band b = ny nz exploited (10/3) N^3 + 6 N^2 b
    eig_ms = sum(stages[k][0] for k in ("potrf_R", "sygst", "potrf_L", "sytrd", "stedc",
                                        "ormtr", "trsm_back", "finalize", "post_gemm")
                 if k in stages) / n_steps_timed
    if eig_ms > 0:
        bw = cfg["grid"][1] * cfg["grid"][2]
        fp64 = peaks.get("fp64_tflops", 37.1)
        dense = 17.0 / 3.0 * n ** 3
        banded = 10.0 / 3.0 * n ** 3 + 6.0 * n ** 2 * bw
        rl["eigensolve_roofline"] = {
            "ms_per_step": eig_ms, "bound": "tensor", "unit": "TFLOP/s", "peak": fp64,
            "achieved_dense_count": dense / (eig_ms * 1e-3) / 1e12,
            "frac_dense_count": dense / (eig_ms * 1e-3) / 1e12 / fp64,
            "achieved_banded_count": banded / (eig_ms * 1e-3) / 1e12,
            "frac_banded_count": banded / (eig_ms * 1e-3) / 1e12 / fp64,
            "stages_ms": {k: round(st_avg[k][0], 1) for k in (
                "potrf_R", "sygst", "potrf_L", "sy2sb", "sb2st", "stedc", "q2_apply",
                "q1_apply", "sytrd", "ormtr", "trsm_back", "finalize", "post_gemm")
                if k in st_avg},
            "note": "dense count (17/3) N^3 is the one-stage LAPACK sequence with a dense R; "
                    "the banded count uses R's band b = ny nz (SURVEY 8(d))"}

    # ---- TD1 comparator (bounded: a few hundred steps, extrapolated) and CPU baseline
    extra = {}
    if rank == 0 and not args.no_td1:
        extra["td1_comparator"] = td1_comparator(m, cfg, args.td1_steps, n_rhs)
        extra["td1_comparator"]["modal_vs_cholesky_end_to_end"] = (
            extra["td1_comparator"]["extrapolated_total_s"] / (t_max / args.steps))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, cfg, units, v_host)
        del v_host
    if rank == 0:
        line = {
            "metric": "end-to-end transient wall time (eigensolve + steps); mode-steps/sec",
            "value": value, "unit": "mode-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded plate generator, SURVEY.md §8(d))",
            "config": workload_config(args, cfg, n, world),
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "roofline": rl,
            "stage_ms_per_step": {k: round(v[0], 3) for k, v in st_avg.items()},
            "cpu_baseline": cpu,
            "implicit_v": implicit,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if dist:
        from paper_2407_11993_b200 import parallel
        if rank == 0:
            print("communicator: " + json.dumps(parallel.communicator_info()), file=sys.stderr)
        parallel.detach_communicator()
        dist.destroy_process_group()


def run_c4(args, cfg, rank, world, local_rank):
    """configs[3] (N = 120,000 minus the notch, L = 115 GB) on ONE B200: the modal path as
    the implicit-V eigensolve (em_sygv_implicit_band: L reduced in place, R in band storage,
    V^T applied to [R_D | L_D | C^T] only) + 100,000 TD2 steps, and the Cholesky
    comparator in place (em_td1_plan_create_band). L is regenerated on the device before
    every step (the step consumes it) outside the timed region; each step is timed with
    CUDA events around the solve + scan."""
    import ctypes
    import torch
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import synth
    if world > 1:
        if rank == 0:
            print(json.dumps({"metric": "end-to-end transient wall time (eigensolve + steps); "
                              "mode-steps/sec", "config": {"workload": "C4"},
                              "unavailable": "C4 on >1 GPU needs the distributed eigensolve "
                                             "(not built); C4 runs on one GPU"}), flush=True)
        return
    torch.cuda.set_device(local_rank)
    lib, ctx = nat.load_library(), nat.context()
    nx, ny, nz = cfg["grid"]
    m = synth.device_plate_model(nx, ny, nz, n_ports=cfg["n_ports"], n_sources=cfg["n_sources"],
                                 n_obs=cfg["n_obs"], notch=True, r_dense=False,
                                 ldl=(synth.Plate(nx, ny, nz, notch=True).n + 31) // 32 * 32)
    n = m["plate"].n
    ldl = m["ldl"]
    bw, rb = m["r_bw"], m["r_band"]
    T, n_obs = cfg["steps"], cfg["n_obs"]
    i_d, i0 = synth.drive_table(cfg["drive"], T, cfg["dt"], cfg["n_ports"], cfg["n_sources"],
                                plate=m["plate"])
    table = np.ascontiguousarray(np.concatenate([i_d, i0], axis=1))
    table_dev = nat.device_vector(table.reshape(-1))
    ct = nat.device_colmajor(m["c"]).reshape(n, n_obs).t().contiguous()   # C^T columns
    y0 = torch.cat([m["r_d"], m["l_d"], ct], dim=0).contiguous()           # (2 + n_obs, n)
    k = y0.shape[0]
    yp = torch.empty_like(y0)
    tau = nat.empty(n)
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    q = nat.zeros(n)
    Y = nat.empty(T, n_obs)
    log(f"C4: n = {n}, band {bw}, k = {k}, L {8 * n * n / 1e9:.1f} GB")

    def step(timed_events=None):
        m["regen_l"]()
        yp.copy_(y0)
        torch.cuda.synchronize()
        if timed_events:
            timed_events[0].record()
        piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
        nat.check(lib.em_sygv_implicit_band(ctx, n, nat.ptr(m["l_i"]), ldl, nat.ptr(rb), bw + 1,
                                            bw,
                                            nat.ptr(tau), nat.ptr(yp), n, k, None, None,
                                            nat.EM_SYGV_L_WORKSPACE, ctypes.byref(piv),
                                            ctypes.byref(which)), "em_sygv_implicit_band")
        cv = yp[2:].t().contiguous()
        plan = ctypes.c_void_p()
        nat.check(lib.em_td2_plan_create(ctx, n, 1, 0, nat.ptr(tau), nat.ptr(one),
                                         nat.ptr(yp[0:1]), nat.ptr(yp[1:2]), nat.ptr(yp[0:1]),
                                         cfg["dt"], cfg["thetas"][0], ctypes.byref(plan)),
                  "em_td2_plan_create")
        nat.check(lib.em_td2_set_observables(plan, n_obs, nat.ptr(cv), n_obs, None, 0),
                  "em_td2_set_observables")
        q.zero_()
        nat.check(lib.em_td2_run(plan, T, nat.ptr(table_dev), nat.ptr(q), nat.ptr(Y), 1, None),
                  "em_td2_run")
        lib.em_td2_plan_destroy(plan)
        if timed_events:
            timed_events[1].record()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    nat.profile(True)
    l0 = nat.launches()
    total = 0.0
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            step(ev)
            total += ev[0].elapsed_time(ev[1]) / 1e3
    launches = nat.launches() - l0
    stages = nat.stage_times()
    nat.profile(False)
    units = n * T
    st_avg = {kk: (v[0] / args.steps, v[1] / args.steps) for kk, v in stages.items()}
    peaks = load_peaks()
    rl = roofline(st_avg, n, peaks, k=k) or {}
    eig_ms = sum(st_avg[kk][0] for kk in ("potrf_R", "sygst", "sytrd", "stedc", "ormtr",
                                          "finalize") if kk in st_avg)
    fp64 = peaks.get("fp64_tflops", 37.1)
    red = 4.0 / 3.0 * n ** 3  # the dense -> band reduction, the only n^3 term left
    rl["eigensolve_roofline"] = {
        "ms_per_step": eig_ms, "bound": "tensor", "unit": "TFLOP/s", "peak": fp64,
        "achieved_reduction_count": red / (eig_ms * 1e-3) / 1e12,
        "frac_reduction_count": red / (eig_ms * 1e-3) / 1e12 / fp64,
        "note": "implicit V: (4/3) N^3 of the band reduction is the whole cubic count; the "
                "back-transforms act on k = 2 + n_obs columns (O(N^2 k))"}
    y_host = Y[-1].cpu().numpy()
    del yp, q
    # the Cholesky comparator in L's storage (bounded number of steps, extrapolated)
    td1 = None
    if not args.no_td1:
        m["regen_l"]()
        steps1 = min(args.td1_steps, T)
        plan = ctypes.c_void_p()
        piv = ctypes.c_int64(-1)
        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        e0.record()
        nat.check(lib.em_td1_plan_create_band(ctx, n, 1, 0, nat.ptr(m["l_i"]), ldl, nat.ptr(rb),
                                              bw + 1, bw, nat.ptr(m["r_d"]), nat.ptr(m["l_d"]),
                                              None, cfg["dt"], cfg["thetas"][0],
                                              nat.EM_TD1_L_WORKSPACE, ctypes.byref(plan),
                                              ctypes.byref(piv)), "em_td1_plan_create_band")
        e1.record()
        c_dev = nat.device_colmajor(m["c"])
        nat.check(lib.em_td1_set_observables(plan, n_obs, nat.ptr(c_dev), n_obs, None, 0))
        state = nat.zeros(n)
        y1 = nat.empty(steps1, n_obs)
        nat.profile(True)
        e2.record()
        nat.check(lib.em_td1_run(plan, steps1, nat.ptr(table_dev), nat.ptr(state), nat.ptr(y1), 1,
                                 None), "em_td1_run")
        e3.record()
        torch.cuda.synchronize()
        st1 = nat.stage_times()
        nat.profile(False)
        lib.em_td1_plan_destroy(plan)
        # the same theta-method in the Cholesky basis: its first steps must reproduce the
        # modal run's observables (a full-size parity property of the C4 path)
        ya, yb = y1.cpu().numpy(), Y[:steps1].cpu().numpy()
        td1_vs_td2 = float(np.linalg.norm(ya - yb) / np.linalg.norm(yb))
        setup = e0.elapsed_time(e1) / 1e3
        per_step = e2.elapsed_time(e3) / 1e3 / steps1
        fb = 8.0 * n * (n + 1) / 2
        fwd, bwd = st1.get("td1_fwd", (0.0, 1)), st1.get("td1_bwd", (0.0, 1))
        hbm = peaks.get("hbm_gbs", 6550.4)
        td1 = {"method": "td1 (GPU Cholesky theta-method, factor in L's storage, R as CSR)",
               "setup_s": setup, "per_step_ms": per_step * 1e3, "steps_timed": steps1,
               "extrapolated_total_s": setup + per_step * T,
               "trsv_fwd_GBps": fb / (fwd[0] / fwd[1] * 1e-3) / 1e9 if fwd[1] else None,
               "trsv_bwd_GBps": fb / (bwd[0] / bwd[1] * 1e-3) / 1e9 if bwd[1] else None,
               "hbm_peak_GBps": hbm,
               "td1_vs_td2_observables_rel_l2": td1_vs_td2,
               "modal_vs_cholesky_end_to_end": (setup + per_step * T) / (total / args.steps)}
    line = {
        "metric": "end-to-end transient wall time (eigensolve + steps); mode-steps/sec",
        "value": units * args.steps / total, "unit": "mode-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded notched plate generator, SURVEY.md §8(d))",
        "config": {"workload": f"C4: N={n} notched plate {cfg['grid']}, implicit-V eigensolve "
                               f"+ {T} TD2 steps x theta {list(cfg['thetas'])}, {n_obs} "
                               "observables", "N": n, "T": T, "n_obs": n_obs,
                   "mode_steps_per_step": units, "eigensolve": "implicit V (no V formed)",
                   "l2": f"inputs larger than L2 (L {8 * n * n / 1e9:.1f} GB)",
                   "parallelism": "single GPU"},
        "e2e": None,
        "e2e_note": "not measured at C4: the host copy of L alone is 115 GB",
        "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": rl,
        "stage_ms_per_step": {kk: round(v[0], 3) for kk, v in st_avg.items()},
        "cpu_baseline": None, "td1_comparator": td1,
        "last_observables_l2": float(np.linalg.norm(y_host)),
    }
    print(json.dumps(line), flush=True)


def td1_comparator(m, cfg, steps, n_rhs=1):
    """GPU Cholesky theta-method on the same inputs (bounded number of steps)."""
    import ctypes
    import torch
    from paper_2407_11993_b200 import _native as nat
    lib, ctx = nat.load_library(), nat.context()
    n = m["plate"].n
    n_p, n_s = cfg["n_ports"], cfg["n_sources"]
    th = cfg["thetas"][-1]
    steps = min(steps, cfg["steps"])
    plan = ctypes.c_void_p()
    piv = ctypes.c_int64(-1)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    nat.check(lib.em_td1_plan_create(ctx, n, n_p, n_s, nat.ptr(m["l_i"]), n, nat.ptr(m["r_i"]), n,
                                     nat.ptr(m["r_d"]) if n_p else None,
                                     nat.ptr(m["l_d"]) if n_p else None,
                                     nat.ptr(m["m0_dev"]) if n_s else None, cfg["dt"], th,
                                     ctypes.byref(plan), ctypes.byref(piv)), "em_td1_plan_create")
    e1.record()
    nat.check(lib.em_td1_set_observables(plan, cfg["n_obs"], nat.ptr(m["c_dev"]), cfg["n_obs"],
                                         None, 0), "em_td1_set_observables")
    state = nat.zeros(n)
    y = nat.empty(steps, cfg["n_obs"])
    nat.profile(True)
    e1b = torch.cuda.Event(enable_timing=True)
    e1b.record()
    nat.check(lib.em_td1_run(plan, steps, nat.ptr(m["table_dev"]), nat.ptr(state), nat.ptr(y), 1,
                             None), "em_td1_run")
    e2.record()
    torch.cuda.synchronize()
    st = nat.stage_times()
    nat.profile(False)
    lib.em_td1_plan_destroy(plan)
    setup = e0.elapsed_time(e1) / 1e3
    per_step = e1b.elapsed_time(e2) / 1e3 / steps
    nth = len(cfg["thetas"])
    # a sweep needs one Cholesky run per right-hand side (same factor)
    total = nth * (setup + per_step * cfg["steps"] * n_rhs)
    fwd = st.get("td1_fwd", (0.0, 1))
    symv = st.get("td1_symv", (0.0, 1))
    bwd = st.get("td1_bwd", (0.0, 1))
    factor_bytes = 8.0 * n * (n + 1) / 2
    hbm = load_peaks().get("hbm_gbs", 6550.4)
    return {
        "method": "td1 (GPU Cholesky theta-method, same inputs)",
        "setup_s_per_theta": setup, "per_step_ms": per_step * 1e3, "steps_timed": steps,
        "extrapolated_total_s": total,
        "modal_vs_cholesky_end_to_end": None,  # filled by the caller
        "trsv_fwd_GBps": factor_bytes / (fwd[0] / fwd[1] * 1e-3) / 1e9 if fwd[1] else None,
        "trsv_bwd_GBps": factor_bytes / (bwd[0] / bwd[1] * 1e-3) / 1e9 if bwd[1] else None,
        "r_product_ms_per_step": symv[0] / symv[1] if symv[1] else None,
        "r_product": "CSR SpMV of the stencil R (dense symv when R is not sparse)",
        "hbm_peak_GBps": hbm,
    }


def cpu_baseline(n, cfg, units, v_host=None):
    """The reference algorithm on this host's cores (oracle port), bounded samples,
    extrapolated per component (oracle/cpu_baseline.py)."""
    from oracle import cpu_baseline as cb
    n_rhs = (cfg["n_ports"] + cfg["n_sources"]) if cfg.get("sweep") else 1
    est = cb.estimate(n, cfg["n_ports"], cfg["n_sources"], cfg["steps"],
                      len(cfg["thetas"]) * n_rhs, cfg["dt"], v_full=v_host)
    return {"value": units / est["total_s"], "unit": "mode-steps/s", "cores": est["cores"],
            "kind": "port", "sample": est["sample"], "extrapolated": True,
            "extrapolated_total_s": est["total_s"], "components_s": est["components"],
            "fits": est["fits"], "cpu_model": est["cpu_model"],
            "per_step_ms": est["per_step_ms"],
            "from_modal_gemv_ms_fit": est["from_modal_gemv_ms_fit"],
            "from_modal_gemv_ms_full_n": est["from_modal_gemv_ms_full_n"]}


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference algorithm on the host cores (oracle port of its
    numba kernels + numpy BLAS), rank 0 only. Each step is one bounded sample of the
    workload (every eigensolve stage on small plates, the step kernel at the full N, the
    V @ q GEMV at three orders); `value` is the full workload's mode-steps/s extrapolated
    from the step's sample, `ms_per_step` the sample's own wall time."""
    if rank != 0:
        return
    from oracle import cpu_baseline as cb
    from paper_2407_11993_b200 import synth
    nx, ny, nz = cfg["grid"]
    n = synth.Plate(nx, ny, nz, notch=cfg.get("notch", False)).n
    n_rhs = (cfg["n_ports"] + cfg["n_sources"]) if cfg.get("sweep") else 1
    units = n * cfg["steps"] * len(cfg["thetas"]) * n_rhs

    def sample():
        return cb.estimate(n, cfg["n_ports"], cfg["n_sources"], cfg["steps"],
                           len(cfg["thetas"]) * n_rhs, cfg["dt"])
    for _ in range(args.warmup):
        sample()
    totals, walls = [], []
    est = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        est = sample()
        walls.append(time.perf_counter() - t0)
        totals.append(est["total_s"])
    t = statistics.median(totals)
    value = units / t
    line = {
        "impl": "reference",
        "metric": "end-to-end transient wall time (eigensolve + steps); mode-steps/sec",
        "value": value, "unit": "mode-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded plate generator, SURVEY.md §8(d))",
        "config": workload_config(args, cfg, n, world),
        "value_kind": "extrapolated: the full workload's mode-steps/s from each step's bounded "
                      "sample (median over steps); ms_per_step is the sample's wall time",
        "extrapolated_total_s": t,
        "extrapolated_spread": [min(totals), max(totals)],
        "cpu_baseline": {"value": value, "unit": "mode-steps/s", "cores": est["cores"],
                         "kind": "port", "sample": est["sample"], "extrapolated": True,
                         "cpu_model": est["cpu_model"]},
        "e2e": {"value": value, "unit": "mode-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "components_s": est["components"],
        "fits": est["fits"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C3")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--td1-steps", type=int, default=300)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-td1", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-implicit", action="store_true")
    ap.add_argument("--grid", default=None,
                    help="nx,ny,nz override (debugging a configuration's code path at a "
                         "smaller plate; the workload string names the grid)")
    ap.add_argument("--implicit-steps", type=int, default=1)
    ap.add_argument("--two-stage", type=int, default=None,
                    help="smallest n for the two-stage tridiagonalisation (default: library)")
    ap.add_argument("--profile-fine", action="store_true",
                    help="one extra untimed step with per-call stage events (stderr)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = dict(CONFIGS[args.config])
    if args.grid:
        cfg["grid"] = tuple(int(v) for v in args.grid.split(","))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if args.config == "C4":
        run_c4(args, cfg, rank, world, local_rank)
        return
    run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
