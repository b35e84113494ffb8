"""Drive each hot kernel once or a few times at C2 scale (N = 16,384) through the
C ABI, for ncu captures and CUDA-event timings (measurement tool, not product).

    python tools/prof_kernels.py [symv|gemm|td2|td1|all]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_11993_b200 import _native as nat  # noqa: E402


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main(which):
    ctx, lib = nat.context(), nat.load_library()
    g = torch.Generator(device="cuda").manual_seed(7)
    out = {}
    n = 16384
    if "SYMV_KEEP_MB" in os.environ:  # EM_CFG_SYMV_L2_KEEP_MB (every branch)
        nat.check(lib.em_config(ctx, 3, int(os.environ["SYMV_KEEP_MB"])))
    if which in ("symv", "all"):
        a = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
        x = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
        y = torch.empty_like(x)
        t = timed(lambda: nat.check(lib.em_symv_lower(ctx, n, 1.0, nat.ptr(a), n, nat.ptr(x), 0.0,
                                                      nat.ptr(y))))
        out["symv_n16384_s"] = t
        out["symv_GBps_algorithmic"] = 8 * n * n / 2 / t / 1e9
        del a
    if which in ("gemm", "all"):
        m = 8192
        a = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g)
        b = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g)
        c = torch.empty_like(a)
        t = timed(lambda: nat.check(lib.em_dgemm(ctx, 0, 0, m, m, m, 1.0, nat.ptr(a), m,
                                                 nat.ptr(b), m, 0.0, nat.ptr(c), m)), reps=2)
        out["dgemm_8192_TFps"] = 2 * m ** 3 / t / 1e12
        del a, b, c
    if which in ("td2", "all"):
        n = int(os.environ.get("TD2_N", n))
        T, n_obs = int(os.environ.get("TD2_T", 10000)), int(os.environ.get("TD2_OBS", 32))
        ln = torch.rand(n, device="cuda", dtype=torch.float64, generator=g) * 8 + 0.1
        rn = torch.ones(n, device="cuda", dtype=torch.float64)
        pr = torch.randn(n, device="cuda", dtype=torch.float64, generator=g) * 1e-6
        pl = torch.randn(n, device="cuda", dtype=torch.float64, generator=g) * 1e-6
        cv = torch.randn(n, n_obs, device="cuda", dtype=torch.float64, generator=g)
        tt = np.minimum(5e-7 * np.arange(T + 1) / 5e-6, 1.0)
        drive = nat.device_vector(tt)
        plan = ctypes.c_void_p()
        nat.check(lib.em_td2_plan_create(ctx, n, 1, 0, nat.ptr(ln), nat.ptr(rn), nat.ptr(pr),
                                         nat.ptr(pl), nat.ptr(pr), 5e-7, 0.5, ctypes.byref(plan)))
        nat.check(lib.em_td2_set_observables(plan, n_obs, nat.ptr(cv), n_obs, None, 0))
        q = nat.zeros(n)
        y = nat.empty(T, n_obs)
        t = timed(lambda: nat.check(lib.em_td2_run(plan, T, nat.ptr(drive), nat.ptr(q), nat.ptr(y),
                                                   1, None)))
        out["td2_run_s"] = t
        out["td2_mode_steps_per_s"] = n * T / t
        out["td2_recon_TFps"] = 2 * n_obs * n * T / t / 1e12
        lib.em_td2_plan_destroy(plan)
    if which in ("td1", "all"):
        m = int(os.environ.get("TD1_N", 8192))
        b = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g) / np.sqrt(m)
        lmat = b @ b.T + torch.eye(m, device="cuda", dtype=torch.float64)
        rmat = torch.eye(m, device="cuda", dtype=torch.float64) * 1e-3
        plan = ctypes.c_void_p()
        piv = ctypes.c_int64(-1)
        rd = torch.randn(m, device="cuda", dtype=torch.float64, generator=g)
        nat.check(lib.em_td1_plan_create(ctx, m, 1, 0, nat.ptr(lmat), m, nat.ptr(rmat), m,
                                         nat.ptr(rd), nat.ptr(rd), None, 1e-6, 0.5,
                                         ctypes.byref(plan), ctypes.byref(piv)))
        steps = 50
        drive = nat.device_vector(np.linspace(0, 1, steps + 1))
        s = nat.zeros(m)
        t = timed(lambda: nat.check(lib.em_td1_run(plan, steps, nat.ptr(drive), nat.ptr(s), None, 1,
                                                   None)), reps=1)
        out[f"td1_n{m}_per_step_ms"] = t / steps * 1e3
        out[f"td1_n{m}_factor_GBps"] = 2 * 8 * m * (m + 1) / 2 / (t / steps) / 1e9
        lib.em_td1_plan_destroy(plan)
    if which == "symvsweep":
        big = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
        x = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
        y = torch.empty_like(x)
        for m in (256, 512, 1024, 2048, 3072, 4096, 6144, 8192, 12288, 16384):
            t = timed(lambda: nat.check(lib.em_symv_lower(ctx, m, 1.0, nat.ptr(big), n, nat.ptr(x),
                                                          0.0, nat.ptr(y))), reps=20)
            out[f"symv_{m}"] = {"us": t * 1e6, "GBps": 8 * m * m / 2 / t / 1e9}
        del big
    if which == "symvoff":
        # trailing-block symv at row/column offsets (alignment of the TMA boxes)
        big = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
        x = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
        y = torch.empty_like(x)
        m = n - 256
        base = big.data_ptr()
        offs = [int(v) for v in os.environ.get("SYMV_OFFS", "0,2,4,8,16,32,1").split(",")]
        for off in offs:
            ptr = ctypes.c_void_p(base + 8 * off * (n + 1))
            t = timed(lambda: nat.check(lib.em_symv_lower(ctx, m, 1.0, ptr, n, nat.ptr(x), 0.0,
                                                          nat.ptr(y))), reps=20)
            out[f"symv_off{off}"] = {"us": t * 1e6, "GBps": 8 * m * m / 2 / t / 1e9}
        del big
    if which == "potrf":
        m = int(os.environ.get("POTRF_N", n))
        b = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g) / np.sqrt(m)
        a = (b @ b.T + torch.eye(m, device="cuda", dtype=torch.float64)).contiguous()
        del b
        piv = ctypes.c_int64(-1)
        for rep in range(2):
            w2 = a.clone()
            torch.cuda.synchronize()
            t = timed(lambda: nat.check(lib.em_potrf(ctx, m, nat.ptr(w2), m, ctypes.byref(piv))),
                      reps=1)
            out[f"potrf_{m}_rep{rep}_ms"] = t * 1e3
            out[f"potrf_{m}_TFps"] = m ** 3 / 3 / t / 1e12
        bm = a.clone()
        t = timed(lambda: nat.check(lib.em_trsm_lower(ctx, 0, m, m, nat.ptr(w2), m, nat.ptr(bm), m)),
                  reps=1)
        out[f"trsm_{m}_ms"] = t * 1e3
        out[f"trsm_{m}_TFps"] = m ** 3 / t / 1e12
    if which == "syev":
        m = int(os.environ.get("SYEV_N", n))
        if "SYTRD_DBG" in os.environ:  # em_config debug key 98 (sytrd switches)
            nat.check(lib.em_config(ctx, 98, int(os.environ["SYTRD_DBG"])))
        if "SYMV_KEEP_MB" in os.environ:  # EM_CFG_SYMV_L2_KEEP_MB
            nat.check(lib.em_config(ctx, 3, int(os.environ["SYMV_KEEP_MB"])))
        b = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g)
        a = (b + b.T).contiguous()
        del b
        w = torch.empty(m, device="cuda", dtype=torch.float64)
        u = torch.empty(m, m, device="cuda", dtype=torch.float64)
        for lvl in (1, 2):
            w2 = a.clone()
            nat.profile(lvl)
            nat.check(lib.em_syev(ctx, m, nat.ptr(w2), m, nat.ptr(w), nat.ptr(u), m))
            torch.cuda.synchronize()
            out[f"syev_{m}_level{lvl}"] = nat.stage_times()
            del w2
        nat.profile(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
