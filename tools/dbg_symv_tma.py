"""Run em_syev at a small n under a sytrd debug switch (em_config key 98) and compare
the eigenvalues with numpy (debug tool, not product).  python tools/dbg_symv_tma.py FLAGS N"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_11993_b200 import _native as nat  # noqa: E402

flags, n = int(sys.argv[1]), int(sys.argv[2])
ctx, lib = nat.context(), nat.load_library()
nat.check(lib.em_config(ctx, 98, flags))
rng = np.random.default_rng(1)
b = rng.standard_normal((n, n))
a = b + b.T
ad = nat.device_colmajor(a)
w = torch.empty(n, device="cuda", dtype=torch.float64)
u = torch.empty(n, n, device="cuda", dtype=torch.float64)
rc = lib.em_syev(ctx, n, nat.ptr(ad), n, nat.ptr(w), nat.ptr(u), n)
torch.cuda.synchronize()
msg = lib.em_last_error(ctx)
ref = np.sort(np.linalg.eigvalsh(a))[::-1]
got = np.sort(w.cpu().numpy())[::-1]
print(f"flags={flags} n={n} rc={rc} err={msg} maxrel={np.max(np.abs(got - ref)) / np.max(np.abs(ref)):.3e}")
