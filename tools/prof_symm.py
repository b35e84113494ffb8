"""The band reduction's two products for ncu (measurement tool): the symmetric band product
X = A (V T) (em_dsymm_band_lower, m x 64) and the rank-128 lower update A -= [V W][W V]^T
(em_dgemm_lower, diag_off 127) at order M (default 32768)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_11993_b200 import _native as nat
ctx, lib = nat.context(), nat.load_library()
m = int(os.environ.get("M", "32768"))
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g)
A = (A + A.t()).contiguous()
B = torch.randn(64, m, device="cuda", dtype=torch.float64, generator=g)      # m x 64 col-major
X = torch.zeros(64, m, device="cuda", dtype=torch.float64)
VW = torch.randn(128, m, device="cuda", dtype=torch.float64, generator=g)    # m x 128
WV = torch.randn(128, m, device="cuda", dtype=torch.float64, generator=g)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {}
for name, fn, flop in (
        ("symm_band", lambda: nat.check(lib.em_dsymm_band_lower(ctx, m, 64, nat.ptr(A), m, nat.ptr(B), m,
                                                                 nat.ptr(X), m)), 2.0 * m * m * 64),
        ("syr2k_lower", lambda: nat.check(lib.em_dgemm_lower(ctx, 0, 1, m, m, 128, -1.0, nat.ptr(VW), m,
                                                              nat.ptr(WV), m, 1.0, nat.ptr(A), m, 127)),
         2.0 * (m * m / 2 + 127 * m) * 128)):
    for _ in range(3):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    out[name] = {"ms": e0.elapsed_time(e1), "TFps": flop / e0.elapsed_time(e1) / 1e9}
print({"m": m, **out})
