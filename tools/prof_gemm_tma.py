"""One shape of the TMA-fed DGEMM for ncu (measurement tool): SHAPE=m,n,k,ta,tb BETA=b."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_11993_b200 import _native as nat
ctx, lib = nat.context(), nat.load_library()
m, n, k, ta, tb = (int(x) for x in os.environ.get("SHAPE", "16384,16384,128,0,1").split(","))
beta = float(os.environ.get("BETA", "1"))
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn((m, k) if ta else (k, m), device="cuda", dtype=torch.float64, generator=g)
B = torch.randn((k, n) if tb else (n, k), device="cuda", dtype=torch.float64, generator=g)
C = torch.zeros(n, m, device="cuda", dtype=torch.float64)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(3):
    e0.record()
    nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, -1.0, nat.ptr(A), A.shape[1], nat.ptr(B), B.shape[1],
                           beta, nat.ptr(C), m))
    e1.record()
    torch.cuda.synchronize()
print({"shape": (m, n, k, ta, tb), "beta": beta, "ms": e0.elapsed_time(e1),
       "TFps": 2.0 * m * n * k / e0.elapsed_time(e1) / 1e9})
