import sys, numpy as np
sys.path.insert(0, '.')
from paper_2407_11993_b200 import _native as nat
from paper_2407_11993_b200.linalg import sym_eig
lib = nat.load_library(); ctx = nat.context()
rng = np.random.default_rng(1)
for n, dotr in [(1500, 2048), (1500, 512), (3000, 2048), (3000, 4096), (5000, 2048), (2100, 8192), (2000, 2048), (8000, 2048)]:
    a = rng.standard_normal((n, n)); a = (a + a.T) / 2
    ref = np.linalg.eigvalsh(a)[::-1]
    lib.em_config(ctx, 99, dotr); lib.em_config(ctx, 2, 1)
    lam, u = sym_eig(a)
    print(n, dotr, np.abs(lam - ref).max() / np.abs(ref).max(), flush=True)
