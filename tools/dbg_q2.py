"""Debug: per-column check of the two-stage eigenvectors (em_syev, Q2 mode given)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2407_11993_b200 import _native as nat  # noqa: E402


def main():
    n = int(sys.argv[1])
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dbg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    lib, ctx = nat.load_library(), nat.context()
    nat.check(lib.em_config(ctx, 94, dbg))
    nat.set_two_stage_min(0)
    nat.check(lib.em_config(ctx, 97, mode))
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    a = b + b.T
    ad = nat.device_vector(a.reshape(-1))
    w = torch.empty(n, device="cuda", dtype=torch.float64)
    u = torch.empty(n * n, device="cuda", dtype=torch.float64)
    nat.check(lib.em_syev(ctx, n, nat.ptr(ad), n, nat.ptr(w), nat.ptr(u), n), "em_syev")
    U = u.reshape(n, n)  # row j = eigenvector j
    A = torch.from_numpy(a).cuda()
    res = (U @ A - w[:, None] * U).norm(dim=1).cpu().numpy()
    bad = np.where(res > 1e-8 * np.abs(w.cpu().numpy()).max())[0]
    print("n", n, "mode", mode, "dbg", dbg, "bad columns", len(bad), bad[:20], bad[-20:] if len(bad) else "")
    if len(bad):
        print("bad // 8 units:", np.unique(bad // 8)[:50])


if __name__ == "__main__":
    main()
