"""Two-stage Q2 back-transform probe: em_syev with the two-stage reduction forced, Q2 in
column-strip form (debug key 97 = 0) or the wavefront grouped-GEMM form (97 = 1);
prints the fine stage times (q2_apply, q1_apply, sy2sb, sb2st) of one call.

    python tools/q2_probe.py N [mode]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2407_11993_b200 import _native as nat  # noqa: E402


def main():
    n = int(sys.argv[1])
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    lib, ctx = nat.load_library(), nat.context()
    nat.set_two_stage_min(0)
    nat.check(lib.em_config(ctx, 97, mode))
    g = torch.Generator(device="cuda").manual_seed(n)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
    a0 = (b + b.T).contiguous()
    w = torch.empty(n, device="cuda", dtype=torch.float64)
    u = torch.empty(n * n, device="cuda", dtype=torch.float64)
    for it in range(2):
        a = a0.clone()
        torch.cuda.synchronize()
        if it == 1:
            nat.profile(2)
        nat.check(lib.em_syev(ctx, n, nat.ptr(a), n, nat.ptr(w), nat.ptr(u), n), "em_syev")
        torch.cuda.synchronize()
    st = nat.stage_times()
    print({k: v for k, v in st.items() if k in ("sy2sb", "sb2st", "q2_apply", "q1_apply", "stedc")})


if __name__ == "__main__":
    main()
