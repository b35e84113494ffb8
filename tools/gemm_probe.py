"""DGEMM shape sweep: the library's DMMA GEMM (em_dgemm) vs cuBLAS (torch.matmul) on the
shapes the eigensolve uses (measurement tool, not product)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_11993_b200 import _native as nat  # noqa: E402


def timed(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


ctx, lib = nat.context(), nat.load_library()
if "GEMM_TMA" in os.environ:  # em_config debug key 95: 0 off, 1 auto, 2..5 forced TMA config
    nat.check(lib.em_config(ctx, 95, int(os.environ["GEMM_TMA"])))
if "GEMM_CFG" in os.environ:  # em_config debug key 96: 0 auto, 2 64x64 tiles, 3 128x64
    nat.check(lib.em_config(ctx, 96, int(os.environ["GEMM_CFG"])))
g = torch.Generator(device="cuda").manual_seed(3)
shapes = [  # (m, n, k, ta, tb, label)
    (8192, 8192, 8192, 0, 0, "square 8k"),
    (16384, 16384, 128, 0, 1, "syr2k-like K=128 (full)"),
    (16384, 16384, 256, 1, 0, "rank-256 update"),
    (256, 16384, 16384, 1, 0, "ormtr W = V^T Z (K=16k)"),
    (16384, 16384, 256, 0, 0, "ormtr Z -= V W"),
    (16384, 16384, 512, 0, 0, "rank-512 update"),
    (512, 16384, 16384, 1, 0, "W = V^T Z (512 rows)"),
    (4096, 4096, 4096, 0, 1, "square 4k NT"),
    (16384, 16384, 16384, 0, 0, "square 16k"),
]
BETA = float(os.environ.get("BETA", "0"))
out = []
for m, n, k, ta, tb, label in shapes:
    a = torch.randn((k, m) if ta else (m, k), device="cuda", dtype=torch.float64, generator=g)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", dtype=torch.float64, generator=g)
    c = torch.zeros(m, n, device="cuda", dtype=torch.float64)
    # column-major views: X (rows x cols) col-major == X^T row-major torch tensor
    # em_dgemm(C = op(A) op(B)), A col-major m x k (ta=0) stored as torch (k, m) row-major
    A = a.t().contiguous() if not ta else a.t().contiguous()
    B = b.t().contiguous() if not tb else b.t().contiguous()
    lda = A.shape[1]
    ldb = B.shape[1]
    ct = torch.zeros(n, m, device="cuda", dtype=torch.float64)  # col-major m x n
    t_own = timed(lambda: nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 1.0, nat.ptr(A), lda,
                                                 nat.ptr(B), ldb, BETA, nat.ptr(ct), m)))
    aa = a.t() if ta else a
    bb = b.t() if tb else b
    if BETA == 0.0:
        t_cub = timed(lambda: torch.matmul(aa, bb, out=c))
    else:
        t_cub = timed(lambda: torch.addmm(c, aa, bb, beta=BETA, out=c))
    fl = 2.0 * m * n * k
    # one checked product (beta = 0) against cuBLAS
    nat.check(lib.em_dgemm(ctx, ta, tb, m, n, k, 1.0, nat.ptr(A), lda, nat.ptr(B), ldb, 0.0,
                           nat.ptr(ct), m))
    torch.matmul(aa, bb, out=c)
    err = float((ct.t() - c).abs().max()) / float(c.abs().max())
    out.append({"beta": BETA, "shape": label, "m": m, "n": n, "k": k, "own_TFps": fl / t_own / 1e12,
                "cublas_TFps": fl / t_cub / 1e12, "rel_err_vs_cublas": err,
                "tma": os.environ.get("GEMM_TMA", "auto")})
    del a, b, c, A, B, ct
for o in out:
    print(json.dumps(o))
