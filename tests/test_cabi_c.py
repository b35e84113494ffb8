"""The drop-in boundary from C: tests/cabi/sygv_demo.c includes only
include/eddymodes_b200.h and links libeddymodes_b200.so (no Python, no torch)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(REPO, "paper_2407_11993_b200")


def _build(tmp_path):
    if shutil.which("nvcc") is None and shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "sygv_demo")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-O2", "-std=c11", os.path.join(REPO, "tests", "cabi", "sygv_demo.c"),
           "-I", os.path.join(REPO, "include"), "-I", os.path.join(cuda, "include"),
           "-L", LIBDIR, "-leddymodes_b200", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_caller_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_caller_runs(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    vals = dict(zip(out[0::2], out[1::2]))
    n = int(vals["n"])
    i = np.arange(n)
    d = np.abs(i[:, None] - i[None, :]).astype(float)
    L = 1.0 / (1.0 + d) + np.eye(n)
    R = np.diag(2.0 + 0.01 * i) - 0.5 * (d == 1.0)
    from scipy.linalg import eigh
    tau = eigh(L, R, eigvals_only=True)[::-1]
    assert abs(float(vals["tau0"]) - tau[0]) < 1e-12 * tau[0]
    assert abs(float(vals["taulast"]) - tau[-1]) < 1e-12 * tau[0]
    assert float(vals["res"]) < 1e-12
    assert float(vals["td2_relerr"]) < 1e-12
    assert int(vals["launches"]) > 0
    # em_sygv_range: both column shards equal the full solve's columns (em_info: one-stage)
    assert float(vals["shard_err"]) < 1e-12
    assert int(vals["path"]) == 1
