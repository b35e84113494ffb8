"""The distributed band reduction (csrc/sytrd2.cu sy2sb with a communicator: columns owned
in 64-column blocks round-robin, panel broadcasts, all-reduced partial symmetric products,
owner-only trailing updates) in TWO and THREE processes, every rank on cuda:0 (this run has
one GPU, which NCCL refuses for several ranks: the callback backend carries the collectives
through torch.distributed / gloo, staged on the host, so no kernel of one rank waits on
another). Every rank must end with the eigenvalues and eigenvectors of the single-process
solve; the reference's distributed run is ScaLAPACK PDSYGVX.
The NCCL backend itself is exercised with a one-rank communicator."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(n):
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    return b + b.T


def _rank_main(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import parallel
    from tests.test_gpu_sytrd_variants import _syev
    info = parallel.attach_communicator(dist)
    assert info["nranks"] == world and info["rank"] == rank and info["backend"] == "callbacks"
    nat.set_two_stage_min(0)
    w, u = _syev(_matrix(n))
    after = parallel.communicator_info()
    torch.cuda.synchronize()
    np.savez(f"{out}.{rank}.npz", w=w, u=u, allreduces=after["allreduces"],
             broadcasts=after["broadcasts"], bytes=after["bytes"])
    parallel.detach_communicator()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1536), (3, 1346), (2, 2050)])
def test_distributed_band_reduction_equals_single_rank(tmp_path, world, n):
    import torch.multiprocessing as mp
    from paper_2407_11993_b200 import _native as nat
    from tests.test_gpu_sytrd_variants import _syev
    out = str(tmp_path / "r")
    mp.spawn(_rank_main, args=(world, _free_port(), n, out), nprocs=world, join=True)
    res = [np.load(f"{out}.{r}.npz") for r in range(world)]
    a = _matrix(n)
    nat.set_two_stage_min(0)
    try:
        w1, u1 = _syev(a)
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    scale = np.abs(ref).max()
    from paper_2407_11993_b200 import parallel
    want = parallel.band_reduction_collectives(n, world)
    for r in res:
        # one broadcast per panel + the last columns, one all-reduce per panel
        assert int(r["broadcasts"]) == want["broadcasts"]
        assert int(r["allreduces"]) == want["allreduces"]
        assert int(r["bytes"]) == want["bytes"]
        assert np.max(np.abs(r["w"] - ref)) < 1e-12 * scale * n
        assert np.max(np.abs(r["w"] - w1)) < 1e-12 * scale * n
        u = r["u"]
        assert np.max(np.abs(u.T @ u - np.eye(n))) < 1e-12 * n
        assert np.max(np.abs(a @ u - u * r["w"])) < 1e-11 * scale * n
    # every rank reduced the same band: identical spectra and vectors across ranks
    for r in res[1:]:
        np.testing.assert_array_equal(r["w"], res[0]["w"])
        np.testing.assert_array_equal(r["u"], res[0]["u"])


def test_nccl_backend_single_rank_communicator():
    """em_comm_unique_id / em_comm_init_nccl load NCCL at run time and build a communicator
    (one rank: this box has one GPU); the eigensolve runs unchanged under it."""
    import ctypes
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import parallel
    from tests.test_gpu_sytrd_variants import _syev
    lib, ctx = nat.load_library(), nat.context()
    uid = ctypes.create_string_buffer(128)
    nat.check(lib.em_comm_unique_id(ctx, uid), "em_comm_unique_id")
    assert any(uid.raw)
    nat.check(lib.em_comm_init_nccl(ctx, 1, 0, uid), "em_comm_init_nccl")
    try:
        info = parallel.communicator_info()
        assert info == {"nranks": 1, "rank": 0, "backend": "nccl", "allreduces": 0,
                        "broadcasts": 0, "bytes": 0}
        a = _matrix(300)
        w, _ = _syev(a)
        assert np.max(np.abs(w - np.sort(np.linalg.eigvalsh(a))[::-1])) < 1e-10
    finally:
        parallel.detach_communicator()
    assert parallel.communicator_info()["backend"] == "none"


def _rank_sharded(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import linalg, parallel
    from paper_2407_11993_b200.synth import plate_model
    m = plate_model(20, 18, 4, n_ports=1, n_sources=1, n_obs=4)
    parallel.attach_communicator(dist)
    nat.set_two_stage_min(0)
    sb = parallel.sharded_generalized_eig(linalg.SymMatrix(m["l_i"]), linalg.SymMatrix(m["r_i"]),
                                          dist)
    info = parallel.communicator_info()
    torch.cuda.synchronize()
    np.savez(f"{out}.{rank}.npz", tau=sb.tau, lo=sb.lo, hi=sb.hi, l_n=sb.l_n, r_n=sb.r_n,
             v=sb.v_dev.cpu().numpy(), allreduces=info["allreduces"])
    parallel.detach_communicator()
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_generalized_eig_over_distributed_reduction(tmp_path):
    """The whole multi-GPU eigensolve path on a plate pencil (N = 1,440): distributed band
    reduction + column-restricted divide and conquer + column-sharded back-transforms; the
    two ranks' mode ranges tile the single-process solve (modal.generalized_eig,
    reference modal.py:46-81): tau < 1e-10 relative, and L v = tau R v for every column."""
    import torch.multiprocessing as mp
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import linalg, modal
    from paper_2407_11993_b200.synth import plate_model
    world = 2
    out = str(tmp_path / "r")
    mp.spawn(_rank_sharded, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [np.load(f"{out}.{r}.npz") for r in range(world)]
    m = plate_model(20, 18, 4, n_ports=1, n_sources=1, n_obs=4)
    n = m["l_i"].shape[0]
    nat.set_two_stage_min(0)
    try:
        basis = modal.generalized_eig(linalg.SymMatrix(m["l_i"]), linalg.SymMatrix(m["r_i"]))
    finally:
        nat.set_two_stage_min(nat.TWO_STAGE_MIN_DEFAULT)
    assert res[0]["lo"] == 0 and res[0]["hi"] == res[1]["lo"] and res[1]["hi"] == n
    for r in res:
        assert int(r["allreduces"]) == (n - 1) // 64
        lo, hi = int(r["lo"]), int(r["hi"])
        assert np.max(np.abs(r["tau"] - basis.tau) / basis.tau) < 1e-10
        assert np.max(np.abs(r["l_n"] - basis.l_n[lo:hi]) / basis.l_n[lo:hi]) < 1e-9
        v = r["v"].T                                   # (n, n_local), column-major on device
        resid = m["l_i"] @ v - (m["r_i"] @ v) * r["tau"][lo:hi]
        scale = np.linalg.norm(m["l_i"], 2)
        assert np.max(np.linalg.norm(resid, axis=0) / np.linalg.norm(v, axis=0)) < 1e-10 * scale
