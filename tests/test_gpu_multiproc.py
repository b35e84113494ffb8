"""The multi-GPU product path end to end in TWO processes (world size 2, gloo over
127.0.0.1), both ranks on cuda:0 (this run has one GPU; gloo reduces on the host, so no
kernel of one rank waits on the other's): each rank solves its column shard of the
generalized eigenproblem (parallel.sharded_generalized_eig -> em_sygv_range), builds its
ShardedTd2 from its own columns and integrates its modes; the partial observables are
all-reduced per time block. The gathered result must equal the single-process solve
(modal.generalized_eig + Td2Stepper, the reference's API) and the reference's own golden
trajectory. Covers ShardedTd2.run and .run_sweep (the C5 layout)."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _drive_table(g, n_p, n_s):
    from oracle import oracle as O
    dt, steps = float(g["dt"]), int(g["steps"])
    sd = O.tone_sampler([[(0.7, 2e4, 0.3), (0.2, 5e4, 1.1)]])
    s0 = O.tone_sampler([[(1.0, 1e4, 0.0)]])
    return np.ascontiguousarray(np.concatenate([O.sample_table(sd, steps, dt),
                                                O.sample_table(s0, steps, dt)], axis=1))


def _rank_main(rank, world, port, name, block, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11993_b200 import _native as nat
    from paper_2407_11993_b200 import parallel, reduction
    g = golden(name)
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], g["m0"],
                               port_names=("p0",), source_names=("s0",))
    sb = parallel.sharded_generalized_eig(rm.l_i, rm.r_i, dist)
    st = parallel.ShardedTd2(rm, sb, float(g["dt"]), 0.5, g["c"], dist=dist, block=block)
    tab = nat.device_vector(_drive_table(g, 1, 1).reshape(-1))
    y = st.run(tab, int(g["steps"]))
    ys = st.run_sweep(tab, int(g["steps"]))
    torch.cuda.synchronize()
    np.savez(f"{out}.{rank}.npz", y=y.cpu().numpy(), ys=ys.cpu().numpy(), tau=sb.tau,
             lo=sb.lo, hi=sb.hi, l_n=sb.l_n, r_n=sb.r_n)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,block", [("plate_small", 64), ("plate_200", 300)])
def test_two_rank_sharded_solve_equals_single_device(tmp_path, name, block):
    import torch.multiprocessing as mp
    from paper_2407_11993_b200 import modal, reduction, transient
    world = 2
    out = str(tmp_path / "r")
    mp.spawn(_rank_main, args=(world, _free_port(), name, block, out), nprocs=world, join=True)
    res = [np.load(f"{out}.{r}.npz") for r in range(world)]
    g = golden(name)
    rm = reduction.from_blocks(g["r_i"], g["l_i"], g["r_d"], g["l_d"], g["m0"],
                               port_names=("p0",), source_names=("s0",))
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    n = basis.n_modes
    # the shards tile the modes; tau is replicated; l_n, r_n are the single solve's
    assert res[0]["lo"] == 0 and res[0]["hi"] == res[1]["lo"] and res[1]["hi"] == n
    for r in res:
        np.testing.assert_array_equal(r["tau"], basis.tau)
        lo, hi = int(r["lo"]), int(r["hi"])
        assert np.max(np.abs(r["l_n"] - basis.l_n[lo:hi]) / basis.l_n[lo:hi]) < 1e-12
        assert np.max(np.abs(r["r_n"] - basis.r_n[lo:hi])) < 1e-12
    # every rank holds the all-reduced observables
    np.testing.assert_array_equal(res[0]["y"], res[1]["y"])
    i_d, i0 = _drive_table(g, 1, 1)[:, :1], _drive_table(g, 1, 1)[:, 1:]
    _, y1, _ = transient.Td2Stepper(rm, basis, float(g["dt"]), 0.5).run(
        i_d, i0, capture_state=False, observables=(g["c"], None))
    assert rel_l2(res[0]["y"], y1) < 1e-12
    # and the reference's own run_transient trajectory (golden) to the north-star tolerance
    assert rel_l2(res[0]["y"], g["td2_obs_theta0.5"]) < 1e-8
    # the sweep: one trajectory per drive channel, summing to the superposed run
    ys = res[0]["ys"]
    assert ys.shape[0] == 2 and rel_l2(ys.sum(axis=0), y1) < 1e-12
