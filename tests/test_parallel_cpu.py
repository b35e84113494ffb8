"""Multi-rank host logic of the mode-sharded TD2 stepping (paper_2407_11993_b200.parallel),
run on CPU with the gloo backend and world_size 2. Each rank integrates only its
own mode range (here with the CPU oracle standing in for the device scan), the
partial observables are summed with the same reduce_partials the device path
uses, and the result must equal the unsharded run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import golden, rel_l2


def test_shard_ranges_cover_and_balance():
    from paper_2407_11993_b200.parallel import shard_ranges, time_blocks
    for n in (1, 7, 96, 16384, 120000):
        for world in (1, 2, 3, 4, 8):
            r = shard_ranges(n, world)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in r]
            assert max(sizes) - min(sizes) <= 1
    tb = time_blocks(10000, 2048)
    assert tb[0] == (0, 2048) and tb[-1] == (8192, 10000)
    assert sum(k1 - k0 for k0, k1 in tb) == 10000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_observables(lo, hi, block):
    """Per-rank partial C V[:, lo:hi] Q[lo:hi] of the plate_small TD2 run, produced
    block by block (carry state kept across blocks) like ShardedTd2.run."""
    from oracle import oracle as O
    from paper_2407_11993_b200.parallel import time_blocks
    g = golden("plate_small")
    b = O.Basis(v=g["v"], tau=g["tau"], l_n=g["l_n"], r_n=g["r_n"], vt_r=None)
    dt, steps = float(g["dt"]), int(g["steps"])
    sd = O.tone_sampler([[(0.7, 2e4, 0.3), (0.2, 5e4, 1.1)]])
    s0 = O.tone_sampler([[(1.0, 1e4, 0.0)]])
    itab, i0tab = O.sample_table(sd, steps, dt), O.sample_table(s0, steps, dt)
    st = O.Td2(b, g["r_d"], g["l_d"], g["m0"], dt, 0.5)
    cv = g["c"] @ g["v"]
    q = np.zeros(b.tau.shape[0])
    y = np.zeros((steps, g["c"].shape[0]))
    for k0, k1 in time_blocks(steps, block):
        for k in range(k0, k1):
            f = st.forcing(itab[k], itab[k + 1] - itab[k], i0tab[k + 1] - i0tab[k])
            # only the owned modes advance (the others are never read)
            qn = q.copy()
            O.lib().orc_td2_step(O._p(qn), O._p(st._rn), O._p(st._c), dt,
                                 O._p(np.ascontiguousarray(f)), qn.shape[0])
            q[lo:hi] = qn[lo:hi]
            y[k] = cv[:, lo:hi] @ q[lo:hi]
    return y


def _worker(rank, world, port, block, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11993_b200.parallel import reduce_partials, shard_ranges
    g = golden("plate_small")
    lo, hi = shard_ranges(g["v"].shape[1], world)[rank]
    part = torch.from_numpy(_partial_observables(lo, hi, block))
    reduce_partials(part, dist)
    if rank == 0:
        np.save(out, part.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("block", [64, 300])
def test_sharded_td2_observables_equal_unsharded(tmp_path, block):
    world = 2
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(world, _free_port(), block, out), nprocs=world, join=True)
    y = np.load(out)
    g = golden("plate_small")
    ref = g["td2_obs_theta0.5"]
    assert rel_l2(y, ref) < 1e-12


def _partial_sweep(lo, hi, block):
    """Per-rank partial sweep (each drive channel alone) of the plate_small TD2 run over
    modes [lo, hi), block by block with the per-channel carry states (ShardedTd2.run_sweep)."""
    from oracle import oracle as O
    from paper_2407_11993_b200.parallel import time_blocks
    g = golden("plate_small")
    b = O.Basis(v=g["v"], tau=g["tau"], l_n=g["l_n"], r_n=g["r_n"], vt_r=None)
    dt, steps = float(g["dt"]), int(g["steps"])
    sd = O.tone_sampler([[(0.7, 2e4, 0.3), (0.2, 5e4, 1.1)]])
    s0 = O.tone_sampler([[(1.0, 1e4, 0.0)]])
    itab, i0tab = O.sample_table(sd, steps, dt), O.sample_table(s0, steps, dt)
    st = O.Td2(b, g["r_d"], g["l_d"], g["m0"], dt, 0.5)
    cv = g["c"] @ g["v"]
    y = np.zeros((2, steps, g["c"].shape[0]))
    for ch in range(2):
        it = itab if ch == 0 else 0 * itab
        i0 = i0tab if ch == 1 else 0 * i0tab
        q = np.zeros(b.tau.shape[0])
        for k0, k1 in time_blocks(steps, block):
            for k in range(k0, k1):
                f = st.forcing(it[k], it[k + 1] - it[k], i0[k + 1] - i0[k])
                qn = q.copy()
                O.lib().orc_td2_step(O._p(qn), O._p(st._rn), O._p(st._c), dt,
                                     O._p(np.ascontiguousarray(f)), qn.shape[0])
                q[lo:hi] = qn[lo:hi]
                y[ch, k] = cv[:, lo:hi] @ q[lo:hi]
    return y


def _sweep_worker(rank, world, port, block, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11993_b200.parallel import reduce_partials, shard_ranges
    g = golden("plate_small")
    lo, hi = shard_ranges(g["v"].shape[1], world)[rank]
    part = torch.from_numpy(_partial_sweep(lo, hi, block))
    reduce_partials(part, dist)
    if rank == 0:
        np.save(out, part.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sweep_sums_to_the_reference_run(tmp_path):
    """The C5 layout: sweep channels x sharded modes, one all-reduce of the partial
    per-channel observables; the channels then superpose to the reference trajectory."""
    world = 2
    out = str(tmp_path / "ys.npy")
    mp.spawn(_sweep_worker, args=(world, _free_port(), 128, out), nprocs=world, join=True)
    y = np.load(out)
    g = golden("plate_small")
    assert y.shape[0] == 2
    assert rel_l2(y.sum(axis=0), g["td2_obs_theta0.5"]) < 1e-12


def test_band_reduction_partition_host_logic():
    """The distributed band reduction's partition (csrc/sytrd2.cu) as the host sees it:
    64-column blocks dealt round-robin, and the collective counts / bytes communicator_info()
    reports per eigensolve (the GPU tests compare the library's counters with these)."""
    from paper_2407_11993_b200 import parallel
    assert [parallel.band_block_owner(c, 3) for c in (0, 63, 64, 127, 128, 191, 192)] == \
        [0, 0, 1, 1, 2, 2, 0]
    # every rank owns the same number of blocks up to one (balance of the shrinking matrix)
    for world in (2, 3, 8):
        for n in (1346, 1536, 50000):
            blocks = [parallel.band_block_owner(c, world) for c in range(0, n, 64)]
            counts = [blocks.count(r) for r in range(world)]
            assert max(counts) - min(counts) <= 1
    c = parallel.band_reduction_collectives(1536, 2)
    assert c["broadcasts"] == 24 and c["allreduces"] == 23
    assert parallel.band_reduction_collectives(1536, 1) == {"broadcasts": 0, "allreduces": 0,
                                                            "bytes": 0}
    # C3: 781 panels, ~10 GB of broadcasts + ~20 GB of all-reduced partials
    c3 = parallel.band_reduction_collectives(50000, 8)
    assert c3["allreduces"] == 781 and 29e9 < c3["bytes"] < 31e9
    with pytest.raises(ValueError):
        parallel.band_block_owner(5, 0)
