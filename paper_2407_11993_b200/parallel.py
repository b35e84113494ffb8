"""Multi-GPU modal solve: column-sharded eigensolve + mode-sharded stepping
(north-star (a) and (b)).

Eigensolve (`sharded_generalized_eig`, em_sygv_range): every rank reduces the pencil
to tridiagonal form and solves it (Cholesky of R, two-sided reduction, tridiagonalisation,
divide and conquer: replicated), then back-transforms ONLY the eigenvector columns of its
own contiguous mode range (Q2, Q1, G^-T: 2/3 of the eigensolve's flops at C3) and forms
their sign fix, l_n and r_n. The ranks exchange nothing: rank r's columns are exactly the
modes its stepping shard owns, so V is never gathered.

After the eigensolve the modes never interact (transient.py:116-166: every
mode's update uses only its own r_n, c_n and forcing row), so the TD2 stepping
shards naturally: rank r owns a contiguous range of modes, integrates them with
its own fused scan (em_td2_run) and produces PARTIAL observables
Y_r = (C V)[:, modes_r] Q_r. The only exchange is one all-reduce (sum) of the
partial observables per time block; it runs on a side stream overlapped with
the next block's scan. One process per GPU, torch.distributed (NCCL on GPUs,
gloo for the CPU tests).

`ShardedTd2` is the device path. `shard_ranges` / `reduce_partials` are the
pure host logic, shared with the CPU tests (tests/test_parallel_cpu.py), where
the per-rank partial observables are produced by a test-side executor.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import linalg
from .errors import DimensionMismatch, NotPositiveDefinite


# ---- the library's own communicator (distributed band reduction) -----------------------
_ALLREDUCE_T = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
_BCAST_T = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_int)
_comm_keepalive: list = []


class _DevView:
    """Zero-copy view of `count` doubles at a device address (for torch.as_tensor)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 2}


def attach_communicator(dist, backend: str | None = None) -> dict:
    """Give the library a communicator over the ranks of `dist` (torch.distributed), so the
    band reduction of every eigensolve on this context is distributed (csrc/sytrd2.cu).

    backend "nccl": the library's own NCCL communicator on the context stream — rank 0's
    ncclUniqueId is handed out through torch.distributed, the data path never touches
    torch. backend "callbacks": collectives through torch.distributed itself (gloo in the
    tests, where several ranks share one GPU, which NCCL refuses). Default: "nccl" when
    torch.distributed runs on NCCL, else "callbacks". Returns communicator_info()."""
    t = nat.torch()
    lib, ctx = nat.load_library(), nat.context()
    world, rank = _world_rank(dist)
    if world <= 1:
        nat.check(lib.em_comm_destroy(ctx), "em_comm_destroy")
        return communicator_info()
    if backend is None:
        backend = "nccl" if dist.get_backend() == "nccl" else "callbacks"
    if backend == "nccl":
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            nat.check(lib.em_comm_unique_id(ctx, uid), "em_comm_unique_id")
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0)
        uid = ctypes.create_string_buffer(box[0], 128)
        nat.check(lib.em_comm_init_nccl(ctx, world, rank, uid), "em_comm_init_nccl")
    elif backend == "callbacks":
        def _allreduce(_user, ptr, count):
            try:
                buf = t.as_tensor(_DevView(ptr, count), device="cuda")
                dist.all_reduce(buf)
                t.cuda.synchronize()
                return 0
            except Exception:  # noqa: BLE001 (reported through the status code)
                return 1

        def _bcast(_user, ptr, count, root):
            try:
                buf = t.as_tensor(_DevView(ptr, count), device="cuda")
                dist.broadcast(buf, src=root)
                t.cuda.synchronize()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cbs = (_ALLREDUCE_T(_allreduce), _BCAST_T(_bcast))
        _comm_keepalive[:] = [cbs]
        nat.check(lib.em_comm_init_callbacks(ctx, world, rank,
                                             ctypes.cast(cbs[0], ctypes.c_void_p),
                                             ctypes.cast(cbs[1], ctypes.c_void_p), None),
                  "em_comm_init_callbacks")
    else:
        raise ValueError(f"unknown communicator backend {backend!r}")
    return communicator_info()


def detach_communicator() -> None:
    nat.check(nat.load_library().em_comm_destroy(nat.context()), "em_comm_destroy")
    _comm_keepalive.clear()


def communicator_info() -> dict:
    info = (ctypes.c_int64 * 6)()
    nat.check(nat.load_library().em_comm_info(nat.context(), info), "em_comm_info")
    return {"nranks": info[0], "rank": info[1],
            "backend": ("none", "nccl", "callbacks")[info[2]], "allreduces": info[3],
            "broadcasts": info[4], "bytes": info[5]}


BAND_BLOCK = 64  # columns per ownership block of the distributed band reduction (= its band)


def band_block_owner(col: int, world: int) -> int:
    """Rank owning global column `col` of the trailing matrix in the distributed band
    reduction (csrc/sytrd2.cu): 64-column blocks dealt round-robin."""
    if world < 1 or col < 0:
        raise ValueError("world size must be >= 1 and the column non-negative")
    return (col // BAND_BLOCK) % world


def band_reduction_collectives(n: int, world: int) -> dict:
    """Collectives the distributed band reduction of an order-n matrix issues per eigensolve
    (what communicator_info() counts): one broadcast per 64-column panel (its finished
    columns from the diagonal block down, plus tau) and one for the columns right of the
    last panel; one all-reduce of the n x 64 partial symmetric product per panel."""
    if world <= 1 or n <= BAND_BLOCK:
        return {"broadcasts": 0, "allreduces": 0, "bytes": 0}
    panels = (n - 1) // BAND_BLOCK
    last = panels * BAND_BLOCK                      # first column right of the last panel
    bcast = sum((n - k * BAND_BLOCK) * BAND_BLOCK + BAND_BLOCK for k in range(panels))
    bcast += (n - last) ** 2
    widths = [min(BAND_BLOCK, n - (k + 1) * BAND_BLOCK) for k in range(panels)]
    allred = sum(n * w for w in widths)
    return {"broadcasts": panels + 1, "allreduces": panels, "bytes": 8 * (bcast + allred)}


def shard_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced mode ranges [lo, hi) per rank (sizes differ by <= 1)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def time_blocks(steps: int, block: int) -> list[tuple[int, int]]:
    """[k0, k1) step ranges of the per-block exchange."""
    return [(k, min(k + block, steps)) for k in range(0, steps, block)]


def reduce_partials(partial, dist, group=None):
    """Sum partial observables over all ranks in place (fixed reduction order by
    the collective; deterministic for a fixed world size)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


def _world_rank(dist):
    if dist is not None and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


class ShardBasis:
    """One rank's share of a column-sharded ModalBasis (modal.py:22-43): time constants
    of ALL modes (descending), the rank's mode range [lo, hi), its eigenvector columns
    V[:, lo:hi] on the device (v_dev: torch (hi - lo, N) = column-major N x (hi - lo)),
    and l_n, r_n of its modes."""

    def __init__(self, tau, lo: int, hi: int, v_dev, l_n, r_n):
        self.tau = np.asarray(tau, dtype=float)
        self.lo, self.hi = int(lo), int(hi)
        self.v_dev = v_dev
        self.l_n = np.asarray(l_n, dtype=float)
        self.r_n = np.asarray(r_n, dtype=float)

    @property
    def n_modes(self) -> int:
        return self.tau.shape[0]

    @property
    def n_local(self) -> int:
        return self.hi - self.lo


def sharded_generalized_eig(l_i, r_i, dist=None, mode_range: tuple[int, int] | None = None
                            ) -> ShardBasis:
    """This rank's share of generalized_eig (modal.py:46-81): modes shard_ranges(N,
    world)[rank] (or mode_range). Inputs as modal.generalized_eig (host SymMatrix / numpy,
    or device tensors); raises NotPositiveDefinite with the reference's `what` strings."""
    t = nat.torch()
    if isinstance(l_i, t.Tensor) and isinstance(r_i, t.Tensor):
        ld = l_i.to(dtype=t.float64).contiguous()
        rd = r_i.to(dtype=t.float64).contiguous()
        own = False
    else:
        lm = l_i.full if isinstance(l_i, linalg.SymMatrix) else np.asarray(l_i, dtype=float)
        rm = r_i.full if isinstance(r_i, linalg.SymMatrix) else np.asarray(r_i, dtype=float)
        if lm.shape != rm.shape:
            raise DimensionMismatch("L_i and R_i must have the same shape")
        ld = nat.device_symmetric(lm) if isinstance(l_i, linalg.SymMatrix) else \
            nat.device_colmajor(lm)
        rd = nat.device_symmetric(rm) if isinstance(r_i, linalg.SymMatrix) else \
            nat.device_colmajor(rm)
        own = True
    if ld.shape != rd.shape:
        raise DimensionMismatch("L_i and R_i must have the same shape")
    n = ld.shape[0]
    world, rank = _world_rank(dist)
    lo, hi = mode_range if mode_range is not None else shard_ranges(n, world)[rank]
    m = hi - lo
    tau = nat.empty(max(n, 1))
    v = nat.empty(max(m, 1), n)
    ln, rn = nat.empty(max(m, 1)), nat.empty(max(m, 1))
    piv, which = ctypes.c_int64(-1), ctypes.c_int(-1)
    lib = nat.load_library()
    rc = lib.em_sygv_range(nat.context(), n, nat.ptr(ld), n, nat.ptr(rd), n, lo, hi,
                           nat.ptr(tau), nat.ptr(v), n, nat.ptr(ln), nat.ptr(rn), None, n,
                           1 if own else 0, ctypes.byref(piv), ctypes.byref(which))
    if rc == nat.EM_ERR_NOT_PD:
        what = "modal resistance matrix" if which.value == 0 else "modal inductance matrix"
        raise NotPositiveDefinite(int(piv.value), what)
    nat.check(rc, "em_sygv_range")
    return ShardBasis(tau.cpu().numpy()[:n], lo, hi, v[:m], ln.cpu().numpy()[:m],
                      rn.cpu().numpy()[:m])


class ShardedTd2:
    """TD2 stepping of the modes [lo, hi) owned by this rank.

    basis: ModalBasis (device V, all modes) or this rank's ShardBasis (its columns only);
    rm: ReducedModel; observables C (n_obs x N). run(drive_table (T+1 x n_c), steps) ->
    full observables (T x n_obs) on every rank (partials all-reduced per time block of
    `block` steps)."""

    def __init__(self, rm, basis, dt: float, theta: float, c_obs: np.ndarray, dist=None,
                 block: int = 2048, mode_range: tuple[int, int] | None = None):
        t = nat.torch()
        self.dist = dist
        world = dist.get_world_size() if (dist is not None and dist.is_initialized()) else 1
        rank = dist.get_rank() if world > 1 else 0
        n = basis.n_modes
        if isinstance(basis, ShardBasis):
            self.lo, self.hi = basis.lo, basis.hi
            v_loc = basis.v_dev                           # this rank's columns (n x n_loc)
            ln_loc, rn_loc = basis.l_n, basis.r_n
        else:
            # mode_range overrides the rank's shard (single-process emulation in tests)
            self.lo, self.hi = mode_range if mode_range is not None else \
                shard_ranges(n, world)[rank]
            v_loc = basis.v_dev[self.lo:self.hi]          # columns lo..hi of V (n x n_loc)
            ln_loc, rn_loc = basis.l_n[self.lo:self.hi], basis.r_n[self.lo:self.hi]
        self.n_loc = self.hi - self.lo
        self.block = block
        self.n_p, self.n_s = rm.n_ports, rm.n_sources
        nd = 2 * self.n_p + self.n_s
        ctx, lib = nat.context(), nat.load_library()
        # P_loc = V[:, lo:hi]^T [R_D | L_D | M0]  (n_loc x nd)
        if nd:
            drv = np.concatenate([rm.r_d.reshape(n, self.n_p), rm.l_d.reshape(n, self.n_p),
                                  rm.m0.reshape(n, self.n_s)], axis=1)
            ddrv = nat.device_colmajor(drv)
            self.proj = nat.empty(nd, self.n_loc)
            nat.check(lib.em_dgemm(ctx, 1, 0, self.n_loc, nd, n, 1.0, nat.ptr(v_loc), n,
                                   nat.ptr(ddrv), n, 0.0, nat.ptr(self.proj), self.n_loc),
                      "em_dgemm")
        else:
            self.proj = nat.zeros(1, max(self.n_loc, 1))
        # CV_loc = C V[:, lo:hi]  (n_obs x n_loc)
        c = np.atleast_2d(np.asarray(c_obs, dtype=float))
        self.n_obs = c.shape[0]
        cd = nat.device_colmajor(c)
        self.cv = nat.empty(self.n_loc, self.n_obs)
        nat.check(lib.em_dgemm(ctx, 0, 0, self.n_obs, self.n_loc, n, 1.0, nat.ptr(cd), self.n_obs,
                               nat.ptr(v_loc), n, 0.0, nat.ptr(self.cv), self.n_obs), "em_dgemm")
        self.ln = nat.device_vector(ln_loc)
        self.rn = nat.device_vector(rn_loc)
        p_r = self.proj[0:self.n_p] if self.n_p else self.proj[0:1]
        p_l = self.proj[self.n_p:2 * self.n_p] if self.n_p else self.proj[0:1]
        p_m = self.proj[2 * self.n_p:] if self.n_s else self.proj[0:1]
        plan = ctypes.c_void_p()
        nat.check(lib.em_td2_plan_create(ctx, self.n_loc, self.n_p, self.n_s, nat.ptr(self.ln),
                                         nat.ptr(self.rn), nat.ptr(p_r), nat.ptr(p_l),
                                         nat.ptr(p_m), float(dt), float(theta),
                                         ctypes.byref(plan)), "em_td2_plan_create")
        self._plan = plan
        nat.check(lib.em_td2_set_observables(plan, self.n_obs, nat.ptr(self.cv), self.n_obs, None,
                                             0), "em_td2_set_observables")
        self.q = nat.zeros(max(self.n_loc, 1))
        self.q_sweep = None
        self._comm_stream = t.cuda.Stream()

    def __del__(self):
        if getattr(self, "_plan", None):
            nat.load_library().em_td2_plan_destroy(self._plan)
            self._plan = None

    def run(self, drive_dev, steps: int):
        """drive_dev: device drive table ((steps+1) x (n_p+n_s)). Returns Y (steps x n_obs)."""
        t = nat.torch()
        lib = nat.load_library()
        n_c = self.n_p + self.n_s
        y = nat.zeros(steps, self.n_obs)
        main = t.cuda.current_stream()
        pending = []
        for k0, k1 in time_blocks(steps, self.block):
            yb = y[k0:k1]
            # the carry state q advances block by block; the drive rows k0..k1 are a view
            dptr = nat.ptr(drive_dev[k0 * n_c:]) if n_c else nat.ptr(drive_dev)
            nat.check(lib.em_td2_run(self._plan, k1 - k0, dptr, nat.ptr(self.q), nat.ptr(yb), 1,
                                     None), "em_td2_run")
            if self.dist is not None and self.dist.is_initialized() and \
                    self.dist.get_world_size() > 1:
                ev = t.cuda.Event()
                ev.record(main)
                with t.cuda.stream(self._comm_stream):
                    self._comm_stream.wait_event(ev)
                    pending.append(self.dist.all_reduce(yb, op=self.dist.ReduceOp.SUM,
                                                        async_op=True))
        for h in pending:
            h.wait()
        main.wait_stream(self._comm_stream)
        return y

    def run_sweep(self, drive_dev, steps: int):
        """Excitation sweep over this rank's modes (BASELINE configs[4]: 64 right-hand
        sides, modes sharded across GPUs): every drive channel integrated alone
        (em_td2_run_sweep); the partial observables (n_c x block x n_obs) are summed over
        ranks once per time block. Returns Y (n_c, steps, n_obs) on every rank."""
        t = nat.torch()
        lib = nat.load_library()
        n_c = self.n_p + self.n_s
        if self.q_sweep is None:
            self.q_sweep = nat.zeros(n_c, max(self.n_loc, 1))
        y = nat.zeros(n_c, steps, self.n_obs)
        main = t.cuda.current_stream()
        pending = []
        for k0, k1 in time_blocks(steps, self.block):
            yb = nat.empty(n_c, k1 - k0, self.n_obs)
            nat.check(lib.em_td2_run_sweep(self._plan, k1 - k0, nat.ptr(drive_dev[k0 * n_c:]),
                                           nat.ptr(self.q_sweep), nat.ptr(yb), 1),
                      "em_td2_run_sweep")
            if self.dist is not None and self.dist.is_initialized() and \
                    self.dist.get_world_size() > 1:
                ev = t.cuda.Event()
                ev.record(main)
                with t.cuda.stream(self._comm_stream):
                    self._comm_stream.wait_event(ev)
                    pending.append((self.dist.all_reduce(yb, op=self.dist.ReduceOp.SUM,
                                                         async_op=True), yb, k0, k1))
            else:
                y[:, k0:k1] = yb
        for h, yb, k0, k1 in pending:
            h.wait()
        main.wait_stream(self._comm_stream)
        for _, yb, k0, k1 in pending:
            y[:, k0:k1] = yb
        return y
