"""Seeded synthetic conducting plates (the BASELINE.json configs).

The reference's own inputs come from a filament-network front end
(pkg/src/eddymodes/assembly.py, network.py) that is out of scope here; the
paper's 100,676-DOF tube mesh is not available. These plates stand in for it,
following SURVEY.md §8(d):

* grid nx*ny*nz voxels of edge h, C-order index i = (ix*ny + iy)*nz + iz,
  centroid x_i = (ix+1/2, iy+1/2, iz+1/2) h;
* R = rho*K7 + 1e-3*I (K7: 6 on the diagonal, -1 per face neighbour);
* L_ij = 1e-7 (a_i . a_j) / (|x_i - x_j| + h/2), a_i = (cos t_i, sin t_i, 0),
  t_i ~ U[0, 2pi) seeded (SPD by Schoenberg + Schur);
* one SeedSequence child stream each for the angles, source profiles,
  observables, notch and batched-source tones.

The generator is shared by the CPU oracle, the tests and the benchmark so
every path sees bit-identical inputs. It builds numpy arrays; the big
configurations are generated in row chunks.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MU0_4PI = 1e-7
RHO = 1.7e-8
R_SHIFT = 1e-3
DEFAULT_SEED = 20240807

# child-stream slots of SeedSequence(seed).spawn(5)
_ANGLES, _SOURCES, _OBS, _NOTCH, _TONES = range(5)


@dataclass
class Plate:
    nx: int
    ny: int
    nz: int
    h: float = 1e-3
    seed: int = DEFAULT_SEED
    notch: bool = False
    keep: np.ndarray = field(default=None, repr=False)   # voxel ids kept (after notch)

    def __post_init__(self):
        n_all = self.nx * self.ny * self.nz
        keep = np.arange(n_all)
        if self.notch:
            rng = self.rng(_NOTCH)
            # a 2-voxel-wide slot along y through all iz at a seeded x position
            ix0 = int(rng.integers(self.nx // 4, 3 * self.nx // 4))
            iy0 = int(rng.integers(self.ny // 4, self.ny // 2))
            ix, iy, _ = np.unravel_index(keep, (self.nx, self.ny, self.nz))
            slot = (ix >= ix0) & (ix < ix0 + 2) & (iy >= iy0) & (iy < iy0 + self.ny // 3)
            keep = keep[~slot]
        self.keep = keep

    @property
    def n(self) -> int:
        return int(self.keep.shape[0])

    def rng(self, slot: int) -> np.random.Generator:
        ss = np.random.SeedSequence(self.seed).spawn(5)[slot]
        return np.random.default_rng(ss)

    def centroids(self) -> np.ndarray:
        ix, iy, iz = np.unravel_index(self.keep, (self.nx, self.ny, self.nz))
        return (np.stack([ix, iy, iz], axis=1) + 0.5) * self.h

    def directions(self) -> np.ndarray:
        theta = self.rng(_ANGLES).uniform(0.0, 2 * np.pi, size=self.nx * self.ny * self.nz)
        theta = theta[self.keep]
        return np.stack([np.cos(theta), np.sin(theta), np.zeros_like(theta)], axis=1)

    # --- matrices -------------------------------------------------------------

    def resistance(self) -> np.ndarray:
        """Dense R = rho*K7 + 1e-3*I (stored dense, as the reference does)."""
        n = self.n
        r = np.zeros((n, n))
        pos = -np.ones(self.nx * self.ny * self.nz, dtype=np.int64)
        pos[self.keep] = np.arange(n)
        ix, iy, iz = np.unravel_index(self.keep, (self.nx, self.ny, self.nz))
        r[np.arange(n), np.arange(n)] = RHO * 6.0 + R_SHIFT
        for d, (sx, sy, sz) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
            jx, jy, jz = ix + sx, iy + sy, iz + sz
            ok = (jx < self.nx) & (jy < self.ny) & (jz < self.nz)
            j_all = np.ravel_multi_index((jx[ok], jy[ok], jz[ok]), (self.nx, self.ny, self.nz))
            jj = pos[j_all]
            ii = np.arange(n)[ok]
            m = jj >= 0
            r[ii[m], jj[m]] = -RHO
            r[jj[m], ii[m]] = -RHO
        return r

    def resistance_band(self) -> tuple[np.ndarray, int]:
        """R in LAPACK lower band storage, (bw + 1, N) with band[i - j, j] = R[i, j] for
        0 <= i - j <= bw — the same stencil as resistance(), without the N x N array."""
        n = self.n
        pos = -np.ones(self.nx * self.ny * self.nz, dtype=np.int64)
        pos[self.keep] = np.arange(n)
        ix, iy, iz = np.unravel_index(self.keep, (self.nx, self.ny, self.nz))
        pairs = []
        for sx, sy, sz in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
            jx, jy, jz = ix + sx, iy + sy, iz + sz
            ok = (jx < self.nx) & (jy < self.ny) & (jz < self.nz)
            j_all = np.ravel_multi_index((jx[ok], jy[ok], jz[ok]), (self.nx, self.ny, self.nz))
            jj = pos[j_all]
            ii = np.arange(n)[ok]
            m = jj >= 0
            pairs.append((ii[m], jj[m]))
        bw = max([int(np.max(np.abs(jj - ii))) for ii, jj in pairs if ii.size] or [0])
        band = np.zeros((bw + 1, n))
        band[0, :] = RHO * 6.0 + R_SHIFT
        for ii, jj in pairs:
            lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
            band[hi - lo, lo] = -RHO
        return band, bw

    def inductance(self, rows: slice | None = None) -> np.ndarray:
        """Dense L (or a row block of it)."""
        x = self.centroids()
        a = self.directions()
        rows = rows or slice(0, self.n)
        xr, ar = x[rows], a[rows]
        d = np.sqrt(((xr[:, None, :] - x[None, :, :]) ** 2).sum(-1))
        # elementwise (not BLAS) so the result does not depend on the BLAS thread count
        dot = ar[:, None, 0] * a[None, :, 0] + ar[:, None, 1] * a[None, :, 1]
        return MU0_4PI * dot / (d + self.h / 2)

    def inductance_full(self, chunk: int = 1024) -> np.ndarray:
        n = self.n
        out = np.empty((n, n))
        for s in range(0, n, chunk):
            out[s:s + chunk] = self.inductance(slice(s, min(s + chunk, n)))
        return out

    # --- couplings and observables -----------------------------------------

    def source_profiles(self, n_s: int) -> np.ndarray:
        """m0 columns ~ N(0,1) (induced-voltage spatial profiles)."""
        return self.rng(_SOURCES).standard_normal((self.n, n_s))

    def observables(self, n_obs: int) -> np.ndarray:
        """Dense pickup matrix C ~ N(0,1)/sqrt(N), shape (n_obs, N)."""
        return self.rng(_OBS).standard_normal((n_obs, self.n)) / np.sqrt(self.n)

    def port_columns(self, r: np.ndarray | None = None, chunk: int = 1024):
        """Electrode-path couplings for one port: the return path is a uniform
        x-directed current sheet of 1 A (s_j = 1/(ny*nz) per voxel).
        L_D[i] = 1e-7 sum_j (a_i.x) s_j / (r_ij + h/2);  R_D = (rho K7)((a.x) o s).
        """
        x = self.centroids()
        a = self.directions()
        s = 1.0 / (self.ny * self.nz)
        ax = a[:, 0]
        n = self.n
        l_d = np.empty(n)
        for st in range(0, n, chunk):
            sl = slice(st, min(st + chunk, n))
            d = np.sqrt(((x[sl, None, :] - x[None, :, :]) ** 2).sum(-1))
            l_d[sl] = MU0_4PI * ax[sl] * (s / (d + self.h / 2)).sum(axis=1)
        if r is None:
            r = self.resistance()
        k7rho = r - R_SHIFT * np.eye(n)
        r_d = k7rho @ (ax * s)
        return r_d[:, None], l_d[:, None]

    def tones(self, n_s: int, fmin: float = 1e3, fmax: float = 1e5):
        """Seeded log-uniform frequencies and uniform phases (batched sweep)."""
        rng = self.rng(_TONES)
        f = np.exp(rng.uniform(np.log(fmin), np.log(fmax), size=n_s))
        ph = rng.uniform(0.0, 2 * np.pi, size=n_s)
        return f, ph


# --- the BASELINE.json configurations ------------------------------------------

CONFIGS = {
    # name: (nx, ny, nz, extra)
    "C1": dict(grid=(40, 25, 2), theta=(0.5,), dt=1e-6, steps=2000, n_obs=16, n_ports=0,
               n_sources=1, drive="tone10k"),
    "C2": dict(grid=(64, 64, 4), theta=(1.0, 0.5), dt=5e-7, steps=10000, n_obs=32, n_ports=1,
               n_sources=0, drive="ramp5us"),
    "C3": dict(grid=(125, 100, 4), theta=(0.5,), dt=2e-7, steps=100000, n_obs=64, n_ports=1,
               n_sources=1, drive="tone50k"),
    "C4": dict(grid=(200, 150, 4), theta=(0.5,), dt=1e-7, steps=100000, n_obs=128, n_ports=1,
               n_sources=0, drive="trapezoid", notch=True),
    "C5": dict(grid=(150, 100, 4), theta=(0.5,), dt=2e-7, steps=100000, n_obs=64, n_ports=0,
               n_sources=64, drive="batched"),
}


def plate_model(nx: int, ny: int, nz: int, n_ports: int = 0, n_sources: int = 1,
                n_obs: int = 16, seed: int = DEFAULT_SEED, notch: bool = False,
                h: float = 1e-3) -> dict:
    """All inputs of one plate configuration as numpy arrays:
    r_i, l_i (N x N), r_d, l_d (N x n_ports), m0 (N x n_sources), c (n_obs x N)."""
    p = Plate(nx, ny, nz, h=h, seed=seed, notch=notch)
    r = p.resistance()
    l = p.inductance_full()
    if n_ports:
        r_d, l_d = p.port_columns(r)
    else:
        r_d = np.zeros((p.n, 0))
        l_d = np.zeros((p.n, 0))
    m0 = p.source_profiles(n_sources) if n_sources else np.zeros((p.n, 0))
    c = p.observables(n_obs)
    return dict(plate=p, r_i=r, l_i=l, r_d=r_d, l_d=l_d, m0=m0, c=c)


def device_plate_model(nx: int, ny: int, nz: int, n_ports: int = 0, n_sources: int = 1,
                       n_obs: int = 16, seed: int = DEFAULT_SEED, notch: bool = False,
                       h: float = 1e-3, r_dense: bool = True, ldl: int | None = None) -> dict:
    """plate_model with the O(N^2) parts generated on the device (em_synth_plate):
    l_i, r_i (torch, (N, N) symmetric), r_d, l_d (torch (n_ports, N) = column-major
    N x n_ports), plus host m0 (N x n_sources) and c (n_obs x N).
    r_dense=False: no dense R; r_band (torch (N, bw + 1) = column-major lower band storage)
    and r_bw instead (the N = 120,000 plate: L alone is 115 GB). ldl: L's leading dimension
    (torch (N, ldl)); a multiple of 32 lets the eigensolve reduce L in place."""
    from . import _native as nat
    p = Plate(nx, ny, nz, h=h, seed=seed, notch=notch)
    n = p.n
    theta = p.rng(_ANGLES).uniform(0.0, 2 * np.pi, size=nx * ny * nz)[p.keep]
    pos = -np.ones(nx * ny * nz, dtype=np.int64)
    pos[p.keep] = np.arange(n)
    t = nat.torch()
    keep_d = t.from_numpy(p.keep.astype(np.int64)).to("cuda")
    pos_d = t.from_numpy(pos).to("cuda")
    ang_d = nat.device_vector(theta)
    ldl = n if ldl is None else int(ldl)
    L = nat.empty(n, ldl)
    R = nat.empty(n, n) if r_dense else None
    ld = nat.zeros(max(n_ports, 1), n)
    rd = nat.zeros(max(n_ports, 1), n)
    lib = nat.load_library()
    nat.check(lib.em_synth_plate(nat.context(), nx, ny, nz, h, RHO, R_SHIFT, n, nat.ptr(keep_d),
                                 nat.ptr(pos_d), nat.ptr(ang_d), nat.ptr(L), ldl,
                                 nat.ptr(R) if R is not None else None, n,
                                 nat.ptr(ld) if n_ports else None,
                                 nat.ptr(rd) if n_ports else None), "em_synth_plate")
    m0 = p.source_profiles(n_sources) if n_sources else np.zeros((n, 0))
    c = p.observables(n_obs)
    out = dict(plate=p, l_i=L, r_i=R, l_d=ld[:n_ports], r_d=rd[:n_ports], m0=m0, c=c, ldl=ldl)

    def regen_l():
        """Regenerate L into out["l_i"] (after an in-place solve consumed it)."""
        nat.check(lib.em_synth_plate(nat.context(), nx, ny, nz, h, RHO, R_SHIFT, n,
                                     nat.ptr(keep_d), nat.ptr(pos_d), nat.ptr(ang_d),
                                     nat.ptr(out["l_i"]), ldl, None, n, None, None),
                  "em_synth_plate")
    out["regen_l"] = regen_l
    if not r_dense:
        band, bw = p.resistance_band()
        out["r_band"] = nat.device_colmajor(band)  # (N, bw + 1): column-major (bw + 1) x N
        out["r_bw"] = bw
    return out


def drive_table(kind: str, steps: int, dt: float, n_ports: int, n_sources: int,
                plate: Plate | None = None):
    """Drive samples at t_k = k*dt, k = 0..steps: (i_d (steps+1, n_p), i0 (steps+1, n_s)).
    Sinusoids follow the reference sampler (transient.py:198-245): sum of
    amp*sin(omega*t + phase) with omega = 2*pi*f."""
    t = dt * np.arange(steps + 1)
    i_d = np.zeros((steps + 1, n_ports))
    i0 = np.zeros((steps + 1, n_sources))
    if kind == "tone10k":
        i0[:, 0] = 1.0 * np.sin(2 * np.pi * 1e4 * t + 0.0)
    elif kind == "tone50k":
        i0[:, 0] = 1.0 * np.sin(2 * np.pi * 5e4 * t + 0.0)
        i_d[:, 0] = np.minimum(t / 5e-6, 1.0)
    elif kind == "ramp5us":
        i_d[:, 0] = np.minimum(t / 5e-6, 1.0)
    elif kind == "trapezoid":
        t_end = steps * dt
        rise = np.minimum(t / 5e-6, 1.0)
        fall = np.clip((t_end / 2 + 5e-6 - t) / 5e-6, 0.0, 1.0)
        i_d[:, 0] = np.minimum(rise, fall)
    elif kind == "batched":
        f, ph = plate.tones(n_sources)
        i0[:] = np.sin(2 * np.pi * f[None, :] * t[:, None] + ph[None, :])
    else:
        raise ValueError(kind)
    return i_d, i0
