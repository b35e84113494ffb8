"""Model and eigenbasis storage, mirroring `eddymodes.matrixio`
(E/matrixio.py) plus the binary formats the text cache cannot serve at N >= 16k.

* `write_cache` / `read_cache`: the reference's line-oriented text cache
  (E/matrixio.py:27-131), same grammar and the same bytes for the same model (repr of
  every float). The `model` section (filament network text) belongs to the geometry
  front end outside this path: it is skipped on read (net = None) and `net` must be
  None on write.
* `write_cache_binary` / `read_cache_binary`: the same content as one binary file:
  a JSON header (names, shapes, the basis counts) followed by raw little-endian FP64 /
  int64 blocks; symmetric R_I, L_I are stored as their packed lower triangles (half
  the bytes). A C2 model (N = 16,384) is 2.2 GB instead of ~20 GB of text.
* `save_basis` / `load_basis`: a ModalBasis (V, V^T R, tau, l_n, r_n) straight from /
  to device memory, streamed through pinned host buffers in 256 MB chunks with the
  device copies of one chunk overlapping the file I/O of the other (an eigenbasis
  computed once serves every later drive and time step).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import linalg
from .errors import ParseError, ValidationError
from .modal import ModalBasis
from .reduction import ReducedModel, project_external


@dataclass(frozen=True)
class CurrentBasis:
    """Branch-current basis carried by a cache (E/assembly.py:153-170): w (branches x
    basis vectors, entries in {-1, 0, +1}), fundamental cycles then electrode paths."""

    w: np.ndarray
    n_cycles: int
    n_paths: int


# --- text cache (E/matrixio.py) ------------------------------------------------------

def _write_matrix(fh, name: str, m: np.ndarray, integer: bool):
    m = np.atleast_2d(m)
    kind = "i" if integer else "f"
    fh.write(f"matrix {name} {m.shape[0]} {m.shape[1]} {kind}\n")
    for row in m:
        if integer:
            fh.write(" ".join(str(int(v)) for v in row) + "\n")
        else:
            fh.write(" ".join(repr(float(v)) for v in row) + "\n")


def write_cache(path, rm: ReducedModel, net=None, e: np.ndarray | None = None,
                header_lines: tuple[str, ...] = ()):
    """E/matrixio.py:38-62."""
    if net is not None:
        raise ValidationError("the network model section needs the geometry front end; "
                              "pass net=None")
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(f"# {line}\n")
        fh.write(f"meta ports {','.join(rm.port_names) or '-'}\n")
        fh.write(f"meta sources {','.join(rm.source_names) or '-'}\n")
        _write_matrix(fh, "R_I", rm.r_i.full, False)
        _write_matrix(fh, "L_I", rm.l_i.full, False)
        _write_matrix(fh, "R_D", rm.r_d, False)
        _write_matrix(fh, "L_D", rm.l_d, False)
        _write_matrix(fh, "M0", rm.m0, False)
        _write_matrix(fh, "LIFT", rm.lift, False)
        _write_matrix(fh, "K", rm.k, False)
        if e is not None:
            _write_matrix(fh, "E", e, True)
        if rm.basis is not None:
            fh.write(f"meta basis {rm.basis.n_cycles} {rm.basis.n_paths}\n")
            _write_matrix(fh, "W", rm.basis.w, True)


def _assemble(matrices: dict, ports, sources, basis_counts):
    if "R_I" in matrices:
        needed = {"L_I", "R_D", "L_D", "M0", "LIFT", "K"}
        missing = needed - set(matrices)
        if missing:
            raise ParseError(f"cache is missing matrices: {sorted(missing)}", None)
        basis = None
        if basis_counts is not None and "W" in matrices:
            basis = CurrentBasis(w=matrices["W"].astype(np.int64), n_cycles=basis_counts[0],
                                 n_paths=basis_counts[1])
        return ReducedModel(r_i=linalg.SymMatrix(matrices["R_I"]),
                            l_i=linalg.SymMatrix(matrices["L_I"]),
                            r_d=matrices["R_D"], l_d=matrices["L_D"], m0=matrices["M0"],
                            lift=matrices["LIFT"], k=matrices["K"], basis=basis,
                            source_names=tuple(sources), port_names=tuple(ports))
    if {"R_X", "L_X", "E"} <= set(matrices):
        return project_external(matrices["R_X"], matrices["L_X"],
                                matrices["E"].astype(np.int64), port_names=tuple(ports))
    raise ParseError("cache holds neither a reduced model nor an R_X/L_X/E triple", None)


def read_cache(path):
    """E/matrixio.py:65-131. Returns (ReducedModel, None): a `model` section is skipped."""
    matrices: dict[str, np.ndarray] = {}
    meta: dict[str, list[str]] = {}
    basis_counts = None
    with open(path) as fh:
        lines = fh.read().splitlines()
    i, n = 0, len(lines)
    while i < n:
        line = lines[i].strip()
        i += 1
        if not line or line.startswith("#"):
            continue
        toks = line.split()
        if toks[0] == "model":
            i += int(toks[1])
        elif toks[0] == "meta" and toks[1] in ("ports", "sources"):
            val = toks[2] if len(toks) > 2 else "-"
            meta[toks[1]] = [] if val == "-" else val.split(",")
        elif toks[0] == "meta" and toks[1] == "basis":
            basis_counts = (int(toks[2]), int(toks[3]))
        elif toks[0] == "matrix":
            name, rows, cols, kind = toks[1], int(toks[2]), int(toks[3]), toks[4]
            data = []
            for r in range(rows):
                vals = lines[i + r].split()
                if len(vals) != cols:
                    raise ParseError(f"matrix {name}: row {r} has {len(vals)} "
                                     f"values, expected {cols}", i + r + 1)
                data.append([float(v) for v in vals])
            i += rows
            arr = np.array(data) if rows else np.zeros((0, cols))
            matrices[name] = arr.astype(np.int64) if kind == "i" else arr
        else:
            raise ParseError(f"unrecognized cache line: {line!r}", i)
    return _assemble(matrices, meta.get("ports", []), meta.get("sources", []),
                     basis_counts), None


# --- binary model cache -----------------------------------------------------------------

_MAGIC_MODEL = b"EMB200M1"
_MAGIC_BASIS = b"EMB200B1"


def _packed_lower(a: np.ndarray) -> np.ndarray:
    return a[np.tril_indices(a.shape[0])]


def _unpack_lower(p: np.ndarray, n: int) -> np.ndarray:
    a = np.zeros((n, n))
    a[np.tril_indices(n)] = p
    return a  # SymMatrix mirrors the lower triangle


def _write_blob(path, magic: bytes, header: dict, blocks: list[np.ndarray]):
    hb = json.dumps(header).encode()
    with open(path, "wb") as fh:
        fh.write(magic)
        fh.write(np.array([len(hb)], dtype="<u8").tobytes())
        fh.write(hb)
        for b in blocks:
            fh.write(np.ascontiguousarray(b).astype(b.dtype.newbyteorder("<"), copy=False)
                     .tobytes())


def _read_header(fh, magic: bytes) -> dict:
    if fh.read(len(magic)) != magic:
        raise ParseError("not an eddymodes-b200 binary file of this kind", None)
    hl = int(np.frombuffer(fh.read(8), dtype="<u8")[0])
    return json.loads(fh.read(hl).decode())


def write_cache_binary(path, rm: ReducedModel, e: np.ndarray | None = None):
    """The text cache's content in one binary file (symmetric blocks packed)."""
    n = rm.n_internal
    entries, blocks = [], []

    def add(name, arr, kind, packed=False):
        arr = np.asarray(arr)
        entries.append({"name": name, "shape": list(arr.shape), "kind": kind, "packed": packed})
        blocks.append(_packed_lower(arr) if packed else arr.astype("<f8" if kind == "f"
                                                                  else "<i8"))

    add("R_I", rm.r_i.full, "f", True)
    add("L_I", rm.l_i.full, "f", True)
    for name, arr in (("R_D", rm.r_d), ("L_D", rm.l_d), ("M0", rm.m0), ("LIFT", rm.lift),
                      ("K", rm.k)):
        add(name, np.asarray(arr, dtype=float), "f")
    if e is not None:
        add("E", np.asarray(e, dtype=np.int64), "i")
    header = {"n": n, "ports": list(rm.port_names), "sources": list(rm.source_names),
              "matrices": entries}
    if rm.basis is not None:
        add("W", np.asarray(rm.basis.w, dtype=np.int64), "i")
        header["basis"] = [int(rm.basis.n_cycles), int(rm.basis.n_paths)]
    _write_blob(path, _MAGIC_MODEL, header, blocks)


def read_cache_binary(path):
    """Inverse of write_cache_binary. Returns (ReducedModel, None)."""
    with open(path, "rb") as fh:
        h = _read_header(fh, _MAGIC_MODEL)
        matrices = {}
        for ent in h["matrices"]:
            shape = tuple(ent["shape"])
            if ent["packed"]:
                cnt = shape[0] * (shape[0] + 1) // 2
                p = np.frombuffer(fh.read(8 * cnt), dtype="<f8")
                matrices[ent["name"]] = _unpack_lower(p, shape[0])
            else:
                cnt = int(np.prod(shape)) if shape else 1
                dt = "<f8" if ent["kind"] == "f" else "<i8"
                a = np.frombuffer(fh.read(8 * cnt), dtype=dt).reshape(shape)
                matrices[ent["name"]] = a.astype(np.float64 if ent["kind"] == "f" else np.int64)
    counts = tuple(h["basis"]) if "basis" in h else None
    return _assemble(matrices, h["ports"], h["sources"], counts), None


# --- eigenbasis (device <-> file) ---------------------------------------------------------

_CHUNK = 256 << 20  # bytes per pinned staging buffer


def _stream_out(fh, dev_flat) -> None:
    """Device 1-D float64 tensor -> file, double-buffered through pinned memory."""
    t = nat.torch()
    n = dev_flat.numel()
    step = _CHUNK // 8
    bufs = [t.empty(min(step, max(n, 1)), dtype=t.float64, pin_memory=True) for _ in range(2)]
    evs = [t.cuda.Event(), t.cuda.Event()]
    stream = t.cuda.Stream()
    pending = None
    for k, off in enumerate(range(0, n, step)):
        m = min(step, n - off)
        b = bufs[k & 1]
        with t.cuda.stream(stream):
            stream.wait_stream(t.cuda.current_stream())
            b[:m].copy_(dev_flat[off:off + m], non_blocking=True)
            evs[k & 1].record(stream)
        if pending is not None:  # write the previous chunk while this one copies
            pb, pm, pe = pending
            pe.synchronize()
            fh.write(pb[:pm].numpy().tobytes())
        pending = (b, m, evs[k & 1])
    if pending is not None:
        pb, pm, pe = pending
        pe.synchronize()
        fh.write(pb[:pm].numpy().tobytes())


def _stream_in(fh, count: int):
    """File -> new device 1-D float64 tensor of `count` values, double-buffered."""
    t = nat.torch()
    out = t.empty(max(count, 1), dtype=t.float64, device="cuda")
    step = _CHUNK // 8
    bufs = [t.empty(min(step, max(count, 1)), dtype=t.float64, pin_memory=True)
            for _ in range(2)]
    evs = [None, None]
    stream = t.cuda.Stream()
    for k, off in enumerate(range(0, count, step)):
        m = min(step, count - off)
        b = bufs[k & 1]
        if evs[k & 1] is not None:
            evs[k & 1].synchronize()  # the copy that used this buffer is done
        raw = fh.read(8 * m)
        if len(raw) != 8 * m:
            raise ParseError("truncated eigenbasis file", None)
        b[:m].numpy()[:] = np.frombuffer(raw, dtype="<f8")
        with t.cuda.stream(stream):
            out[off:off + m].copy_(b[:m], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(stream)
            evs[k & 1] = ev
    t.cuda.current_stream().wait_stream(stream)
    stream.synchronize()
    return out[:count]


def save_basis(path, basis: ModalBasis) -> None:
    """Write tau, l_n, r_n and the device V, R V (column-major) to one binary file."""
    n = basis.n_modes
    header = {"n": n, "layout": "V and RV column-major float64 (RV == V^T R row-major)"}
    hb = json.dumps(header).encode()
    with open(path, "wb") as fh:
        fh.write(_MAGIC_BASIS)
        fh.write(np.array([len(hb)], dtype="<u8").tobytes())
        fh.write(hb)
        for vec in (basis.tau, basis.l_n, basis.r_n):
            fh.write(np.ascontiguousarray(vec, dtype="<f8").tobytes())
        if n:
            _stream_out(fh, basis.v_dev.reshape(-1))
            _stream_out(fh, basis.vtr_dev.reshape(-1))


def load_basis(path) -> ModalBasis:
    """Inverse of save_basis: V and V^T R land directly in device memory (host copies
    only on access, as for a freshly computed basis)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        h = _read_header(fh, _MAGIC_BASIS)
        n = int(h["n"])
        vecs = [np.frombuffer(fh.read(8 * n), dtype="<f8").astype(np.float64) for _ in range(3)]
        if n == 0:
            z = np.zeros((0, 0))
            return ModalBasis(v=z, tau=vecs[0], l_n=vecs[1], r_n=vecs[2], vt_r=z)
        if size < fh.tell() + 16 * n * n:
            raise ParseError("truncated eigenbasis file", None)
        v = _stream_in(fh, n * n).reshape(n, n)
        vtr = _stream_in(fh, n * n).reshape(n, n)
    return ModalBasis(tau=vecs[0], l_n=vecs[1], r_n=vecs[2], v_dev=v, vtr_dev=vtr)
