"""ctypes binding of libeddymodes_b200.so (include/eddymodes_b200.h) and the
device-memory plumbing (torch tensors as FP64 device buffers, one CUDA stream
shared with torch).

There is no CPU fallback: if the library or a CUDA device is missing every
entry point raises DeviceError.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, NotPositiveDefinite

_HERE = os.path.dirname(os.path.abspath(__file__))
# EM_LIB_PATH: load another build of the same library (A/B measurements)
LIB_PATH = os.environ.get("EM_LIB_PATH") or os.path.join(_HERE, "libeddymodes_b200.so")

EM_OK, EM_ERR_CUDA, EM_ERR_ARG, EM_ERR_NOT_PD = 0, -1, -2, -3

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "em_init": (_I, [_I, ctypes.POINTER(_P)]),
    "em_finalize": (None, [_P]),
    "em_trim": (_I, [_P]),
    "em_info": (_I, [_P, _I, ctypes.POINTER(_I64)]),
    "em_set_stream": (_I, [_P, _P]),
    "em_last_error": (ctypes.c_char_p, [_P]),
    "em_launch_count": (_I64, [_P]),
    "em_synchronize": (_I, [_P]),
    "em_config": (_I, [_P, _I, _I64]),
    "em_profile": (_I, [_P, _I]),
    "em_stage_times": (_I, [_P, _P, _P, _I]),
    "em_dgemm": (_I, [_P, _I, _I, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64]),
    "em_dgemm_lower": (_I, [_P, _I, _I, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64,
                            _I64]),
    "em_comm_unique_id": (_I, [_P, _P]),
    "em_comm_init_nccl": (_I, [_P, _I, _I, _P]),
    "em_comm_init_callbacks": (_I, [_P, _I, _I, _P, _P, _P]),
    "em_comm_info": (_I, [_P, ctypes.POINTER(_I64)]),
    "em_comm_destroy": (_I, [_P]),
    "em_dsymm_band_lower": (_I, [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _I64]),
    "em_sym_mirror_lower": (_I, [_P, _I64, _P, _I64]),
    "em_sym_mm": (_I, [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _I64]),
    "em_symv_lower": (_I, [_P, _I64, _D, _P, _I64, _P, _D, _P]),
    "em_potrf": (_I, [_P, _I64, _P, _I64, ctypes.POINTER(_I64)]),
    "em_trsm_lower": (_I, [_P, _I, _I64, _I64, _P, _I64, _P, _I64]),
    "em_syev": (_I, [_P, _I64, _P, _I64, _P, _P, _I64]),
    "em_sygv": (_I, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64,
                     ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_ex": (_I, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _I,
                        ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_range": (_I, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P,
                           _I64, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_implicit": (_I, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _I64, _P, _P, _I,
                              ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_implicit_band": (_I, [_P, _I64, _P, _I64, _P, _I64, _I64, _P, _P, _I64, _I64, _P,
                                   _P, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_lh": (_I, [_P, _I64, _P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _I,
                        ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    "em_sygv_h": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I64),
                       ctypes.POINTER(_I)]),
    "em_td2_plan_create": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P, _P, _D, _D, ctypes.POINTER(_P)]),
    "em_td2_plan_create_exact": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P, _P, _D,
                                      ctypes.POINTER(_P)]),
    "em_td2_plan_destroy": (None, [_P]),
    "em_td2_set_observables": (_I, [_P, _I, _P, _I64, _P, _I64]),
    "em_td2_run": (_I, [_P, _I64, _P, _P, _P, _I64, _P]),
    "em_td2_run_sweep": (_I, [_P, _I64, _P, _P, _P, _I64]),
    "em_td2_step": (_I, [_P, _P, _P, _P, _P]),
    "em_td2_forcing": (_I, [_P, _P, _P, _P, _P]),
    "em_td2_step_forcing": (_I, [_P, _P, _P]),
    "em_td1_plan_create": (_I, [_P, _I64, _I, _I, _P, _I64, _P, _I64, _P, _P, _P, _D, _D,
                                ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "em_td1_plan_create_band": (_I, [_P, _I64, _I, _I, _P, _I64, _P, _I64, _I64, _P, _P, _P, _D,
                                     _D, _I, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "em_td1_plan_destroy": (None, [_P]),
    "em_td1_set_observables": (_I, [_P, _I, _P, _I64, _P, _I64]),
    "em_td1_run": (_I, [_P, _I64, _P, _P, _P, _I64, _P]),
    "em_td1_step": (_I, [_P, _P, _P, _P, _P]),
    "em_td1_factor": (_I, [_P, _P, _I64]),
    "em_fd_plan_create": (_I, [_P, _I64, _P, _I64, _P, _I64, ctypes.POINTER(_P),
                               ctypes.POINTER(_I64)]),
    "em_fd_plan_destroy": (None, [_P]),
    "em_fd_solve": (_I, [_P, _D, _P, _P, _P, _P, ctypes.POINTER(_I64)]),
    "em_tone_table": (_I, [_P, _I64, _D, _D, _I, _P, _P, _I64]),
    "em_field_transfer": (_I, [_P, _I64, _P, _P, _P, _I64, _P, _P, ctypes.POINTER(_I64)]),
    "em_synth_plate": (_I, [_P, _I64, _I64, _I64, _D, _D, _D, _I64, _P, _P, _P, _P, _I64, _P,
                            _I64, _P, _P]),
}

_lib = None
_ctx = None
_lock = threading.Lock()


def load_library() -> ctypes.CDLL:
    """Load the shared library (no device needed) and bind every symbol."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("EM_LIB_PATH") and not hasattr(lib, name):
                continue  # an older build under A/B: bind what it has
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def torch():
    import torch as _t
    return _t


def context():
    """The process-wide em_ctx on the current CUDA device, bound to torch's stream."""
    global _ctx
    with _lock:
        if _ctx is None:
            t = torch()
            if not t.cuda.is_available():
                raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
            lib = load_library()
            dev = t.cuda.current_device()
            ctx = _P()
            rc = lib.em_init(dev, ctypes.byref(ctx))
            if rc != EM_OK:
                raise DeviceError(f"em_init failed ({rc})")
            stream = t.cuda.current_stream(dev).cuda_stream
            rc = lib.em_set_stream(ctx, _P(stream))
            if rc != EM_OK:
                raise DeviceError("em_set_stream failed")
            _ctx = ctx
        return _ctx


def check(rc: int, what: str = "") -> None:
    if rc == EM_OK:
        return
    msg = load_library().em_last_error(_ctx)
    msg = msg.decode() if msg else ""
    raise DeviceError(f"{what}: error {rc} {msg}".strip())


def launches() -> int:
    return int(load_library().em_launch_count(_ctx))


STAGES = ("potrf_R", "sygst", "potrf_L", "sytrd", "stedc", "ormtr", "trsm_back", "finalize",
          "post_gemm", "td2_local", "td2_carry", "td2_replay", "td1_symv", "td1_fwd", "td1_bwd",
          "sytrd_symv", "sytrd_syr2k", "stedc_gemm", "stedc_secular", "sy2sb", "sb2st", "q2_apply",
          "q1_apply", "sy2sb_qr")


def profile(level: int = 1) -> None:
    """0 off, 1 top-level stages, 2 also per-call inner stages (sytrd symv, D&C GEMMs)."""
    check(load_library().em_profile(context(), int(level)), "em_profile")


def stage_times() -> dict:
    """{stage: (milliseconds, event pairs)} accumulated since profile(True)."""
    n = len(STAGES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    rc = load_library().em_stage_times(context(), ms, cnt, n)
    if rc < 0:
        check(rc, "em_stage_times")
    return {STAGES[i]: (ms[i], cnt[i]) for i in range(n) if cnt[i]}


EM_SYGV_R_WORKSPACE, EM_SYGV_L_WORKSPACE = 1, 2
EM_TD1_L_WORKSPACE = 1
EM_CFG_TWO_STAGE_MIN = 1


TWO_STAGE_MIN_DEFAULT = 16000  # the library's default (csrc/sygv.cu g_two_stage_min)


def set_two_stage_min(n: int) -> None:
    """Smallest order that uses the two-stage tridiagonalisation (library default
    TWO_STAGE_MIN_DEFAULT, and only when its extra storage fits on the device)."""
    check(load_library().em_config(context(), EM_CFG_TWO_STAGE_MIN, int(n)), "em_config")


def trim() -> None:
    """Release the device memory the library keeps cached between calls (em_trim)."""
    check(load_library().em_trim(context()), "em_trim")


def last_eig_path() -> int:
    """1 = one-stage, 2 = two-stage tridiagonalisation in the last eigensolve (em_info)."""
    v = ctypes.c_int64(0)
    check(load_library().em_info(context(), 1, ctypes.byref(v)), "em_info")
    return int(v.value)


def synchronize() -> None:
    torch().cuda.current_stream().synchronize()


# --- device buffers ------------------------------------------------------------------
# A column-major (m x n) device matrix is held as a torch tensor of shape (n, m),
# contiguous: element (i, j) lives at j*m + i.

def device_colmajor(a: np.ndarray):
    """Host (m x n) matrix -> device column-major buffer (tensor shaped (n, m))."""
    t = torch()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    return t.from_numpy(np.ascontiguousarray(a.T)).to("cuda")


def device_symmetric(a: np.ndarray):
    """Upload an EXACTLY symmetric host matrix (e.g. SymMatrix.full): its row-major
    bytes are its column-major bytes, so no host transpose copy is made."""
    t = torch()
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def device_vector(x: np.ndarray):
    t = torch()
    return t.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to("cuda")


def empty(*shape):
    t = torch()
    return t.empty(*shape, dtype=t.float64, device="cuda")


def zeros(*shape):
    t = torch()
    return t.zeros(*shape, dtype=t.float64, device="cuda")


def host_colmajor(buf, m: int, n: int) -> np.ndarray:
    """Device column-major buffer (tensor (n, m)) -> host C-contiguous (m x n)."""
    return np.ascontiguousarray(buf.reshape(n, m).cpu().numpy().T)


def ptr(t) -> _P:
    return _P(t.data_ptr()) if t is not None else _P(0)


def raise_not_pd(rc: int, pivot: int, what: str) -> None:
    if rc == EM_ERR_NOT_PD:
        raise NotPositiveDefinite(int(pivot), what)
