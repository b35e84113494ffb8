"""paper_2407_11993_b200: B200-native (sm_100a) modal-decomposition transient
solver — a drop-in for the hot path of the reference package `eddymodes`
(arXiv 2407.11993): generalized eigensolve, modal theta-method (TD2) and the
Cholesky theta-method comparator (TD1), behind the reference's solver API.

    from paper_2407_11993_b200 import modal, transient, linalg, reduction
    basis = modal.generalized_eig(rm.l_i, rm.r_i)
    res = transient.run_transient(rm, None, drive, cfg, modal=basis)

The numerics run in libeddymodes_b200.so (hand-written CUDA for sm_100a,
include/eddymodes_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import errors, linalg, modal, network, reduction, synth, transient  # noqa: F401
from .errors import EddymodesError  # noqa: F401
