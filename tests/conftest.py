"""Shared fixtures and helpers (mirrors pkg/tests/conftest.py of the reference)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(20240807)


def eigen_groups(tau, rtol=1e-8):
    """Index ranges of numerically equal time constants (reference conftest.py:62-71)."""
    groups, start = [], 0
    for i in range(1, len(tau) + 1):
        if i == len(tau) or abs(tau[i] - tau[start]) > rtol * abs(tau[start]):
            groups.append((start, i))
            start = i
    return groups


def modal_directions_match(v1, tau1, v2, tol=1e-12, rtol=1e-8):
    """Equal invariant subspaces per degenerate group (reference conftest.py:74-92):
    sign-fixed unit columns for simple modes, QR projectors for clusters."""
    for a, b in eigen_groups(tau1, rtol):
        if b - a == 1:
            x = v1[:, a] / np.linalg.norm(v1[:, a])
            y = v2[:, a] / np.linalg.norm(v2[:, a])
            if x @ y < 0:
                y = -y
            if np.abs(x - y).max() > tol:
                return False
        else:
            q1, _ = np.linalg.qr(v1[:, a:b])
            q2, _ = np.linalg.qr(v2[:, a:b])
            if np.abs(q1 @ q1.T - q2 @ q2.T).max() > tol:
                return False
    return True


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
