"""Drive waveform contract consumed by run_transient — the reference's Tone /
DriveSignal / eval_drive (pkg/src/eddymodes/network.py:208-265), unchanged in
meaning. The filament-network geometry (LoopNetwork, tube generator) is a
front end outside this hot path."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class Tone:
    amplitude: float
    frequency: float
    phase: float = 0.0


@dataclass(frozen=True)
class DriveSignal:
    """Multi-sine waveform and the ports/coils it feeds (network.py:215-242)."""

    tones: tuple[Tone, ...]
    ports: tuple[str, ...] = ()
    sources: tuple[str, ...] = ()

    def __post_init__(self):
        tones = tuple(Tone(*t) if not isinstance(t, Tone) else t for t in self.tones)
        object.__setattr__(self, "tones", tones)
        freqs = [t.frequency for t in tones]
        if any(f <= 0 for f in freqs):
            raise ValidationError("tone frequencies must be strictly positive")
        if len(set(freqs)) != len(freqs):
            raise ValidationError("tone frequencies must be distinct within a signal")
        if any(t.amplitude < 0 for t in tones):
            raise ValidationError("tone amplitudes must be >= 0")

    @property
    def frequencies(self) -> np.ndarray:
        return np.array([t.frequency for t in self.tones])


def eval_drive(signal: DriveSignal, t):
    """sum_k I_k sin(2 pi f_k t + phi_k) (network.py:244-252)."""
    t = np.asarray(t, dtype=float)
    if np.any(t < 0):
        raise ValidationError("drive evaluation requires t >= 0")
    out = np.zeros_like(t)
    for tone in signal.tones:
        out = out + tone.amplitude * np.sin(2 * math.pi * tone.frequency * t + tone.phase)
    return out if out.ndim else float(out)


def eval_drive_rate(signal: DriveSignal, t):
    """Analytic time derivative of eval_drive (network.py:255-264)."""
    t = np.asarray(t, dtype=float)
    if np.any(t < 0):
        raise ValidationError("drive evaluation requires t >= 0")
    out = np.zeros_like(t)
    for tone in signal.tones:
        w = 2 * math.pi * tone.frequency
        out = out + tone.amplitude * w * np.cos(w * t + tone.phase)
    return out if out.ndim else float(out)
