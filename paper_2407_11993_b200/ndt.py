"""Crack signatures: the last post-processing step of the reference's
NDT experiment (pkg/src/eddymodes/ndt.py:201-240) — defect minus background phasors per
(probe angle, tone). The experiment driver around it (tube generation, spec files) is
outside this path."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import IndexMismatch
from .frequency import PhasorSet


@dataclass(frozen=True)
class CrackSignature:
    """Complex phasor difference per (probe angle, tone) (ndt.py:201-226)."""

    entries: dict
    probe_angles: tuple

    def __getitem__(self, key):
        return self.entries[key]

    @property
    def frequencies(self) -> tuple:
        return tuple(sorted({f for (_, f) in self.entries}))

    def magnitude_by_angle(self, f: float) -> np.ndarray:
        return np.array([abs(complex(self.entries[(a, f)])) for a in self.probe_angles])

    def normalized(self) -> "CrackSignature":
        """Per tone, every entry over the largest magnitude across the probes (0 when
        the tone is identically zero)."""
        out = {}
        for f in self.frequencies:
            peak = self.magnitude_by_angle(f).max()
            for a in self.probe_angles:
                out[(a, f)] = self.entries[(a, f)] / peak if peak > 0 else 0j
        return CrackSignature(entries=out, probe_angles=self.probe_angles)


def crack_signature(defect_phasors: PhasorSet, background_phasors: PhasorSet) -> CrackSignature:
    """defect - background for every (probe, tone), keyed by probe angle (ndt.py:229-240);
    IndexMismatch unless both sets hold the same keys and probe angles."""
    if defect_phasors.entries.keys() != background_phasors.entries.keys():
        raise IndexMismatch("phasor sets do not share the same (probe, tone) keys")
    if tuple(defect_phasors.probe_angles) != tuple(background_phasors.probe_angles):
        raise IndexMismatch("phasor sets do not share probe angles")
    angles = tuple(defect_phasors.probe_angles)
    diff = {(angles[p], f): z - background_phasors.entries[(p, f)]
            for (p, f), z in defect_phasors.entries.items()}
    return CrackSignature(entries=diff, probe_angles=angles)
