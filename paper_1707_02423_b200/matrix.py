"""Transition-matrix type and size normalisation (reference ``matrix.py``).

``TransitionMatrix`` is the hot path's input type and keeps the reference's
contract (``pkg/src/sasscfg/matrix.py:24-42``): square, nonnegative,
float64, read-only entries.  ``interpolate_to`` runs on the GPU
(``cfgsim_interpolate``) and is bit-identical to the reference's bilinear
formula (``matrix.py:74-106``); inside the pair kernel the same
interpolation is fused into the per-pair prologue.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import BadTarget

ROW_STOCHASTIC = "row_stochastic"
GLOBAL = "global"
RAW_COUNTS = "raw_counts"
INTERPOLATED = "interpolated"


@dataclass(frozen=True)
class TransitionMatrix:
    kernel_id: str
    entries: np.ndarray
    ordering: tuple[int, ...]
    mode: str

    def __post_init__(self):
        entries = np.asarray(self.entries, dtype=float)
        if entries.ndim != 2 or entries.shape[0] != entries.shape[1]:
            raise ValueError(f"entries must be square, got shape {entries.shape}")
        if (entries < 0).any():
            raise ValueError("entries must be nonnegative")
        entries.setflags(write=False)
        object.__setattr__(self, "entries", entries)

    @property
    def n(self) -> int:
        return self.entries.shape[0]


def interpolate_to(m: TransitionMatrix, target_n: int, *, device: int | None = None) -> TransitionMatrix:
    """Bilinear rescale to ``target_n`` (``matrix.py:74-106``); returns ``m``
    itself when the size already matches (``matrix.py:85-86``)."""
    if target_n < m.n:
        raise BadTarget(f"target dimension {target_n} < source dimension {m.n}")
    if target_n == m.n:
        return m
    src = np.ascontiguousarray(m.entries, dtype=np.float64)
    dst = np.empty((target_n, target_n))
    dev = nat.default_device() if device is None else device
    nat.check(nat.lib.cfgsim_interpolate(dev, m.n, nat.ptr(src), target_n, nat.ptr(dst)))
    return TransitionMatrix(m.kernel_id, dst, m.ordering, INTERPOLATED)


def normalize_pair(a: TransitionMatrix, b: TransitionMatrix, *, device: int | None = None):
    """Common size by upscaling the smaller (``matrix.py:109-114``)."""
    if a.n == b.n:
        return a, b
    target = max(a.n, b.n)
    return interpolate_to(a, target, device=device), interpolate_to(b, target, device=device)
