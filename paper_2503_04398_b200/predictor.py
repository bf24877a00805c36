"""Serving-side table types the online path reads (host mirror).

Mirrors the two table types of the reference the hot path consumes —
`TokenDeviceTable` (predictor.py:39-54) and `DeviceNGramTable`
(predictor.py:57-82) — and the history code `encode_history`
(predictor.py:149-154).  The offline builders (confidence tables, OOV
extrapolation, n-gram counting) are out of scope: bundles are
produced by the reference's solver and read with `tables.read_bundle`.

Objects of the reference's own classes are accepted everywhere these are
(duck typing on the attribute names).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PROVENANCE_PROFILED = 0
PROVENANCE_EXTRAPOLATED = 1
PROVENANCE_FALLBACK = 2


@dataclass(frozen=True)
class TokenDeviceTable:
    """𝒯 / 𝒯p: token -> cluster label (int16) with a float32 confidence."""

    labels: np.ndarray
    confidence: np.ndarray
    provenance: np.ndarray
    n_clusters: int

    def __post_init__(self):
        for name, dt in (("labels", np.int16), ("confidence", np.float32),
                         ("provenance", np.uint8)):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=dt))


@dataclass(frozen=True)
class DeviceNGramTable:
    """𝒜 / 𝒜p: E^n history rows x E next-device probabilities.

    `best` is the row argmax (first maximum wins) as int16 and `confidence`
    the row maximum as float32; unobserved rows are all-zero so their
    confidence is 0 and the token table wins the strict comparison.
    """

    n: int
    n_clusters: int
    probs: np.ndarray
    counts: np.ndarray

    @property
    def best(self) -> np.ndarray:
        return np.argmax(self.probs, axis=1).astype(np.int16)

    @property
    def confidence(self) -> np.ndarray:
        return np.max(self.probs, axis=1).astype(np.float32)

    @property
    def observed(self) -> np.ndarray:
        return np.asarray(self.counts).sum(axis=1) > 0


def encode_history(history, n_clusters: int) -> np.ndarray:
    """Base-E code of a device sequence; the newest layer is the least
    significant digit (predictor.py:149-154)."""
    h = np.asarray(history, dtype=np.int64)
    width = h.shape[-1]
    place = np.power(np.int64(n_clusters), np.arange(width - 1, -1, -1, dtype=np.int64))
    return h @ place
