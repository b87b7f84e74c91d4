"""Substrate pieces the hot-path API needs: `as_matrix`, `WeightStack` (core.py:22-29, 89-148).

Host-side validation only; no arithmetic runs here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ShapeError

Matrix = np.ndarray
AXIS_COLUMN = "column"
AXIS_ROW = "row"


def as_matrix(a, name: str = "matrix") -> Matrix:
    """Validate and normalise to a 2-D float64 C-order array (reference core.py:22-29)."""
    m = np.ascontiguousarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got shape {m.shape}")
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise ShapeError(f"{name} must have at least one row and column, got {m.shape}")
    return m


@dataclass
class WeightStack:
    """Ordered named linear layers, Y = W_n @ X, with a TP axis tag per layer (core.py:89-118)."""

    layers: list[tuple[str, Matrix]]
    axes: list[str] = field(default_factory=list)

    def __post_init__(self):
        names = [n for n, _ in self.layers]
        if len(set(names)) != len(names):
            raise ShapeError("layer names must be unique")
        self.layers = [(n, as_matrix(w, f"layer {n!r}")) for n, w in self.layers]
        for (n0, w0), (n1, w1) in zip(self.layers, self.layers[1:]):
            if w1.shape[1] != w0.shape[0]:
                raise ShapeError(f"layer {n1!r} input dim {w1.shape[1]} does not match layer {n0!r} "
                                 f"output dim {w0.shape[0]}")
        if not self.axes:
            self.axes = [AXIS_COLUMN] * len(self.layers)
        if len(self.axes) != len(self.layers):
            raise ShapeError("one axis tag required per layer")
        for ax in self.axes:
            if ax not in (AXIS_COLUMN, AXIS_ROW):
                raise ShapeError(f"unknown partition axis {ax!r}")

    def __len__(self) -> int:
        return len(self.layers)

    @property
    def names(self) -> list[str]:
        return [n for n, _ in self.layers]

    @property
    def weights(self) -> list[Matrix]:
        return [w for _, w in self.layers]

    def input_dim(self) -> int:
        return self.layers[0][1].shape[1]
